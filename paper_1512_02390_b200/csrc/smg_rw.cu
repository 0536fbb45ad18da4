// Restriction without a halo: one warp per FINE element, ring + fixup
// (subsystem 3; multigrid.py:188-193 restrict_residual, :112-124 row-assigned P).
//
// restrict_kernel (smg_transfer.cu) stages, per coarse element, the fine
// element AND its left / lower / corner neighbours (their high-side vertex
// terms), and runs the full passes on the halo too: at p_f = 32 it executes
// 3.1x the algorithmic FMAs and reads every fine value four times from L2
// (ncu: FP64 pipe 46 % busy for a bandwidth-bound operation, long-scoreboard
// and barrier stalls).  Here a warp owns one fine element and nothing else:
//   y pass: lane b = fine column; the p_f rows stream from global memory
//           (coalesced row segments, no shared-memory staging) into
//           t[ay] = sum_{a<p_f} J[a][ay] F[a][b], ay = 0..p_c;
//   x pass: lane ay = coarse row; C[ay][ax] = sum_{b<p_f} J[b][ax] T[ay][b]
//           with T read from a per-warp shared buffer (odd pitch) and J as
//           uniform parameter-bank operands;
//   the own coarse nodes (ay, ax < p_c) are written coalesced; the high-side
//   row and column (ay = p_c or ax = p_c: nodes owned by the upper / right /
//   corner elements) go to a ring workspace of 2 p_c + 1 doubles per element.
// restrict_fixup adds the three ring terms to the low-side nodes in a fixed
// order (lower, left, corner): deterministic, no atomics.
#include "smg_transfer.cuh"

namespace smg {

constexpr int kRwWarps = 4;

template <int PC, int PF>
__global__ void __launch_bounds__(32 * kRwWarps) restrict_warp_kernel(const __grid_constant__ TrArgs A,
                                                                      double* __restrict__ ring) {
  SMG_PDL_ENTRY();
  constexpr int NC = PC + 1, TP = PF | 1, CP = NC | 1;   // odd pitches: conflict-free row reads
  static_assert(PF <= 32 && NC <= 32, "one lane per fine column / coarse row");
  __shared__ double Ts[kRwWarps][NC * TP];
  __shared__ double Cs[kRwWarps][NC * CP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * kRwWarps + warp;
  const int n_el = A.n_x * A.n_y;
  if (e >= n_el) return;
  const int ey = e / A.n_x, ex = e - ey * A.n_x;
  const int Nxf = A.n_x * PF, Nxc = A.n_x * PC;
  double* T = Ts[warp];
  double* C = Cs[warp];
  // ---- y pass (lane = fine column b)
  if (lane < PF) {
    const double* col = A.src + (size_t)(ey * PF) * Nxf + ex * PF + lane;
    double t[NC];
#pragma unroll
    for (int ay = 0; ay < NC; ++ay) t[ay] = 0.0;
    // chunks of CH rows, the next chunk's loads issued before this chunk's FMAs (ncu: 63 %
    // of the stall samples sat on the first FMA of a chunk waiting for its loads)
    constexpr int CH = 8;
    static_assert(PF % CH == 0, "row chunks");
    double f[CH], g[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) f[q] = col[(size_t)q * Nxf];
#pragma unroll
    for (int a0 = 0; a0 < PF; a0 += CH) {
      if (a0 + CH < PF) {
#pragma unroll
        for (int q = 0; q < CH; ++q) g[q] = col[(size_t)(a0 + CH + q) * Nxf];
      }
#pragma unroll
      for (int q = 0; q < CH; ++q)
#pragma unroll
        for (int ay = 0; ay < NC; ++ay) t[ay] = fma(A.J[(a0 + q) * NC + ay], f[q], t[ay]);
#pragma unroll
      for (int q = 0; q < CH; ++q) f[q] = g[q];
    }
#pragma unroll
    for (int ay = 0; ay < NC; ++ay) T[ay * TP + lane] = t[ay];
  }
  __syncwarp();
  // ---- x pass (lane = coarse row ay)
  if (lane < NC) {
    const double* trow = T + lane * TP;
    double c[NC];
#pragma unroll
    for (int ax = 0; ax < NC; ++ax) c[ax] = 0.0;
#pragma unroll
    for (int b = 0; b < PF; ++b) {
      const double tb = trow[b];
#pragma unroll
      for (int ax = 0; ax < NC; ++ax) c[ax] = fma(A.J[b * NC + ax], tb, c[ax]);
    }
#pragma unroll
    for (int ax = 0; ax < NC; ++ax) C[lane * CP + ax] = c[ax];
  }
  __syncwarp();
  // ---- own coarse nodes, coalesced rows of p_c doubles
  for (int idx = lane; idx < PC * PC; idx += 32) {
    const int ay = idx / PC, ax = idx - ay * PC;
    A.dst[(size_t)(ey * PC + ay) * Nxc + ex * PC + ax] = C[ay * CP + ax];
  }
  // ---- ring: [0, p_c] the top row (ay = p_c, corner last), then the right column ay = 0..p_c-1
  double* R = ring + (size_t)e * (2 * PC + 1);
  for (int k = lane; k < 2 * PC + 1; k += 32) R[k] = k <= PC ? C[PC * CP + k] : C[(k - PC - 1) * CP + PC];
}

// One thread per low-side coarse node of an element: bottom row (ay = 0, ax = 0..p_c-1), then
// the left column (ax = 0, ay = 1..p_c-1).
template <int PC>
__global__ void __launch_bounds__(256) restrict_fixup(double* __restrict__ dst, const double* __restrict__ ring,
                                                      int n_x, int n_y) {
  SMG_PDL_ENTRY();
  constexpr int PER = 2 * PC - 1, RS = 2 * PC + 1;
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long)n_x * n_y * PER) return;
  const int e = (int)(gid / PER), k = (int)(gid - (long)e * PER);
  const int ey = e / n_x, ex = e - ey * n_x;
  const int ay = k < PC ? 0 : k - PC + 1, ax = k < PC ? k : 0;
  const int eyl = wrapi(ey - 1, n_y), exl = wrapi(ex - 1, n_x);
  double* d = dst + (size_t)(ey * PC + ay) * ((size_t)n_x * PC) + ex * PC + ax;
  double v = *d;
  if (ay == 0) v += ring[(size_t)(eyl * n_x + ex) * RS + ax];                 // top row of the lower element
  if (ax == 0) v += ring[(size_t)(ey * n_x + exl) * RS + PC + 1 + ay];        // right column of the left element
  if (ay == 0 && ax == 0) v += ring[(size_t)(eyl * n_x + exl) * RS + PC];     // corner of the lower-left element
  *d = v;
}

template <int PC, int PF>
int rw_launch(const TrArgs& A, double* ring, cudaStream_t st) {
  const int n_el = A.n_x * A.n_y;
  launch(restrict_warp_kernel<PC, PF>, dim3((n_el + kRwWarps - 1) / kRwWarps), dim3(32 * kRwWarps), 0, st, A, ring);
  int rc = check_launch("restrict_warp_kernel");
  if (rc) return rc;
  const long nb = (long)n_el * (2 * PC - 1);
  launch(restrict_fixup<PC>, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, st, A.dst, (const double*)ring, A.n_x,
         A.n_y);
  return check_launch("restrict_fixup");
}

// Prolongation, one warp per fine element (multigrid.py:180-185; same passes as the
// restriction above, transposed): the element's (p_c+1)^2 coarse values land in a per-warp
// buffer; x pass: lane ay = coarse row, T[ay][b] = sum_ax J[b][ax] C[ay][ax] for the p_f
// owned fine columns (J as uniform operands, 4 columns in flight); y pass: lane b = fine
// column, out[a][b] (+)= sum_ay J[a][ay] T[ay][b], 8 rows in flight, rows written coalesced.
// No halo beyond the element's own high-side coarse nodes, no ring.
template <int PC, int PF>
__global__ void __launch_bounds__(32 * kRwWarps) prolong_rw_kernel(const __grid_constant__ TrArgs A) {
  SMG_PDL_ENTRY();
  constexpr int NC = PC + 1, TP = PF | 1, CP = NC | 1;
  static_assert(PF <= 32 && NC <= 32, "one lane per fine column / coarse row");
  __shared__ double Ts[kRwWarps][NC * TP];
  __shared__ double Cs[kRwWarps][NC * CP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * kRwWarps + warp;
  const int n_el = A.n_x * A.n_y;
  if (e >= n_el) return;
  const int ey = e / A.n_x, ex = e - ey * A.n_x;
  const int Nxf = A.n_x * PF, Nxc = A.n_x * PC, Nyc = A.n_y * PC;
  double* T = Ts[warp];
  double* C = Cs[warp];
  for (int i = lane; i < NC * NC; i += 32) {
    const int ay = i / NC, ax = i - ay * NC;
    C[ay * CP + ax] = A.src[(size_t)wrapi(ey * PC + ay, Nyc) * Nxc + wrapi(ex * PC + ax, Nxc)];
  }
  __syncwarp();
  // ---- x pass (lane = coarse row ay)
  if (lane < NC) {
    double c[NC];
#pragma unroll
    for (int ax = 0; ax < NC; ++ax) c[ax] = C[lane * CP + ax];
    constexpr int BB = 4;
    static_assert(PF % BB == 0, "fine columns in flight");
#pragma unroll
    for (int b0 = 0; b0 < PF; b0 += BB) {
      double t[BB];
#pragma unroll
      for (int q = 0; q < BB; ++q) t[q] = 0.0;
#pragma unroll
      for (int ax = 0; ax < NC; ++ax)
#pragma unroll
        for (int q = 0; q < BB; ++q) t[q] = fma(A.J[(b0 + q) * NC + ax], c[ax], t[q]);
#pragma unroll
      for (int q = 0; q < BB; ++q) T[lane * TP + b0 + q] = t[q];
    }
  }
  __syncwarp();
  // ---- y pass (lane = fine column b)
  if (lane < PF) {
    double t[NC];
#pragma unroll
    for (int ay = 0; ay < NC; ++ay) t[ay] = T[ay * TP + lane];
    double* out = A.dst + (size_t)(ey * PF) * Nxf + ex * PF + lane;
    constexpr int CH = 8;
    static_assert(PF % CH == 0, "row chunks");
#pragma unroll
    for (int a0 = 0; a0 < PF; a0 += CH) {
      double o[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) o[q] = A.accumulate ? out[(size_t)(a0 + q) * Nxf] : 0.0;
      double s[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) s[q] = 0.0;
#pragma unroll
      for (int ay = 0; ay < NC; ++ay)
#pragma unroll
        for (int q = 0; q < CH; ++q) s[q] = fma(A.J[(a0 + q) * NC + ay], t[ay], s[q]);
#pragma unroll
      for (int q = 0; q < CH; ++q) out[(size_t)(a0 + q) * Nxf] = A.accumulate ? o[q] + s[q] : s[q];
    }
  }
}

template <int PC, int PF>
int prw_launch(const TrArgs& A, cudaStream_t st) {
  const int n_el = A.n_x * A.n_y;
  launch(prolong_rw_kernel<PC, PF>, dim3((n_el + kRwWarps - 1) / kRwWarps), dim3(32 * kRwWarps), 0, st, A);
  return check_launch("prolong_rw_kernel");
}

// restrict_fixup alone (the fused residual + restriction of smg_opw.cu filled dst and the ring)
int rw_fixup(int pc, double* dst, const double* ring, int n_x, int n_y, cudaStream_t st) {
  if (pc != 8 && pc != 4 && pc != 2) return 1;
  const long nb = (long)n_x * n_y * (2 * pc - 1);
  if (pc == 8) launch(restrict_fixup<8>, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, st, dst, ring, n_x, n_y);
  else if (pc == 4) launch(restrict_fixup<4>, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, st, dst, ring, n_x, n_y);
  else launch(restrict_fixup<2>, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, st, dst, ring, n_x, n_y);
  return check_launch("restrict_fixup");
}

PrwFn prw_dispatch(int pc, int pf) {
  if (pc == 16 && pf == 32) return &prw_launch<16, 32>;
  if (pc == 12 && pf == 24) return &prw_launch<12, 24>;
  if (pc == 8 && pf == 16) return &prw_launch<8, 16>;
  return nullptr;
}

RwFn rw_dispatch(int pc, int pf) {
  if (pc == 16 && pf == 32) return &rw_launch<16, 32>;
  if (pc == 12 && pf == 24) return &rw_launch<12, 24>;
  if (pc == 8 && pf == 16) return &rw_launch<8, 16>;
  return nullptr;
}

}  // namespace smg
