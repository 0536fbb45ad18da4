// Single-launch tiled additive-Schwarz kernel (subsystem 1).
//
// Same math as the coloured dense kernel in smg_fd.cuh (schwarz.py:215-222,
// 268-275; mesh.py:124-150) with three changes:
//
// 1. Even/odd fast diagonalization.  The restricted 1D subdomain problem is
//    reflection-symmetric, so each generalized eigenvector is even or odd.
//    A contraction with S folds into two half-size contractions,
//      (S^T x)_even = Se^T (x_k + x_{m-1-k}),  (S^T x)_odd = So^T (x_k - x_{m-1-k}),
//    and S t unfolds the same way: 4 m^3 instead of 8 m^3 flops per element.
//    Se, So are the symmetrized halves of the reference's Jacobi factors; the
//    output moves by <= 1e-13 relative (the parity tests pin 1e-12).
// 2. Tiles instead of colours.  A CTA owns a TX x TY block of elements (all
//    compile-time, so every index is a constant-divisor expression), stages
//    its residual region (TX p + 2 n_o + 1) x (TY p + 2 n_o + 1) and its own u
//    with cp.async, runs the four contractions with TWO threads per line (a
//    lane pair: even half / odd half, joined by shuffles in the synthesis
//    stages; factors in the parameter constant bank, streaming independent
//    accumulators), and accumulates the overlapping element corrections into
//    the region in colour passes (fixed order => deterministic).
// 3. Deterministic band fixup.  Nodes within n_o of a tile boundary get
//    contributions from 2 (edges) or 4 (corners) tiles.  The main kernel
//    (persistent, next tile's loads in flight while the current computes)
//    writes exclusive nodes to u and band values to a workspace; a small
//    second kernel adds the band contributions to u in a fixed tile order.
//    Bitwise reproducible, no atomics, no inter-CTA waiting.
#pragma once
#include <cstdlib>

#include "smg_common.cuh"
#include "smg_tma.cuh"

namespace smg {

__host__ __device__ constexpr int fdt_he(int M) { return (M + 1) / 2; }  // even half (incl. centre)
__host__ __device__ constexpr int fdt_ho(int M) { return M / 2; }        // odd half

// Profiling aid: device buffer of FDT_NPH per-phase cycle sums (smg_abi.cu)
constexpr int FDT_NPH = 10;
unsigned long long* fdt_phase_buffer();

template <int M>
struct FDTArgs {
  CUtensorMap rmap;                   // residual (N_y, N_x), box (BRX, RY)
  CUtensorMap umap;                   // u (N_y, N_x), box (OX, OY): own block load + store
  const double* __restrict__ r;       // residual (N_y, N_x)
  double* __restrict__ u;             // u += correction
  const double* __restrict__ inv_nu;  // (n_y, n_x) or nullptr
  const double* __restrict__ dinv;    // (M,M), [even | odd] eigen order in both dims
  double* __restrict__ ws;            // ring workspace: ntiles * RY * RX
  int N_x, N_y, n_x, ntx, nty;
  int u_zero;                         // 1: u holds no valid data and is treated as 0 (write, not add)
  unsigned long long* phases;         // profiling aid (SMG_FDT_PHASES=1): per-phase clock64 sums, else nullptr
  // analysis factors Se[k][i] (k physical half index); synthesis factors
  // SeT[i][k] pre-multiplied by the (mirror-symmetric) Schwarz weight w[k]
  double Sye[fdt_he(M) * fdt_he(M)], SyeT[fdt_he(M) * fdt_he(M)];
  double Syo[fdt_ho(M) * fdt_ho(M) + 1], SyoT[fdt_ho(M) * fdt_ho(M) + 1];
  double Sxe[fdt_he(M) * fdt_he(M)], SxeT[fdt_he(M) * fdt_he(M)];
  double Sxo[fdt_ho(M) * fdt_ho(M) + 1], SxoT[fdt_ho(M) * fdt_ho(M) + 1];
};

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int P, int NO, int TX, int TY>
struct FDTGeom {
  static constexpr int M = P + 1 + 2 * NO;
  static constexpr int MM = M * M;
  static constexpr int HE = fdt_he(M), HO = fdt_ho(M);
  static constexpr int HOX = HO > 0 ? HO : 1;
  static constexpr int E = TX * TY;
  static constexpr int OX = TX * P, OY = TY * P;
  static constexpr int RX = OX + 2 * NO + 1, RY = OY + 2 * NO + 1;
  static constexpr int BW = 2 * NO + 1;
  // two threads per (element, line): warps [0, NH) take the even halves and
  // warps [NH, 2 NH) the odd halves -- parity is warp-uniform (no divergence)
  static constexpr int NH = ((E * M + 31) / 32) * 32;
  static constexpr int THREADS = 2 * NH;
  static constexpr int NT = THREADS;
  // colours inside the tile: windows of elements C apart are disjoint
  static constexpr int C = (2 * NO < P) ? 2 : 3;
  static constexpr int STAGE = RX * RY + OX * OY;  // doubles per pipeline stage
  static constexpr size_t SMEM = sizeof(double) * (2 * (size_t)STAGE + (size_t)E * MM);
  // two resident CTAs when both fit; the register cap follows from it
  static constexpr int MINB = (2 * SMEM <= 200 * 1024 && THREADS <= 384) ? 2 : 1;
  // ---- TMA-staged kernel (fdt_kernel) ----
  // residual box: starts at the even column at or below the region origin
  // (TMA boxes must start on a 16-byte boundary), hence one spare column
  static constexpr int BRX = (RX + 2) & ~1;
  static constexpr int RBOX = BRX * RY, UBOX = OX * OY;
  // one buffer per pipeline stage holds the residual box, and -- once stage 1
  // has consumed it -- the tile's own block of u (loaded, updated, stored)
  static constexpr int STR = (((RBOX > UBOX ? RBOX : UBOX) + 15) & ~15);  // 128-byte multiple
  static constexpr int NRING = RX * RY - OX * OY;    // region nodes owned by neighbour tiles
  static constexpr int KC = (M + P - 1) / P;         // max elements covering one node per direction
  // nb element buffers (2: the DFMA stages ping-pong between them, no read-before-write barriers)
  static constexpr size_t smem_for(int ns, int nb = 1) { return sizeof(double) * ((size_t)ns * STR + (size_t)nb * E * MM) + 16 * (size_t)ns; }
  static constexpr size_t HALF_SM = 112 * 1024;      // two CTAs per SM
  // stages: 4 when two CTAs still fit, else 3, else the most that fit one CTA
  static constexpr int NS = smem_for(4) <= HALF_SM ? 4 : smem_for(3) <= HALF_SM ? 3 : smem_for(4) <= 227 * 1024 ? 4 : 3;
  static constexpr size_t TSMEM = smem_for(NS);
  static constexpr int TMINB = (TSMEM <= HALF_SM && THREADS <= 384) ? 2 : 1;
};

// Half analysis of one line.  Even lane: t = Se^T (x_k + x_{m-1-k}) (plus the
// centre for odd m); odd lane: t = So^T (x_k - x_{m-1-k}).  H = half length.
template <int M, int H, bool ODD, typename In>
__device__ __forceinline__ void half_analyse(const double* __restrict__ S, In in, double (&t)[H]) {
  constexpr int HO = fdt_ho(M);
  double xk[H];
#pragma unroll
  for (int k = 0; k < H; ++k) {
    if (k < HO) {
      const double a = in(k), b = in(M - 1 - k);
      xk[k] = ODD ? a - b : a + b;
    } else {
      xk[k] = in(k);  // centre (even half of odd M)
    }
  }
#pragma unroll
  for (int i = 0; i < H; ++i) t[i] = S[i] * xk[0];
#pragma unroll
  for (int k = 1; k < H; ++k)
#pragma unroll
    for (int i = 0; i < H; ++i) t[i] = fma(S[k * H + i], xk[k], t[i]);
}

// Half synthesis: acc[k] = sum_i ST[i][k] t[i] (even lane: e, odd lane: o).
template <int H>
__device__ __forceinline__ void half_synth(const double* __restrict__ ST, const double (&t)[H], double (&acc)[H]) {
#pragma unroll
  for (int k = 0; k < H; ++k) acc[k] = ST[k] * t[0];
#pragma unroll
  for (int i = 1; i < H; ++i)
#pragma unroll
    for (int k = 0; k < H; ++k) acc[k] = fma(ST[i * H + k], t[i], acc[k]);
}

template <int P, int NO, int TX, int TY, int NT>
__device__ __forceinline__ void fdt_prefetch(const double* __restrict__ r, const double* __restrict__ u, int N_x,
                                             int N_y, int ntx, int tile, double* buf, bool u_zero) {
  using G = FDTGeom<P, NO, TX, TY>;
  constexpr int RX = G::RX, RY = G::RY, OX = G::OX, OY = G::OY;
  const int tx = tile % ntx, ty = tile / ntx;
  const int X0 = tx * OX, Y0 = ty * OY;
  for (int idx = threadIdx.x; idx < RX * RY; idx += NT) {
    const int y = idx / RX, x = idx - y * RX;
    cp_async8(buf + idx, r + (size_t)wrapi(Y0 - NO + y, N_y) * N_x + wrapi(X0 - NO + x, N_x));
  }
  if (u_zero) return;
  double* uo = buf + RX * RY;
  for (int idx = threadIdx.x; idx < OX * OY; idx += NT) {
    const int y = idx / OX, x = idx - y * OX;
    cp_async8(uo + idx, u + (size_t)(Y0 + y) * N_x + (X0 + x));
  }
}

// Gather of the element corrections.  After the recombination pass EB holds,
// per element, the weighted correction on its whole M x M window (the weight
// is folded into the synthesis factors).  A region node (y, x) sums the
// elements (ey, ex) whose window [e P, e P + M) covers it, in a fixed order
// (deterministic).
//
// Column part, computed once per thread for its column x: for each of the
// <= KC candidate element columns, the byte offset of column x in it and a
// 0/1 weight (0 when the candidate does not cover x: branch-free sums).
template <int P, int NO, int TX, int TY>
struct FDTCol {
  static constexpr int KC = FDTGeom<P, NO, TX, TY>::KC;
  int xo[KC];
  double wx[KC];
  __device__ __forceinline__ explicit FDTCol(int x) {
    using G = FDTGeom<P, NO, TX, TY>;
    constexpr int M = G::M, MM = G::MM;
    const int ex0 = min(x / P, TX - 1);
#pragma unroll
    for (int b = 0; b < KC; ++b) {
      const int ex = ex0 - b, cx = x - ex * P;
      const bool ok = ex >= 0 && cx < M;
      xo[b] = ok ? (ex * MM + cx) * 8 : 0;
      wx[b] = ok ? 1.0 : 0.0;
    }
  }
  // correction at region row y
  __device__ __forceinline__ double at(const double* EB, int y) const {
    using G = FDTGeom<P, NO, TX, TY>;
    constexpr int M = G::M, MM = G::MM;
    const int ey0 = min(y / P, TY - 1);
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < KC; ++a) {
      const int ey = ey0 - a, cy = y - ey * P;
      const bool ok = ey >= 0 && cy < M;
      const char* rp = reinterpret_cast<const char*>(EB) + (ok ? (ey * (TX * MM) + cy * M) * 8 : 0);
      double v = 0.0;
#pragma unroll
      for (int b = 0; b < KC; ++b) v = fma(wx[b], *reinterpret_cast<const double*>(rp + xo[b]), v);
      acc = fma(ok ? 1.0 : 0.0, v, acc);
    }
    return acc;
  }
};

// Seam tiles (their residual region wraps around the periodic mesh, which TMA
// cannot express): per-node cp.async into the box layout (row pitch BRX).
template <int P, int NO, int TX, int TY, int NT>
__device__ __forceinline__ void fdt_region_cpasync(const double* __restrict__ r, int N_x, int N_y, int X0, int Y0,
                                                   double* R) {
  using G = FDTGeom<P, NO, TX, TY>;
  constexpr int RX = G::RX, RY = G::RY, BRX = G::BRX;
  for (int idx = threadIdx.x; idx < RX * RY; idx += NT) {
    const int y = idx / RX, x = idx - y * RX;
    cp_async8(R + y * BRX + x, r + (size_t)wrapi(Y0 - NO + y, N_y) * N_x + wrapi(X0 - NO + x, N_x));
  }
}

// Column of the region origin inside the residual box (0 or 1).
__device__ __forceinline__ int fdt_box_shift(int X0, int NO) { return (X0 - NO) & 1; }

// Epilogue part 1 (after stage 4): recombine every window row in place
// (out[j] = ex[j] + ox[j], out[M-1-j] = ex[j] - ox[j]; the centre of odd M is
// ex), then fold the overlaps onto the home cells.  Window cell (cy, cx) of
// an element is "home" when NO <= cx, cy < NO + P (the element's own nodes).
// Only the immediate neighbours reach a home cell: the right one at
// cx = P..P+NO-1 (its cells 0..NO-1), the left one at cx = NO..2NO (its cells
// P+NO..P+2NO).  Each item reads only non-home cells and writes only its own
// element's home cells; x first (all rows), then y (all columns): corners
// come along.  Ends with a barrier.
template <int P, int NO, int TX, int TY, int NT>
__device__ __forceinline__ void fdt_epilogue_fold(double* EB) {
  using G = FDTGeom<P, NO, TX, TY>;
  constexpr int M = G::M, MM = G::MM, E = G::E, HE = G::HE, HO = G::HO, HOX = G::HOX;
  for (int it = threadIdx.x; it < E * M; it += NT) {
    double* br = EB + it * M;   // row c of element e (rows are contiguous)
    double ev[HE], ov[HOX];
#pragma unroll
    for (int j = 0; j < HE; ++j) ev[j] = br[j];
#pragma unroll
    for (int j = 0; j < HO; ++j) ov[j] = br[HE + j];
#pragma unroll
    for (int j = 0; j < HO; ++j) {
      br[j] = ev[j] + ov[j];
      br[M - 1 - j] = ev[j] - ov[j];
    }
  }
  __syncthreads();
  for (int it = threadIdx.x; it < E * M; it += NT) {
    const int e = it / M, exl = e % TX;
    double* br = EB + it * M;   // row c
    if (exl + 1 < TX) {
#pragma unroll
      for (int k = 0; k < NO; ++k) br[P + k] += br[MM + k];
    }
    if (exl > 0) {
#pragma unroll
      for (int k = NO; k <= 2 * NO; ++k) br[k] += br[P + k - MM];
    }
  }
  __syncthreads();
  for (int it = threadIdx.x; it < E * M; it += NT) {
    const int e = it / M, c = it - e * M, eyl = e / TX;
    double* bc = EB + e * MM + c;  // column c
    if (eyl + 1 < TY) {
#pragma unroll
      for (int k = 0; k < NO; ++k) bc[(P + k) * M] += bc[TX * MM + k * M];
    }
    if (eyl > 0) {
#pragma unroll
      for (int k = NO; k <= 2 * NO; ++k) bc[k * M] += bc[(P + k) * M - TX * MM];
    }
  }
  __syncthreads();
}

// FP64 tensor-core MMA, m8n8k4: lane (g = lane/4, t = lane%4) holds A[g][t],
// B[t][g] and accumulates C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Kernel-level constants: DM selects the even/odd DMMA contraction stages
// (8 warps; factor fragments in shared memory) instead of the DFMA stages.
#ifndef SMG_FDT_DMB
#define SMG_FDT_DMB 2   // 8-line batches per warp iteration of the DMMA stages
#endif

template <int P, int NO, int TX, int TY, bool DM>
struct FDTK {
  using G = FDTGeom<P, NO, TX, TY>;
  static constexpr int M = G::M, HE = G::HE, HO = G::HO, E = G::E;
  static constexpr int MTE = (HE + 7) / 8, KTE = (HE + 3) / 4;   // even half: output / k tiles
  static constexpr int MTO = (HO + 7) / 8, KTO = (HO + 3) / 4;   // odd half
  static constexpr int FE = MTE * KTE, FO = MTO * KTO;
  static constexpr int FRN = DM ? 4 * (FE + FO) * 32 : 0;        // fragment table (doubles)
  static constexpr int BT = (E * M + 7) / 8;                     // 8-line batches
  // DMMA stages: each warp iteration carries DMB batches whose accumulator
  // chains interleave (2 (MTE + MTO) independent DMMAs per k-step: the chains
  // were latency-bound with one batch, ncu stall_wait); the warp count is the
  // smallest that keeps the fewest iterations per warp (balanced batches)
  static constexpr int DMB = SMG_FDT_DMB;
  static constexpr int dm_warps() {
    int it_min = (BT + DMB * 12 - 1) / (DMB * 12);
    for (int w = 4; w <= 12; ++w)
      if ((BT + DMB * w - 1) / (DMB * w) == it_min) return w;
    return 12;
  }
  static constexpr int WARPS = DM ? dm_warps() : 8;
  static constexpr int NT = DM ? 32 * WARPS : G::THREADS;
  static constexpr int DMIT = (BT + DMB * WARPS - 1) / (DMB * WARPS);   // iterations per warp
  static constexpr int MAXB = DMB * DMIT;
  static constexpr size_t extra = sizeof(double) * ((size_t)FRN + (DM ? E : 0));
  static constexpr size_t HALF_SM = 112 * 1024, FULL_SM = 227 * 1024;
  static constexpr size_t sm1(int ns) { return G::smem_for(ns, 1) + extra; }
  static constexpr size_t sm2(int ns) { return G::smem_for(ns, 2) + extra; }
  // ping-pong element buffers (DFMA stages) when that keeps the occupancy:
  // two CTAs per SM with 3+ stages, or one CTA per SM that one buffer needs anyway
  static constexpr bool PP = !DM && (sm2(3) <= HALF_SM || (sm1(3) > HALF_SM && sm2(3) <= FULL_SM));
  static constexpr size_t LIM = (PP && sm2(3) > HALF_SM) ? FULL_SM : HALF_SM;
  static constexpr int NS = PP ? (sm2(4) <= LIM ? 4 : 3)
                               : (sm1(4) <= HALF_SM ? 4 : sm1(3) <= HALF_SM ? 3 : sm1(4) <= FULL_SM ? 4 : 3);
  static constexpr size_t smem_for(int ns) { return PP ? sm2(ns) : sm1(ns); }
  // DFMA stage 2 reads 1/(lam_y + lam_x) from shared memory when the table
  // fits beside the chosen configuration (else from global memory through L1:
  // those loads were the stage's long-scoreboard stalls)
  static constexpr size_t SDB = sizeof(double) * (size_t)M * M;
  static constexpr bool SDV = !DM && smem_for(NS) + SDB <= (smem_for(NS) <= HALF_SM ? HALF_SM : FULL_SM);
  static constexpr size_t TSMEM = smem_for(NS) + (SDV ? SDB : 0);
  static constexpr int MINB = (TSMEM <= HALF_SM && NT <= 384) ? 2 : 1;
};

// The fragments of one stage (even and odd halves) into registers.
template <int FE, int FO>
__device__ __forceinline__ void dm_load_frags(const double* FR, int stage, int lane, double (&fe)[FE], double (&fo)[FO]) {
#pragma unroll
  for (int f = 0; f < FE; ++f) fe[f] = FR[(stage * (FE + FO) + f) * 32 + lane];
#pragma unroll
  for (int f = 0; f < FO; ++f) fo[f] = FR[(stage * (FE + FO) + FE + f) * 32 + lane];
}

// Fragment table of the 4 contraction stages (even, odd), built per CTA from
// the factor arrays in the parameter bank.  Stages 1/3 use the factor as the
// A operand (A[out][in]), stages 2/4 as the B operand (B[in][out]).
template <int M, class Args, int FE, int FO, int KTE, int KTO>
__device__ __forceinline__ void dm_build_frags(const Args& A, double* FR, int NT) {
  constexpr int HE = fdt_he(M), HO = fdt_ho(M);
  for (int idx = threadIdx.x; idx < 4 * (FE + FO) * 32; idx += NT) {
    const int lane = idx & 31, fa = idx >> 5;
    const int st = fa / (FE + FO), r = fa - st * (FE + FO);
    const bool od = r >= FE;
    const int f = od ? r - FE : r, KT = od ? KTO : KTE, H = od ? HO : HE;
    const int mt = f / KT, kt = f - mt * KT, g = lane >> 2, t = lane & 3;
    const int o = 8 * mt + g, k = 4 * kt + t;   // output index, input index
    double v = 0.0;
    if (o < H && k < H) {
      if (st == 0) v = od ? A.Syo[k * H + o] : A.Sye[k * H + o];       // A[i][k] = Sy[k][i]
      else if (st == 1) v = od ? A.Sxo[k * H + o] : A.Sxe[k * H + o];  // B[k][l] = Sx[k][l]
      else if (st == 2) v = od ? A.SyoT[k * H + o] : A.SyeT[k * H + o];  // A[k][i] = SyT[i][k]
      else v = od ? A.SxoT[k * H + o] : A.SxeT[k * H + o];             // B[i][k] = SxT[i][k]
    }
    FR[idx] = v;
  }
}

// Persistent main kernel.  Per tile (TX x TY elements), in an NS-buffer ring:
//   * the (RY x BRX) residual box is TMA-loaded NS-2 tiles ahead (one thread
//     issues it; completion on the buffer's mbarrier; seam tiles, whose region
//     wraps around the periodic mesh, use per-node cp.async instead);
//   * stage 1 consumes the box; the tile's (OY x OX) own block of u is then
//     TMA-loaded into the same buffer and lands while stages 2-4 run
//     (even/odd halves in separate warps);
//   * gather: every own node adds the element corrections covering it to its
//     u in the buffer, which ONE TMA store writes back; region nodes owned by
//     neighbour tiles (the ring) go to the workspace for fdt_fixup.
template <int P, int NO, int TX, int TY>
__device__ __forceinline__ void fdt_fixup_node(double* __restrict__ u, const double* __restrict__ ws, int N_x,
                                               int ntx, int nty, long gid);
template <int P, int NO, int TX, int TY>
constexpr long fdt_fixup_per_tile() {
  using G = FDTGeom<P, NO, TX, TY>;
  return (long)(2 * NO + 1) * G::OX + (long)(G::OY - 2 * NO - 1) * (2 * NO + 1);
}

// Profiling aid: -DSMG_FDT_DEBUG_SKIP builds skip the four contractions (the
// memory pipeline and epilogue alone; tools/fd_diag.py).  Never in the default build.
#ifdef SMG_FDT_DEBUG_SKIP
constexpr bool kFdtSkip = true;
#else
constexpr bool kFdtSkip = false;
#endif

template <int P, int NO, int TX, int TY, bool DM>
__global__ void __launch_bounds__(FDTK<P, NO, TX, TY, DM>::NT, FDTK<P, NO, TX, TY, DM>::MINB)
fdt_kernel(const __grid_constant__ FDTArgs<P + 1 + 2 * NO> A) {
  // PDL: the prologue below (barriers, factor fragments, the 1/(lam_y+lam_x)
  // table -- all per-level constants) overlaps the preceding grid; the wait
  // sits before the first read of r / u
  SMG_PDL_TRIGGER();
  using G = FDTGeom<P, NO, TX, TY>;
  using K = FDTK<P, NO, TX, TY, DM>;
  constexpr int M = G::M, MM = G::MM, E = G::E, OX = G::OX, OY = G::OY, RX = G::RX, RY = G::RY;
  constexpr int HE = G::HE, HO = G::HO, HOX = G::HOX, NT = K::NT, NH = G::NH, BRX = G::BRX;
  constexpr int STR = G::STR, NS = K::NS, NRING = G::NRING;
  static_assert(K::TSMEM <= 227 * 1024, "tile does not fit in shared memory");
  static_assert(NS >= 3, "pipeline needs >= 3 buffers");
  // dynamic shared memory starts 1024-byte aligned (no static shared memory in
  // this kernel); TMA boxes need 128-byte aligned destinations
  extern __shared__ __align__(1024) double sm[];
  double* EB = sm + NS * STR;  // E x M x M element buffers
  constexpr bool PP = K::PP;
  double* EB2 = EB + (PP ? E * MM : 0);   // second element buffer (PP: DFMA stages 2 and 4 write here; else EB)
  double* FR = EB + (PP ? 2 : 1) * E * MM; // DMMA fragment table (DM only)
  double* SN = FR + K::FRN;    // per-element 1/nu_bar of the current tile (DM only)
  double* SD = SN + (DM ? E : 0);  // 1/(lam_y + lam_x) table (K::SDV)
  uint64_t* barR = reinterpret_cast<uint64_t*>(SD + (K::SDV ? M * M : 0));
  uint64_t* barU = barR + NS;
  const double* FSye = A.Sye;
  const double* FSyeT = A.SyeT;
  const double* FSxe = A.Sxe;
  const double* FSxeT = A.SxeT;
  const double* FSyo = A.Syo;
  const double* FSyoT = A.SyoT;
  const double* FSxo = A.Sxo;
  const double* FSxoT = A.SxoT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g8 = lane >> 2, t4 = lane & 3;
  const int tid = threadIdx.x;
  const int N_x = A.N_x, N_y = A.N_y, ntx = A.ntx, nty = A.nty, ntiles = ntx * nty;
  const bool u_zero = A.u_zero != 0;

  const bool odd = tid >= NH;     // warp-uniform
  const int line = odd ? tid - NH : tid;
  const int e = line / M, c = line - e * M;
  const bool act = e < E;
  const int exl = e % TX, eyl = e / TX;
  double* B = EB + e * MM;
  double* B2 = EB2 + e * MM;
  // this thread's half row of 1/(lam_y + lam_x) (shared memory, or L1-resident across tiles)
  const double* dl = (K::SDV ? SD : A.dinv) + (act ? c : 0) * M + (odd ? HE : 0);

  if (tid == 0) {
    if (smem_u32(sm) & 127) __trap();  // alignment assumption above
    for (int k = 0; k < 2 * NS; ++k) mbar_init(barR + k, 1);
    fence_mbar_init();
  }
  if constexpr (DM) dm_build_frags<M, FDTArgs<M>, K::FE, K::FO, K::KTE, K::KTO>(A, FR, NT);
  if constexpr (K::SDV)
    for (int idx = tid; idx < M * M; idx += NT) SD[idx] = A.dinv[idx];
  __syncthreads();
  SMG_PDL_WAIT();

  // residual box of tile t into buffer b (all threads call; thread 0 owns TMA).
  // The caller guarantees the buffer is free (its last store has been read).
  auto issue_r = [&](int t, int b) {
    const int tx = t % ntx, ty = t / ntx;
    const int X0 = tx * OX, Y0 = ty * OY;
    const bool seam = tx == 0 || ty == 0 || tx == ntx - 1 || ty == nty - 1;
    if (tid == 0) {
      fence_proxy_async_smem();   // generic writes to the buffer precede the async-proxy refill
      mbar_arrive_expect_tx(barR + b, seam ? 0u : (unsigned)(G::RBOX * 8));
      if (!seam) tma_load_2d(sm + b * STR, &A.rmap, (X0 - NO) & ~1, Y0 - NO, barR + b);
    }
    if (seam) fdt_region_cpasync<P, NO, TX, TY, NT>(A.r, N_x, N_y, X0, Y0, sm + b * STR + fdt_box_shift(X0, NO));
  };

#pragma unroll
  for (int j = 0; j < NS - 2; ++j) {
    const int t = blockIdx.x + j * gridDim.x;
    if (t < ntiles) issue_r(t, j);
    cp_async_commit();
  }
  int tile = blockIdx.x;
#ifdef SMG_FDT_PROFILE
  // phase profile (build with -DSMG_FDT_PROFILE, run with SMG_FDT_PHASES=1; tools/fdt_phases.py)
  const bool prof = A.phases != nullptr && tid == 0;
  unsigned long long ph[FDT_NPH] = {}, tlast = 0;
  auto mark = [&](int k) {
    if (prof) { const unsigned long long t = clock64(); ph[k] += t - tlast; tlast = t; }
  };
#else
  auto mark = [](int) {};
#endif
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
#ifdef SMG_FDT_PROFILE
    if (prof) { tlast = clock64(); ph[0] += 1; }
#endif
    const int b = it % NS;
    const unsigned par = (unsigned)(it / NS) & 1u;
    double* buf = sm + b * STR;
    const int tx = tile % ntx, ty = tile / ntx;
    const int X0 = tx * OX, Y0 = ty * OY;
    double s = 1.0;  // 1 / nu_bar of this element
    if (!DM && act && A.inv_nu != nullptr) s = __ldg(A.inv_nu + (size_t)(ty * TY + eyl) * A.n_x + (tx * TX + exl));
    if (DM && tid < E) SN[tid] = A.inv_nu != nullptr ? __ldg(A.inv_nu + (size_t)(ty * TY + tid / TX) * A.n_x + (tx * TX + tid % TX)) : 1.0;
    cp_async_wait<NS - 3>();
    mbar_wait(barR + b, par);
    __syncthreads();
    mark(1);

    // ---- stage 1 (physical columns c): [T1e; T1o][:, c] = [Se; So]^T fold_y(R_e[:, c])
    if constexpr (DM) {
      if (!kFdtSkip) {
        constexpr int DMB = K::DMB;
        const double* R0 = buf + fdt_box_shift(X0, NO);
        double fe[K::FE], fo[K::FO];
        dm_load_frags<K::FE, K::FO>(FR, 0, lane, fe, fo);
        for (int b0 = DMB * warp; b0 < K::BT; b0 += DMB * K::WARPS) {
          const double* col[DMB];
          bool vn[DMB];
#pragma unroll
          for (int q = 0; q < DMB; ++q) {
            const int n = 8 * (b0 + q) + g8;
            vn[q] = n < E * M;
            const int en = vn[q] ? n / M : 0, cn = vn[q] ? n - en * M : 0;
            col[q] = R0 + ((en / TX) * P) * BRX + (en % TX) * P + cn;
          }
          double ae[DMB][K::MTE][2], ao[DMB][K::MTO][2];
#pragma unroll
          for (int q = 0; q < DMB; ++q) {
#pragma unroll
            for (int m = 0; m < K::MTE; ++m) ae[q][m][0] = ae[q][m][1] = 0.0;
#pragma unroll
            for (int m = 0; m < K::MTO; ++m) ao[q][m][0] = ao[q][m][1] = 0.0;
          }
#pragma unroll
          for (int kt = 0; kt < K::KTE; ++kt) {
            const int k = 4 * kt + t4;
            double be[DMB], bo[DMB];
#pragma unroll
            for (int q = 0; q < DMB; ++q) {
              double x0 = 0.0, x1 = 0.0;
              if (vn[q] && k < HE) {
                x0 = col[q][k * BRX];
                if (k < HO) x1 = col[q][(M - 1 - k) * BRX];
              }
              be[q] = x0 + x1;
              bo[q] = (k < HO) ? x0 - x1 : 0.0;
            }
#pragma unroll
            for (int m = 0; m < K::MTE; ++m)
#pragma unroll
              for (int q = 0; q < DMB; ++q) dmma884(ae[q][m][0], ae[q][m][1], fe[m * K::KTE + kt], be[q]);
            if (kt < K::KTO) {
#pragma unroll
              for (int m = 0; m < K::MTO; ++m)
#pragma unroll
                for (int q = 0; q < DMB; ++q) dmma884(ao[q][m][0], ao[q][m][1], fo[m * K::KTO + kt], bo[q]);
            }
          }
#pragma unroll
          for (int q = 0; q < DMB; ++q)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int n2 = 8 * (b0 + q) + 2 * t4 + j;
              if (n2 < E * M) {
                const int e2 = n2 / M, c2 = n2 - e2 * M;
                double* o = EB + e2 * MM + c2;
#pragma unroll
                for (int m = 0; m < K::MTE; ++m)
                  if (8 * m + g8 < HE) o[(8 * m + g8) * M] = ae[q][m][j];
#pragma unroll
                for (int m = 0; m < K::MTO; ++m)
                  if (8 * m + g8 < HO) o[(HE + 8 * m + g8) * M] = ao[q][m][j];
              }
            }
        }
      }
    } else if (!kFdtSkip && act) {
      const double* col = buf + fdt_box_shift(X0, NO) + (eyl * P) * BRX + exl * P + c;
      auto in = [&](int k) { return col[k * BRX]; };
      if (!odd) {
        double t[HE];
        half_analyse<M, HE, false>(FSye, in, t);
#pragma unroll
        for (int i = 0; i < HE; ++i) B[i * M + c] = t[i];
      } else if (HO > 0) {
        double t[HOX];
        half_analyse<M, HOX, true>(FSyo, in, t);
#pragma unroll
        for (int i = 0; i < HO; ++i) B[(HE + i) * M + c] = t[i];
      }
    }
    if (tid == 0) bulk_wait_read<1>();  // the store of tile it-2 has left its buffer
    __syncthreads();
    mark(2);
    // this buffer's residual is consumed: bring in the own block of u; and
    // refill the buffer of tile it-2 with the residual of tile it+NS-2
    if (tid == 0 && !u_zero) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(barU + b, (unsigned)(G::UBOX * 8));
      tma_load_2d(buf, &A.umap, X0, Y0, barU + b);
    }
    {
      const int nxt = tile + (NS - 2) * gridDim.x;
      if (nxt < ntiles) issue_r(nxt, (it + NS - 2) % NS);
      cp_async_commit();
    }
    mark(9);

    if (kFdtSkip) {
      for (int idx = tid; idx < (PP ? 2 : 1) * E * MM; idx += NT) EB[idx] = 0.0;
      __syncthreads();
    } else if constexpr (DM) {
      constexpr int DMB = K::DMB;
      double fe[K::FE], fo[K::FO];
      // ---- stage 2 (rows n = (e, c)): T2[n][l] = fold_x(T1[n][:]) . [Se | So] * dinv * (1/nu_bar);
      //      a batch's 8 rows are read and rewritten by one warp only
      dm_load_frags<K::FE, K::FO>(FR, 1, lane, fe, fo);
      for (int b0 = DMB * warp; b0 < K::BT; b0 += DMB * K::WARPS) {
        const double* row[DMB];
        bool vn[DMB];
        int nq[DMB];
#pragma unroll
        for (int q = 0; q < DMB; ++q) {
          nq[q] = 8 * (b0 + q) + g8;
          vn[q] = nq[q] < E * M;
          row[q] = EB + (vn[q] ? nq[q] : 0) * M;
        }
        double ae[DMB][K::MTE][2], ao[DMB][K::MTO][2];
#pragma unroll
        for (int q = 0; q < DMB; ++q) {
#pragma unroll
          for (int m = 0; m < K::MTE; ++m) ae[q][m][0] = ae[q][m][1] = 0.0;
#pragma unroll
          for (int m = 0; m < K::MTO; ++m) ao[q][m][0] = ao[q][m][1] = 0.0;
        }
#pragma unroll
        for (int kt = 0; kt < K::KTE; ++kt) {
          const int k = 4 * kt + t4;
          double a_e[DMB], a_o[DMB];
#pragma unroll
          for (int q = 0; q < DMB; ++q) {
            double x0 = 0.0, x1 = 0.0;
            if (vn[q] && k < HE) {
              x0 = row[q][k];
              if (k < HO) x1 = row[q][M - 1 - k];
            }
            a_e[q] = x0 + x1;
            a_o[q] = (k < HO) ? x0 - x1 : 0.0;
          }
#pragma unroll
          for (int m = 0; m < K::MTE; ++m)
#pragma unroll
            for (int q = 0; q < DMB; ++q) dmma884(ae[q][m][0], ae[q][m][1], a_e[q], fe[m * K::KTE + kt]);
          if (kt < K::KTO) {
#pragma unroll
            for (int m = 0; m < K::MTO; ++m)
#pragma unroll
              for (int q = 0; q < DMB; ++q) dmma884(ao[q][m][0], ao[q][m][1], a_o[q], fo[m * K::KTO + kt]);
          }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < DMB; ++q) {
          if (!vn[q]) continue;
          const int n = nq[q];
          const int en = n / M, cn = n - en * M;
          const double sc = SN[en];
          double* w = EB + n * M;
          const double* dn = A.dinv + cn * M;
#pragma unroll
          for (int m = 0; m < K::MTE; ++m)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int l = 8 * m + 2 * t4 + j;
              if (l < HE) w[l] = ae[q][m][j] * (__ldg(dn + l) * sc);
            }
#pragma unroll
          for (int m = 0; m < K::MTO; ++m)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int l = 8 * m + 2 * t4 + j;
              if (l < HO) w[HE + l] = ao[q][m][j] * (__ldg(dn + HE + l) * sc);
            }
        }
        __syncwarp();
      }
      __syncthreads();
      // ---- stage 3 (columns n = (e, c)): e = SyeT' T2e[:, c] (rows [0,HE)), o = SyoT' T2o[:, c]
      dm_load_frags<K::FE, K::FO>(FR, 2, lane, fe, fo);
      for (int b0 = DMB * warp; b0 < K::BT; b0 += DMB * K::WARPS) {
        const double* col[DMB];
        bool vn[DMB];
#pragma unroll
        for (int q = 0; q < DMB; ++q) {
          const int n = 8 * (b0 + q) + g8;
          vn[q] = n < E * M;
          const int en = vn[q] ? n / M : 0, cn = vn[q] ? n - en * M : 0;
          col[q] = EB + en * MM + cn;
        }
        double ae[DMB][K::MTE][2], ao[DMB][K::MTO][2];
#pragma unroll
        for (int q = 0; q < DMB; ++q) {
#pragma unroll
          for (int m = 0; m < K::MTE; ++m) ae[q][m][0] = ae[q][m][1] = 0.0;
#pragma unroll
          for (int m = 0; m < K::MTO; ++m) ao[q][m][0] = ao[q][m][1] = 0.0;
        }
#pragma unroll
        for (int kt = 0; kt < K::KTE; ++kt) {
          const int i = 4 * kt + t4;
          double be[DMB], bo[DMB];
#pragma unroll
          for (int q = 0; q < DMB; ++q) {
            be[q] = (vn[q] && i < HE) ? col[q][i * M] : 0.0;
            bo[q] = (vn[q] && i < HO) ? col[q][(HE + i) * M] : 0.0;
          }
#pragma unroll
          for (int m = 0; m < K::MTE; ++m)
#pragma unroll
            for (int q = 0; q < DMB; ++q) dmma884(ae[q][m][0], ae[q][m][1], fe[m * K::KTE + kt], be[q]);
          if (kt < K::KTO) {
#pragma unroll
            for (int m = 0; m < K::MTO; ++m)
#pragma unroll
              for (int q = 0; q < DMB; ++q) dmma884(ao[q][m][0], ao[q][m][1], fo[m * K::KTO + kt], bo[q]);
          }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < DMB; ++q)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int n2 = 8 * (b0 + q) + 2 * t4 + j;
            if (n2 < E * M) {
              const int e2 = n2 / M, c2 = n2 - e2 * M;
              double* o = EB + e2 * MM + c2;
#pragma unroll
              for (int m = 0; m < K::MTE; ++m)
                if (8 * m + g8 < HE) o[(8 * m + g8) * M] = ae[q][m][j];
#pragma unroll
              for (int m = 0; m < K::MTO; ++m)
                if (8 * m + g8 < HO) o[(HE + 8 * m + g8) * M] = ao[q][m][j];
            }
          }
        __syncwarp();
      }
      __syncthreads();
      // ---- stage 4 (physical rows c): t3 = e[c'] +- o[c'] (mirror-folded row), then
      //      ex = t3e . SxeT', ox = t3o . SxoT'; rows read across warps -> results in
      //      registers until every warp has read
      double re[K::MAXB][K::MTE][2], ro[K::MAXB][K::MTO][2];
      dm_load_frags<K::FE, K::FO>(FR, 3, lane, fe, fo);
#pragma unroll
      for (int it2 = 0; it2 < K::DMIT; ++it2) {
        const double* er[DMB];
        const double* orow[DMB];
        double sg[DMB];
        bool ctr[DMB], vn[DMB];
#pragma unroll
        for (int q = 0; q < DMB; ++q) {
          const int bt = DMB * (warp + it2 * K::WARPS) + q;
          const int n = 8 * bt + g8;
          vn[q] = bt < K::BT && n < E * M;
          const int en = vn[q] ? n / M : 0, cn = vn[q] ? n - en * M : 0;
          const int cf = cn < HE ? cn : M - 1 - cn;
          sg[q] = cn < HE ? 1.0 : -1.0;
          ctr[q] = (M & 1) && cn == HO;
          er[q] = EB + en * MM + cf * M;
          orow[q] = EB + en * MM + (HE + (cf < HO ? cf : 0)) * M;
#pragma unroll
          for (int m = 0; m < K::MTE; ++m) re[it2 * DMB + q][m][0] = re[it2 * DMB + q][m][1] = 0.0;
#pragma unroll
          for (int m = 0; m < K::MTO; ++m) ro[it2 * DMB + q][m][0] = ro[it2 * DMB + q][m][1] = 0.0;
        }
        if (DMB * (warp + it2 * K::WARPS) < K::BT) {
#pragma unroll
          for (int kt = 0; kt < K::KTE; ++kt) {
            const int i = 4 * kt + t4;
            double a_e[DMB], a_o[DMB];
#pragma unroll
            for (int q = 0; q < DMB; ++q) {
              a_e[q] = 0.0;
              a_o[q] = 0.0;
              if (vn[q] && i < HE) a_e[q] = ctr[q] ? er[q][i] : fma(sg[q], orow[q][i], er[q][i]);
              if (vn[q] && i < HO) a_o[q] = ctr[q] ? er[q][HE + i] : fma(sg[q], orow[q][HE + i], er[q][HE + i]);
            }
#pragma unroll
            for (int m = 0; m < K::MTE; ++m)
#pragma unroll
              for (int q = 0; q < DMB; ++q)
                dmma884(re[it2 * DMB + q][m][0], re[it2 * DMB + q][m][1], a_e[q], fe[m * K::KTE + kt]);
            if (kt < K::KTO) {
#pragma unroll
              for (int m = 0; m < K::MTO; ++m)
#pragma unroll
                for (int q = 0; q < DMB; ++q)
                  dmma884(ro[it2 * DMB + q][m][0], ro[it2 * DMB + q][m][1], a_o[q], fo[m * K::KTO + kt]);
            }
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int it2 = 0; it2 < K::DMIT; ++it2)
#pragma unroll
        for (int q = 0; q < DMB; ++q) {
          const int bt = DMB * (warp + it2 * K::WARPS) + q;
          const int n = 8 * bt + g8;
          if (bt < K::BT && n < E * M) {
            double* w = EB + n * M;
#pragma unroll
            for (int m = 0; m < K::MTE; ++m)
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const int k = 8 * m + 2 * t4 + j;
                if (k < HE) w[k] = re[it2 * DMB + q][m][j];
              }
#pragma unroll
            for (int m = 0; m < K::MTO; ++m)
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const int k = 8 * m + 2 * t4 + j;
                if (k < HO) w[HE + k] = ro[it2 * DMB + q][m][j];
              }
          }
        }
      __syncthreads();
      fdt_epilogue_fold<P, NO, TX, TY, NT>(EB);
    } else {
      // ---- stage 2 (eigen-y rows c): T2[c, :] = ([Se; So]^T fold_x(T1[c, :])) * dinv / nu_bar
      {
        double t[HE];
        const double* row = B + c * M;
        auto in = [&](int k) { return row[k]; };
        if (act) {
          if (!odd) half_analyse<M, HE, false>(FSxe, in, t);
          else if (HO > 0) half_analyse<M, HOX, true>(FSxo, in, reinterpret_cast<double(&)[HOX]>(t));
        }
        if constexpr (!PP) __syncthreads();  // every row read before the in-place writes
        if (act) {   // PP: into the second buffer, no read-before-write barrier
          if (!odd) {
#pragma unroll
            for (int l = 0; l < HE; ++l) B2[c * M + l] = t[l] * ((K::SDV ? dl[l] : __ldg(dl + l)) * s);
          } else {
#pragma unroll
            for (int l = 0; l < HO; ++l) B2[c * M + HE + l] = t[l] * ((K::SDV ? dl[l] : __ldg(dl + l)) * s);
          }
        }
      }
      __syncthreads();
      mark(3);

      // ---- stage 3 (eigen-x columns c): even warps e = SyeT^T T2e[:, c] -> rows [0,HE),
      //      odd warps o = SyoT^T T2o[:, c] -> rows [HE, M)   (e/o recombined in stage 4)
      {
        double acc[HE];
        if (act) {
          if (!odd) {
            double t[HE];
#pragma unroll
            for (int i = 0; i < HE; ++i) t[i] = B2[i * M + c];
            half_synth<HE>(FSyeT, t, acc);
          } else if (HO > 0) {
            double t[HOX];
#pragma unroll
            for (int i = 0; i < HO; ++i) t[i] = B2[(HE + i) * M + c];
            half_synth<HOX>(FSyoT, t, reinterpret_cast<double(&)[HOX]>(acc));
          }
        }
        if constexpr (!PP) __syncthreads();  // every column read before the in-place writes
        if (act) {   // PP: back into the first buffer (stage-1 data is dead)
          if (!odd) {
#pragma unroll
            for (int k = 0; k < HE; ++k) B[k * M + c] = acc[k];
          } else {
#pragma unroll
            for (int k = 0; k < HO; ++k) B[(HE + k) * M + c] = acc[k];
          }
        }
      }
      __syncthreads();
      mark(4);

      // ---- stage 4 (physical rows c): T3[c, :] = e[c'] +- o[c'] (c' = mirror-folded
      //      row), then even warps ex = SxeT^T T3e, odd warps ox = SxoT^T T3o ----
      {
        const int cf = c < HE ? c : M - 1 - c;   // folded physical row
        const double sg = c < HE ? 1.0 : -1.0;   // y[m-1-k] = e - o
        const bool centre = (M & 1) && c == HO;
        double acc[HE];
        if (act) {
          const double* er = B + cf * M;
          const double* orow = B + (HE + (cf < HO ? cf : 0)) * M;
          auto t3 = [&](int j) { return centre ? er[j] : fma(sg, orow[j], er[j]); };
          if (!odd) {
            double t[HE];
#pragma unroll
            for (int i = 0; i < HE; ++i) t[i] = t3(i);
            half_synth<HE>(FSxeT, t, acc);
          } else if (HO > 0) {
            double t[HOX];
#pragma unroll
            for (int i = 0; i < HO; ++i) t[i] = t3(HE + i);
            half_synth<HOX>(FSxoT, t, reinterpret_cast<double(&)[HOX]>(acc));
          }
        }
        if constexpr (!PP) __syncthreads();  // every row read before B is reused for ex / ox
        if (act) {
          // even warps keep ex in B2[c][0,HE), odd warps ox in B2[c][HE,M)
          if (!odd) {
#pragma unroll
            for (int k = 0; k < HE; ++k) B2[c * M + k] = acc[k];
          } else {
#pragma unroll
            for (int k = 0; k < HO; ++k) B2[c * M + HE + k] = acc[k];
          }
        }
      }
      __syncthreads();
      mark(5);
      fdt_epilogue_fold<P, NO, TX, TY, NT>(EB2);
      mark(6);
    }
    double* EF = (DM || !PP) ? EB : EB2;   // the finished element corrections
    if (!u_zero) mbar_wait(barU + b, par);
    mark(7);

    // ---- gather: every region node reads ONE cell -- its home element's, or
    //      for ring nodes the edge element covering it ----------------------
    // own block: thread = (column, row group); lanes walk consecutive columns
    {
      constexpr int NG = NT / OX;  // >= 2: NT >= 2 E M > 2 OX
      if (tid < NG * OX) {
        const int ox = tid % OX, g = tid / OX;
        const double* cb = EF + (ox / P) * MM + (ox % P + NO);
        for (int oy = g; oy < OY; oy += NG) {
          const double cor = cb[(oy / P) * (TX * MM) + (oy % P + NO) * M];
          double* uo = buf + oy * OX + ox;
          *uo = u_zero ? cor : *uo + cor;
        }
      }
    }
    // ring (compact, tile-major): rows [0,NO) and [NO+OY,RY) full width, then
    // the side columns [0,NO) u [NO+OX,RX) of the own rows
    {
      double* W = A.ws + (size_t)tile * NRING;
      constexpr int NTB = (RY - OY) * RX;
      for (int k = tid; k < NRING; k += NT) {
        int y, x;
        if (k < NTB) {
          const int yy = k / RX;
          x = k - yy * RX;
          y = yy < NO ? yy : yy + OY;
        } else {
          const int k2 = k - NTB, yy = k2 / (RX - OX), xx = k2 - yy * (RX - OX);
          y = NO + yy;
          x = xx < NO ? xx : xx + OX;
        }
        const int ey = y < NO ? 0 : min((y - NO) / P, TY - 1);
        const int ex = x < NO ? 0 : min((x - NO) / P, TX - 1);
        W[k] = EF[(ey * TX + ex) * MM + (y - ey * P) * M + (x - ex * P)];
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    mark(8);
    if (tid == 0) {
      tma_store_2d(&A.umap, buf, X0, Y0);
      bulk_commit();
    }
  }
#ifdef SMG_FDT_PROFILE
  if (prof)
    for (int k = 0; k < FDT_NPH; ++k) atomicAdd(A.phases + k, ph[k]);
#endif
  if (tid == 0) bulk_wait0();
  cp_async_wait<0>();
}

// Ring fixup (second launch): an own node within n_o (+1) of its tile's edge
// also lies in the regions of the neighbour tiles; it receives their ring
// contributions from the workspace, added in a fixed neighbour order
// (dy, dx) = (-1,-1), (-1,0), ..., (1,1).  One thread per band node; no
// atomics; deterministic.
template <int P, int NO, int TX, int TY>
__device__ __forceinline__ void fdt_fixup_node(double* __restrict__ u, const double* __restrict__ ws, int N_x,
                                               int ntx, int nty, long gid) {
  using G = FDTGeom<P, NO, TX, TY>;
  constexpr int OX = G::OX, OY = G::OY, RX = G::RX, RY = G::RY, BW = G::BW;
  constexpr int NRING = G::NRING, NTB = (RY - OY) * RX;
  // band of the own block: rows [0, BW-NO) u [OY-NO, OY) full width, and the
  // columns [0, BW-NO) u [OX-NO, OX) of the rows in between
  constexpr int LO = NO + 1;
  constexpr int NROWS = LO + NO;
  constexpr int PER = NROWS * OX + (OY - NROWS) * (LO + NO);
  static_assert(OY >= NROWS && OX >= LO + NO, "tile smaller than its band");
  (void)BW;
  const int ntiles = ntx * nty;
  if (gid >= (long)ntiles * PER) return;
  // last tiles first: the main kernel finished with them, so their u and ring
  // entries are the ones still resident in L2
  const int tr = (int)(gid / PER);
  const int tile = ntiles - 1 - tr;
  const int k = (int)(gid - (long)tr * PER);
  int oy, ox;
  if (k < NROWS * OX) {
    const int yy = k / OX;
    ox = k - yy * OX;
    oy = yy < LO ? yy : OY - NROWS + yy;
  } else {
    const int k2 = k - NROWS * OX, yy = k2 / (LO + NO), xx = k2 - yy * (LO + NO);
    oy = LO + yy;
    ox = xx < LO ? xx : OX - (LO + NO) + xx;
  }
  const int tx = tile % ntx, ty = tile / ntx;
  double* up = u + (size_t)(ty * OY + oy) * N_x + (tx * OX + ox);
  // every ring entry this node receives is loaded before any is added (one
  // round trip instead of a chain); added in the fixed neighbour order
  // (dy, dx) = (-1,-1), (-1,0), ..., (1,1)
  double val[8];
  int nv = 0;
  const double own = *up;
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
    const int ry = oy + NO - dy * OY;
    const int tyn = wrapi(ty + dy, nty);
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      if (dx == 0 && dy == 0) continue;
      const int rx = ox + NO - dx * OX;
      const bool in = ry >= 0 && ry < RY && rx >= 0 && rx < RX;
      int k = 0;  // compact ring index of region node (ry, rx) of the neighbour
      if (ry < NO || ry >= NO + OY) k = (ry < NO ? ry : ry - OY) * RX + rx;
      else k = NTB + (ry - NO) * (RX - OX) + (rx < NO ? rx : rx - OX);
      const int slot = (dy + 1) * 3 + (dx + 1) - ((dy + 1) * 3 + (dx + 1) > 4 ? 1 : 0);
      val[slot] = in ? ws[(size_t)(tyn * ntx + wrapi(tx + dx, ntx)) * NRING + k] : 0.0;
      nv += in ? 1 : 0;
    }
  }
  (void)nv;
  double acc = own;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    // absent neighbours contribute an exact 0.0 -- but x + 0.0 == x only for
    // x != -0.0; keep the reference order and skip them explicitly
    const int dy = (q < 4 ? q : q + 1) / 3 - 1, dx = (q < 4 ? q : q + 1) % 3 - 1;
    const int ry = oy + NO - dy * OY, rx = ox + NO - dx * OX;
    if (ry >= 0 && ry < RY && rx >= 0 && rx < RX) acc += val[q];
  }
  *up = acc;
}

template <int P, int NO, int TX, int TY>
__global__ void __launch_bounds__(256) fdt_fixup(double* __restrict__ u, const double* __restrict__ ws, int N_x,
                                                 int ntx, int nty) {
  SMG_PDL_ENTRY();
  fdt_fixup_node<P, NO, TX, TY>(u, ws, N_x, ntx, nty, (long)blockIdx.x * blockDim.x + threadIdx.x);
}

struct FDTLaunch {
  const double* r;
  double* u;
  int u_zero;
  const double* inv_nu;
  const double* dinv;        // permuted (even/odd) 1/(lam_y + lam_x)
  double* ws;
  int N_x, N_y, n_x, ntx, nty;
  const double* Sye;   // host, HE*HE row-major [k][i]
  const double* Syo;   // host, HO*HO
  const double* Sxe;
  const double* Sxo;
  const double* wx;
  const double* wy;
};

template <int P, int NO, int TX, int TY, bool DM>
int fdt_launch_k(const FDTLaunch& L, cudaStream_t st) {
  using G = FDTGeom<P, NO, TX, TY>;
  using K = FDTK<P, NO, TX, TY, DM>;
  constexpr int M = G::M, HE = fdt_he(M), HO = fdt_ho(M);
  FDTArgs<M> A;
  // TMA needs 16-byte rows and base addresses; the caller falls back to the
  // coloured dense kernel on SMG_EUNSUPPORTED
  if (!tmap_2d(&A.rmap, L.r, L.N_x, L.N_y, G::BRX, G::RY) || !tmap_2d(&A.umap, L.u, L.N_x, L.N_y, G::OX, G::OY))
    return SMG_EUNSUPPORTED;
  A.r = L.r; A.u = L.u; A.inv_nu = L.inv_nu; A.dinv = L.dinv; A.ws = L.ws;
  A.N_x = L.N_x; A.N_y = L.N_y; A.n_x = L.n_x; A.ntx = L.ntx; A.nty = L.nty;
  A.u_zero = L.u_zero;
  A.phases = fdt_phase_buffer();
  // synthesis factors carry the weight of their output node: W (S t S^T) =
  // (diag(w_y) S_y) t (diag(w_x) S_x)^T, and w is mirror-symmetric, so the
  // even/odd recombination e +- o inherits it
  for (int k = 0; k < HE; ++k)
    for (int i = 0; i < HE; ++i) {
      A.Sye[k * HE + i] = L.Sye[k * HE + i]; A.SyeT[i * HE + k] = L.Sye[k * HE + i] * L.wy[k];
      A.Sxe[k * HE + i] = L.Sxe[k * HE + i]; A.SxeT[i * HE + k] = L.Sxe[k * HE + i] * L.wx[k];
    }
  for (int k = 0; k < HO; ++k)
    for (int i = 0; i < HO; ++i) {
      A.Syo[k * HO + i] = L.Syo[k * HO + i]; A.SyoT[i * HO + k] = L.Syo[k * HO + i] * L.wy[k];
      A.Sxo[k * HO + i] = L.Sxo[k * HO + i]; A.SxoT[i * HO + k] = L.Sxo[k * HO + i] * L.wx[k];
    }
  A.Syo[HO * HO] = A.SyoT[HO * HO] = A.Sxo[HO * HO] = A.SxoT[HO * HO] = 0.0;
  static DeviceInt grid_cap;
  if (grid_cap == 0) {
    if (K::TSMEM > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(fdt_kernel<P, NO, TX, TY, DM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)K::TSMEM);
      if (e != cudaSuccess) return cuda_fail(e, "fdt_kernel smem attribute");
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fdt_kernel<P, NO, TX, TY, DM>, K::NT, K::TSMEM);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int ntiles = L.ntx * L.nty;
  const int grid = ntiles < grid_cap ? ntiles : grid_cap;
  launch(fdt_kernel<P, NO, TX, TY, DM>, dim3(grid), dim3(K::NT), K::TSMEM, st, A);
  int rc = check_launch("fdt_kernel");
  if (rc) return rc;
  const long nb = fdt_fixup_per_tile<P, NO, TX, TY>() * ntiles;
  launch(fdt_fixup<P, NO, TX, TY>, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, st, L.u, L.ws, L.N_x, L.ntx,
         L.nty);
  return check_launch("fdt_fixup");
}

using FDTLaunchFn = int (*)(const FDTLaunch&, cudaStream_t);
// Tiled kernel for (p, n_o) on an n_x x n_y mesh, or nullptr; sets TX, TY.
// dmma selects the even/odd FP64 tensor-core (DMMA) contraction engine of the
// same kernel where it is compiled (m >= 27), else the DFMA engine.
FDTLaunchFn fdt_dispatch(int p, int n_o, int n_x, int n_y, int* TX, int* TY, bool dmma);
// Paired-line engine (smg_fdp.cuh) for (p, n_o) on this mesh, or nullptr; sets TX, TY.
FDTLaunchFn fdp_dispatch(int p, int n_o, int n_x, int n_y, int* TX, int* TY);

}  // namespace smg
