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
// 3. Deterministic band protocol.  Nodes within n_o of a tile boundary get
//    contributions from 2 (edges) or 4 (corners) tiles.  Each tile stores its
//    band values in a workspace and bumps a per-band counter; the LAST tile to
//    arrive adds all contributions to u in a fixed tile order.  The sum never
//    depends on arrival order: bitwise reproducible, no FP atomics, one launch.
#pragma once
#include "smg_common.cuh"

namespace smg {

__host__ __device__ constexpr int fdt_he(int M) { return (M + 1) / 2; }  // even half (incl. centre)
__host__ __device__ constexpr int fdt_ho(int M) { return M / 2; }        // odd half

template <int M>
struct FDTArgs {
  const double* __restrict__ r;       // residual (N_y, N_x)
  double* __restrict__ u;             // u += correction
  const double* __restrict__ inv_nu;  // (n_y, n_x) or nullptr
  const double* __restrict__ dinv;    // (M,M), [even | odd] eigen order in both dims
  double* __restrict__ ws;            // band workspace: ntiles * RY * RX
  unsigned int* __restrict__ ctr;     // 3 * ntiles counters (x-edge, y-edge, corner), zeroed
  int N_x, N_y, n_x, ntx, nty;
  // analysis factors Se[k][i] (k physical half index), synthesis factors SeT[i][k]
  double Sye[fdt_he(M) * fdt_he(M)], SyeT[fdt_he(M) * fdt_he(M)];
  double Syo[fdt_ho(M) * fdt_ho(M) + 1], SyoT[fdt_ho(M) * fdt_ho(M) + 1];
  double Sxe[fdt_he(M) * fdt_he(M)], SxeT[fdt_he(M) * fdt_he(M)];
  double Sxo[fdt_ho(M) * fdt_ho(M) + 1], SxoT[fdt_ho(M) * fdt_ho(M) + 1];
  double wx[M], wy[M];
};

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

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
  // two threads per (element, line): lane pair = (even half, odd half)
  static constexpr int THREADS = ((2 * E * M + 31) / 32) * 32;
  static constexpr int NT = THREADS;
  // colours inside the tile: windows of elements C apart are disjoint
  static constexpr int C = (2 * NO < P) ? 2 : 3;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)RX * RY + (size_t)E * MM + (size_t)OX * OY);
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

template <int P, int NO, int TX, int TY>
__global__ void __launch_bounds__(FDTGeom<P, NO, TX, TY>::THREADS, FDTGeom<P, NO, TX, TY>::THREADS <= 320 ? 3 : 2)
fdt_kernel(const __grid_constant__ FDTArgs<P + 1 + 2 * NO> A) {
  using G = FDTGeom<P, NO, TX, TY>;
  constexpr int M = G::M, MM = G::MM, E = G::E, OX = G::OX, OY = G::OY, RX = G::RX, RY = G::RY;
  constexpr int HE = G::HE, HO = G::HO, HOX = G::HOX, BW = G::BW, NT = G::NT;
  extern __shared__ double sm[];
  double* R = sm;               // RY x RX: residual region, then accumulated correction
  double* EB = R + RX * RY;     // E x M x M element buffers
  double* UO = EB + E * MM;     // OY x OX own u
  const int tid = threadIdx.x;
  const int tile = blockIdx.x;
  const int tx = tile % A.ntx, ty = tile / A.ntx;
  const int X0 = tx * OX, Y0 = ty * OY;
  const int N_x = A.N_x, N_y = A.N_y;

  // ---- async stage of the residual region and own u ----------------------
  for (int idx = tid; idx < RX * RY; idx += NT) {
    const int y = idx / RX, x = idx - y * RX;
    const int gy = wrapi(Y0 - NO + y, N_y), gx = wrapi(X0 - NO + x, N_x);
    cp_async8(R + idx, A.r + (size_t)gy * N_x + gx);
  }
  for (int idx = tid; idx < OX * OY; idx += NT) {
    const int y = idx / OX, x = idx - y * OX;
    cp_async8(UO + idx, A.u + (size_t)(Y0 + y) * N_x + (X0 + x));
  }

  const bool odd = tid & 1;
  const int line = tid >> 1;
  const int e = line / M, c = line - e * M;
  const bool act = e < E;
  const int exl = e % TX, eyl = e / TX;
  double* B = EB + e * MM;
  double s = 1.0;  // 1 / nu_bar of this element; fetched while the copies fly
  if (act && A.inv_nu != nullptr) s = __ldg(A.inv_nu + (size_t)(ty * TY + eyl) * A.n_x + (tx * TX + exl));
  double dl[HE];   // this lane's half row of 1/(lam_y + lam_x), also prefetched
  {
    const double* dr = A.dinv + (act ? c : 0) * M + (odd ? HE : 0);
#pragma unroll
    for (int l = 0; l < HE; ++l) dl[l] = (l < (odd ? HO : HE)) ? __ldg(dr + l) : 0.0;
  }
  cp_async_wait_all();
  __syncthreads();

  // ---- stage 1 (physical columns): T1[:, c] = S_y^T R_e[:, c] --------------
  if (act) {
    const double* col = R + (eyl * P) * RX + exl * P + c;
    auto in = [&](int k) { return col[k * RX]; };
    if (!odd) {
      double t[HE];
      half_analyse<M, HE, false>(A.Sye, in, t);
#pragma unroll
      for (int i = 0; i < HE; ++i) B[i * M + c] = t[i];
    } else if (HO > 0) {
      double t[HOX];
      half_analyse<M, HOX, true>(A.Syo, in, t);
#pragma unroll
      for (int i = 0; i < HO; ++i) B[(HE + i) * M + c] = t[i];
    }
  }
  __syncthreads();
  for (int idx = tid; idx < RX * RY; idx += NT) R[idx] = 0.0;  // residual consumed

  // ---- stage 2 (eigen-y rows): T2[c, :] = (T1[c, :] S_x) * dinv / nu_bar ----
  {
    double t[HE];
    const double* row = B + c * M;
    auto in = [&](int k) { return row[k]; };
    if (act) {
      if (!odd) half_analyse<M, HE, false>(A.Sxe, in, t);
      else if (HO > 0) half_analyse<M, HOX, true>(A.Sxo, in, reinterpret_cast<double(&)[HOX]>(t));
    }
    __syncthreads();  // every row read before the in-place writes
    if (act) {
      if (!odd) {
#pragma unroll
        for (int l = 0; l < HE; ++l) B[c * M + l] = t[l] * (dl[l] * s);
      } else {
#pragma unroll
        for (int l = 0; l < HO; ++l) B[c * M + HE + l] = t[l] * (dl[l] * s);
      }
    }
  }
  __syncthreads();

  // ---- stage 3 (eigen-x columns): T3[:, c] = S_y T2[:, c] -----------------
  {
    double acc[HE];
#pragma unroll
    for (int k = 0; k < HE; ++k) acc[k] = 0.0;
    if (act) {
      if (!odd) {
        double t[HE];
#pragma unroll
        for (int i = 0; i < HE; ++i) t[i] = B[i * M + c];
        half_synth<HE>(A.SyeT, t, acc);
      } else if (HO > 0) {
        double t[HOX], a2[HOX];
#pragma unroll
        for (int i = 0; i < HO; ++i) t[i] = B[(HE + i) * M + c];
        half_synth<HOX>(A.SyoT, t, a2);
#pragma unroll
        for (int k = 0; k < HO; ++k) acc[k] = a2[k];
      }
    }
    __syncthreads();  // every column read before the in-place writes
#pragma unroll
    for (int k = 0; k < HO; ++k) {
      const double other = __shfl_xor_sync(0xffffffffu, acc[k], 1);
      if (act) {
        if (!odd) B[k * M + c] = acc[k] + other;          // y[k]     = e + o
        else B[(M - 1 - k) * M + c] = other - acc[k];      // y[m-1-k] = e - o
      }
    }
    if ((M & 1) && act && !odd) B[HO * M + c] = acc[HO];
  }
  __syncthreads();

  // ---- stage 4 (physical rows): out[c, :] = W .* (T3[c, :] S_x^T), added
  //      into the region in colour passes (disjoint windows per pass) -------
  {
    double acc[HE];
#pragma unroll
    for (int k = 0; k < HE; ++k) acc[k] = 0.0;
    if (act) {
      if (!odd) {
        double t[HE];
#pragma unroll
        for (int i = 0; i < HE; ++i) t[i] = B[c * M + i];
        half_synth<HE>(A.SxeT, t, acc);
      } else if (HO > 0) {
        double t[HOX], a2[HOX];
#pragma unroll
        for (int i = 0; i < HO; ++i) t[i] = B[c * M + HE + i];
        half_synth<HOX>(A.SxoT, t, a2);
#pragma unroll
        for (int k = 0; k < HO; ++k) acc[k] = a2[k];
      }
    }
    double y[HE];
#pragma unroll
    for (int k = 0; k < HO; ++k) {
      const double other = __shfl_xor_sync(0xffffffffu, acc[k], 1);
      y[k] = odd ? other - acc[k] : acc[k] + other;
    }
    if (M & 1) y[HO] = acc[HO];
    const double wyc = act ? A.wy[c] : 0.0;
    constexpr int C = G::C;
#pragma unroll
    for (int pass = 0; pass < C * C; ++pass) {
      if (act && (eyl % C) * C + (exl % C) == pass) {
        double* dst = R + (eyl * P + c) * RX + exl * P;
        if (!odd) {
#pragma unroll
          for (int k = 0; k < HE; ++k) dst[k] += y[k] * (wyc * A.wx[k]);
        } else {
#pragma unroll
          for (int k = 0; k < HO; ++k) dst[M - 1 - k] += y[k] * (wyc * A.wx[M - 1 - k]);
        }
      }
      __syncthreads();
    }
  }

  // ---- write-out: band nodes to the workspace, publish, then the exclusive
  //      nodes (their stores overlap the counter round trip) ----------------
  double* W = A.ws + (size_t)tile * (RX * RY);
  for (int idx = tid; idx < RX * RY; idx += NT) {
    const int y = idx / RX, x = idx - y * RX;
    const bool band = (x < BW) || (x >= RX - BW) || (y < BW) || (y >= RY - BW);
    if (band) W[idx] = R[idx];
  }
  __threadfence();
  __syncthreads();
  __shared__ int last[8];
  const int ntx = A.ntx, nty = A.nty, ntiles = ntx * nty;
  const int txm = (tx + ntx - 1) % ntx, txp = (tx + 1) % ntx;
  const int tym = (ty + nty - 1) % nty, typ = (ty + 1) % nty;
  unsigned int arrived = 0u;
  if (tid < 8) {
    // 0 left edge, 1 right edge, 2 bottom edge, 3 top edge,
    // 4 lower-left, 5 lower-right, 6 upper-left, 7 upper-right corner;
    // each indexed by the tile on its high side.
    const int hx = (tid == 1 || tid == 5 || tid == 7) ? txp : tx;
    const int hy = (tid == 3 || tid == 6 || tid == 7) ? typ : ty;
    const int kind = tid < 2 ? 0 : (tid < 4 ? 1 : 2);
    arrived = atomicAdd(A.ctr + kind * ntiles + hy * ntx + hx, 1u);
  }
  for (int idx = tid; idx < RX * RY; idx += NT) {
    const int y = idx / RX, x = idx - y * RX;
    const bool band = (x < BW) || (x >= RX - BW) || (y < BW) || (y >= RY - BW);
    if (!band) {
      const int oy = y - NO, ox = x - NO;
      A.u[(size_t)(Y0 + oy) * N_x + (X0 + ox)] = UO[oy * OX + ox] + R[idx];
    }
  }
  if (tid < 8) {
    last[tid] = arrived == (tid < 4 ? 1u : 3u);
    __threadfence();
  }
  __syncthreads();
  constexpr size_t RS = (size_t)RX * RY;
  // x edges: (left tile, right tile) at X = right tile's X0, y-interior rows
#pragma unroll
  for (int sg = 0; sg < 2; ++sg) {
    if (!last[sg]) continue;
    const int tl = sg == 0 ? txm : tx, tr = sg == 0 ? tx : txp;
    const int XB = tr * OX;
    const double* WL = A.ws + (size_t)(ty * ntx + tl) * RS;
    const double* WR = A.ws + (size_t)(ty * ntx + tr) * RS;
    constexpr int NR = RY - 2 * BW;
    for (int idx = tid; idx < NR * BW; idx += NT) {
      const int yy = BW + idx / BW, d = idx % BW - NO;
      const int gx = wrapi(XB + d, N_x), gy = Y0 - NO + yy;
      const double cl = __ldcg(WL + (size_t)yy * RX + (OX + NO + d));
      const double cr = __ldcg(WR + (size_t)yy * RX + (NO + d));
      double* up = A.u + (size_t)gy * N_x + gx;
      *up = (*up + cl) + cr;
    }
    if (tid == 0) A.ctr[ty * ntx + tr] = 0u;
  }
  // y edges: (bottom tile, top tile) at Y = top tile's Y0, x-interior columns
#pragma unroll
  for (int sg = 2; sg < 4; ++sg) {
    if (!last[sg]) continue;
    const int tb = sg == 2 ? tym : ty, tt = sg == 2 ? ty : typ;
    const int YB = tt * OY;
    const double* WB = A.ws + (size_t)(tb * ntx + tx) * RS;
    const double* WT = A.ws + (size_t)(tt * ntx + tx) * RS;
    constexpr int NC = RX - 2 * BW;
    for (int idx = tid; idx < NC * BW; idx += NT) {
      const int d = idx / NC - NO, xx = BW + idx % NC;
      const int gy = wrapi(YB + d, N_y), gx = X0 - NO + xx;
      const double cb = __ldcg(WB + (size_t)(OY + NO + d) * RX + xx);
      const double ct = __ldcg(WT + (size_t)(NO + d) * RX + xx);
      double* up = A.u + (size_t)gy * N_x + gx;
      *up = (*up + cb) + ct;
    }
    if (tid == 0) A.ctr[ntiles + tt * ntx + tx] = 0u;
  }
  // corners: tiles (lo,lo), (hi,lo), (lo,hi), (hi,hi) in that order
#pragma unroll
  for (int sg = 4; sg < 8; ++sg) {
    if (!last[sg]) continue;
    const int hx = (sg == 4 || sg == 6) ? tx : txp;
    const int hy = (sg == 4 || sg == 5) ? ty : typ;
    const int lx = (hx + ntx - 1) % ntx, ly = (hy + nty - 1) % nty;
    const int XB = hx * OX, YB = hy * OY;
    const double* W00 = A.ws + (size_t)(ly * ntx + lx) * RS;
    const double* W10 = A.ws + (size_t)(ly * ntx + hx) * RS;
    const double* W01 = A.ws + (size_t)(hy * ntx + lx) * RS;
    const double* W11 = A.ws + (size_t)(hy * ntx + hx) * RS;
    for (int idx = tid; idx < BW * BW; idx += NT) {
      const int dy = idx / BW - NO, dx = idx % BW - NO;
      const int gy = wrapi(YB + dy, N_y), gx = wrapi(XB + dx, N_x);
      const double c00 = __ldcg(W00 + (size_t)(OY + NO + dy) * RX + (OX + NO + dx));
      const double c10 = __ldcg(W10 + (size_t)(OY + NO + dy) * RX + (NO + dx));
      const double c01 = __ldcg(W01 + (size_t)(NO + dy) * RX + (OX + NO + dx));
      const double c11 = __ldcg(W11 + (size_t)(NO + dy) * RX + (NO + dx));
      double* up = A.u + (size_t)gy * N_x + gx;
      *up = (((*up + c00) + c10) + c01) + c11;
    }
    if (tid == 0) A.ctr[2 * ntiles + hy * ntx + hx] = 0u;
  }
}

struct FDTLaunch {
  const double* r;
  double* u;
  const double* inv_nu;
  const double* dinv;
  double* ws;
  unsigned int* ctr;
  int N_x, N_y, n_x, ntx, nty;
  const double* Sye;   // host, HE*HE row-major [k][i]
  const double* Syo;   // host, HO*HO
  const double* Sxe;
  const double* Sxo;
  const double* wx;
  const double* wy;
};

template <int P, int NO, int TX, int TY>
int fdt_launch(const FDTLaunch& L, cudaStream_t st) {
  using G = FDTGeom<P, NO, TX, TY>;
  constexpr int M = G::M, HE = fdt_he(M), HO = fdt_ho(M);
  FDTArgs<M> A;
  A.r = L.r; A.u = L.u; A.inv_nu = L.inv_nu; A.dinv = L.dinv; A.ws = L.ws; A.ctr = L.ctr;
  A.N_x = L.N_x; A.N_y = L.N_y; A.n_x = L.n_x; A.ntx = L.ntx; A.nty = L.nty;
  for (int k = 0; k < HE; ++k)
    for (int i = 0; i < HE; ++i) {
      A.Sye[k * HE + i] = L.Sye[k * HE + i]; A.SyeT[i * HE + k] = L.Sye[k * HE + i];
      A.Sxe[k * HE + i] = L.Sxe[k * HE + i]; A.SxeT[i * HE + k] = L.Sxe[k * HE + i];
    }
  for (int k = 0; k < HO; ++k)
    for (int i = 0; i < HO; ++i) {
      A.Syo[k * HO + i] = L.Syo[k * HO + i]; A.SyoT[i * HO + k] = L.Syo[k * HO + i];
      A.Sxo[k * HO + i] = L.Sxo[k * HO + i]; A.SxoT[i * HO + k] = L.Sxo[k * HO + i];
    }
  A.Syo[HO * HO] = A.SyoT[HO * HO] = A.Sxo[HO * HO] = A.SxoT[HO * HO] = 0.0;
  for (int i = 0; i < M; ++i) { A.wx[i] = L.wx[i]; A.wy[i] = L.wy[i]; }
  static bool attr = false;
  if (!attr) {
    if (G::SMEM > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(fdt_kernel<P, NO, TX, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)G::SMEM);
      if (e != cudaSuccess) return cuda_fail(e, "fdt_kernel smem attribute");
    }
    attr = true;
  }
  fdt_kernel<P, NO, TX, TY><<<L.ntx * L.nty, G::THREADS, G::SMEM, st>>>(A);
  return check_launch("fdt_kernel");
}

using FDTLaunchFn = int (*)(const FDTLaunch&, cudaStream_t);
// Tiled kernel for (p, n_o) on an n_x x n_y mesh, or nullptr; sets TX, TY.
FDTLaunchFn fdt_dispatch(int p, int n_o, int n_x, int n_y, int* TX, int* TY);

}  // namespace smg
