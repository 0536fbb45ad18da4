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
  int debug_skip;                     // profiling aid: 1 = skip the four contractions
  int u_zero;                         // 1: u holds no valid data and is treated as 0 (write, not add)
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

// Persistent main kernel: CTA walks tiles blockIdx.x, +gridDim.x, ...; the
// next tile's residual region and own u are in flight (cp.async group) while
// the current tile computes.  Exclusive nodes are written to u directly,
// band nodes (within n_o of a tile edge) to the workspace for fdt_fixup.
template <int P, int NO, int TX, int TY>
__global__ void __launch_bounds__(FDTGeom<P, NO, TX, TY>::THREADS, FDTGeom<P, NO, TX, TY>::MINB)
fdt_kernel(const __grid_constant__ FDTArgs<P + 1 + 2 * NO> A) {
  SMG_PDL_ENTRY();
  using G = FDTGeom<P, NO, TX, TY>;
  constexpr int M = G::M, MM = G::MM, E = G::E, OX = G::OX, OY = G::OY, RX = G::RX, RY = G::RY;
  constexpr int HE = G::HE, HO = G::HO, HOX = G::HOX, BW = G::BW, NT = G::NT, NH = G::NH, STAGE = G::STAGE;
  extern __shared__ double sm[];
  double* EB = sm + 2 * STAGE;  // E x M x M element buffers
  const int tid = threadIdx.x;
  const int N_x = A.N_x, N_y = A.N_y, ntx = A.ntx, ntiles = A.ntx * A.nty;

  const bool odd = tid >= NH;     // warp-uniform
  const int line = odd ? tid - NH : tid;
  const int e = line / M, c = line - e * M;
  const bool act = e < E;
  const int exl = e % TX, eyl = e / TX;
  double* B = EB + e * MM;
  // this thread's half row of 1/(lam_y + lam_x) (L1-resident across tiles)
  const double* dl = A.dinv + (act ? c : 0) * M + (odd ? HE : 0);

  int tile = blockIdx.x;
  if (tile < ntiles) fdt_prefetch<P, NO, TX, TY, NT>(A.r, A.u, N_x, N_y, ntx, tile, sm, A.u_zero != 0);
  cp_async_commit();
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    double* R = sm + (it & 1) * STAGE;  // residual region, then accumulated correction
    double* UO = R + RX * RY;           // own u
    {
      const int nxt = tile + gridDim.x;
      if (nxt < ntiles) fdt_prefetch<P, NO, TX, TY, NT>(A.r, A.u, N_x, N_y, ntx, nxt, sm + ((it + 1) & 1) * STAGE, A.u_zero != 0);
      cp_async_commit();
    }
    const int tx = tile % ntx, ty = tile / ntx;
    const int X0 = tx * OX, Y0 = ty * OY;
    double s = 1.0;  // 1 / nu_bar of this element
    if (act && A.inv_nu != nullptr) s = __ldg(A.inv_nu + (size_t)(ty * TY + eyl) * A.n_x + (tx * TX + exl));
    cp_async_wait<1>();
    __syncthreads();

    if (A.debug_skip) {
      for (int idx = tid; idx < RX * RY; idx += NT) R[idx] = 0.0;
      __syncthreads();
    } else {
      // ---- stage 1 (physical columns c): [T1e; T1o][:, c] = [Se; So]^T fold_y(R_e[:, c])
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

      // ---- stage 2 (eigen-y rows c): T2[c, :] = ([Se; So]^T fold_x(T1[c, :])) * dinv / nu_bar
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
            for (int l = 0; l < HE; ++l) B[c * M + l] = t[l] * (__ldg(dl + l) * s);
          } else {
#pragma unroll
            for (int l = 0; l < HO; ++l) B[c * M + HE + l] = t[l] * (__ldg(dl + l) * s);
          }
        }
      }
      __syncthreads();

      // ---- stage 3 (eigen-x columns c): even warps e = SyeT^T T2e[:, c] -> rows [0,HE),
      //      odd warps o = SyoT^T T2o[:, c] -> rows [HE, M)   (e/o recombined in stage 4)
      {
        double acc[HE];
        if (act) {
          if (!odd) {
            double t[HE];
#pragma unroll
            for (int i = 0; i < HE; ++i) t[i] = B[i * M + c];
            half_synth<HE>(A.SyeT, t, acc);
          } else if (HO > 0) {
            double t[HOX];
#pragma unroll
            for (int i = 0; i < HO; ++i) t[i] = B[(HE + i) * M + c];
            half_synth<HOX>(A.SyoT, t, reinterpret_cast<double(&)[HOX]>(acc));
          }
        }
        __syncthreads();  // every column read before the in-place writes
        if (act) {
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
            half_synth<HE>(A.SxeT, t, acc);
          } else if (HO > 0) {
            double t[HOX];
#pragma unroll
            for (int i = 0; i < HO; ++i) t[i] = t3(HE + i);
            half_synth<HOX>(A.SxoT, t, reinterpret_cast<double(&)[HOX]>(acc));
          }
        }
        __syncthreads();  // every row read before B is reused for ex / ox
        if (act) {
          // even warps keep ex in B[c][0,HE), odd warps ox in B[c][HE,M)
          if (!odd) {
#pragma unroll
            for (int k = 0; k < HE; ++k) B[c * M + k] = acc[k];
          } else {
#pragma unroll
            for (int k = 0; k < HO; ++k) B[c * M + HE + k] = acc[k];
          }
        }
      }
      __syncthreads();

      // ---- recombine out[c, j] = W (ex +- ox) and add into the region in colour
      //      passes (disjoint windows per pass); thread = (element, row c, half)
      {
        constexpr int C = G::C;
        const double wyc = act ? A.wy[c] : 0.0;
#pragma unroll
        for (int pass = 0; pass < C * C; ++pass) {
          if (act && (eyl % C) * C + (exl % C) == pass) {
            const double* br = B + c * M;
            double* dst = R + (eyl * P + c) * RX + exl * P;
            if (!odd) {
              // columns j in [0, HE): y[j] = ex[j] + ox[j] (centre: ex only)
#pragma unroll
              for (int j = 0; j < HE; ++j) {
                const double y = j < HO ? br[j] + br[HE + j] : br[j];
                dst[j] += y * (wyc * A.wx[j]);
              }
            } else {
              // columns m-1-j, j in [0, HO): y = ex[j] - ox[j]
#pragma unroll
              for (int j = 0; j < HO; ++j) {
                const double y = br[j] - br[HE + j];
                dst[M - 1 - j] += y * (wyc * A.wx[M - 1 - j]);
              }
            }
          }
          __syncthreads();
        }
      }
    }

    // ---- write-out: exclusive nodes to u, band nodes to the workspace ------
    double* W = A.ws + (size_t)tile * (RX * RY);
    for (int idx = tid; idx < RX * RY; idx += NT) {
      const int y = idx / RX, x = idx - y * RX;
      const bool band = (x < BW) || (x >= RX - BW) || (y < BW) || (y >= RY - BW);
      if (band) {
        W[idx] = R[idx];
      } else {
        const int oy = y - NO, ox = x - NO;
        A.u[(size_t)(Y0 + oy) * N_x + (X0 + ox)] = A.u_zero ? R[idx] : UO[oy * OX + ox] + R[idx];
      }
    }
    __syncthreads();  // this stage buffer is refilled two iterations later
  }
  cp_async_wait<0>();
}

// Band fixup (second launch): every node within n_o of a tile edge receives
// the contributions of the 2 (edge) or 4 (corner) tiles sharing it, summed in
// a fixed tile order: u = (((u + c_lo,lo) + c_hi,lo) + c_lo,hi) + c_hi,hi.
// One thread per band node; deterministic; no atomics.
template <int P, int NO, int TX, int TY>
__global__ void __launch_bounds__(256) fdt_fixup(double* __restrict__ u, const double* __restrict__ ws, int N_x,
                                                 int N_y, int ntx, int nty, int u_zero) {
  SMG_PDL_ENTRY();
  using G = FDTGeom<P, NO, TX, TY>;
  constexpr int OX = G::OX, OY = G::OY, RX = G::RX, RY = G::RY, BW = G::BW;
  constexpr size_t RS = (size_t)RX * RY;
  // per tile: x-edge segment (BW x (OY - BW)) at its left edge, y-edge
  // segment ((OX - BW) x BW) at its bottom edge, corner BW x BW at lower-left
  constexpr int NXE = BW * (OY - BW), NYE = (OX - BW) * BW, NCO = BW * BW;
  constexpr int PER = NXE + NYE + NCO;
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int ntiles = ntx * nty;
  if (gid >= (long)ntiles * PER) return;
  const int tile = (int)(gid / PER);
  int k = (int)(gid - (long)tile * PER);
  const int tx = tile % ntx, ty = tile / ntx;
  const int txm = (tx + ntx - 1) % ntx, tym = (ty + nty - 1) % nty;
  const int X0 = tx * OX, Y0 = ty * OY;
  if (k < NXE) {
    // left x-edge of (tx, ty): rows of its y-interior, d in [-NO, NO]
    const int yy = BW + k / BW, d = k % BW - NO;
    const double cl = ws[(size_t)(ty * ntx + txm) * RS + (size_t)yy * RX + (OX + NO + d)];
    const double cr = ws[(size_t)(ty * ntx + tx) * RS + (size_t)yy * RX + (NO + d)];
    double* up = u + (size_t)(Y0 - NO + yy) * N_x + wrapi(X0 + d, N_x);
    *up = ((u_zero ? 0.0 : *up) + cl) + cr;
    return;
  }
  k -= NXE;
  if (k < NYE) {
    // bottom y-edge of (tx, ty): columns of its x-interior
    const int d = k / (OX - BW) - NO, xx = BW + k % (OX - BW);
    const double cb = ws[(size_t)(tym * ntx + tx) * RS + (size_t)(OY + NO + d) * RX + xx];
    const double ct = ws[(size_t)(ty * ntx + tx) * RS + (size_t)(NO + d) * RX + xx];
    double* up = u + (size_t)wrapi(Y0 + d, N_y) * N_x + (X0 - NO + xx);
    *up = ((u_zero ? 0.0 : *up) + cb) + ct;
    return;
  }
  k -= NYE;
  {
    // lower-left corner of (tx, ty): tiles (txm,tym), (tx,tym), (txm,ty), (tx,ty)
    const int dy = k / BW - NO, dx = k % BW - NO;
    const double c00 = ws[(size_t)(tym * ntx + txm) * RS + (size_t)(OY + NO + dy) * RX + (OX + NO + dx)];
    const double c10 = ws[(size_t)(tym * ntx + tx) * RS + (size_t)(OY + NO + dy) * RX + (NO + dx)];
    const double c01 = ws[(size_t)(ty * ntx + txm) * RS + (size_t)(NO + dy) * RX + (OX + NO + dx)];
    const double c11 = ws[(size_t)(ty * ntx + tx) * RS + (size_t)(NO + dy) * RX + (NO + dx)];
    double* up = u + (size_t)wrapi(Y0 + dy, N_y) * N_x + wrapi(X0 + dx, N_x);
    *up = ((((u_zero ? 0.0 : *up) + c00) + c10) + c01) + c11;
  }
}

struct FDTLaunch {
  const double* r;
  double* u;
  int u_zero;
  const double* inv_nu;
  const double* dinv;        // permuted (even/odd) 1/(lam_y + lam_x)
  const double* dinv_dense;  // natural order (DMMA variant)
  const double* Sx_dev;      // device factors (DMMA variant)
  const double* Sy_dev;
  const double* frag_dev;    // lane-ordered DMMA fragments (fdm_fragments)
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
  {
    const char* dbg = getenv("SMG_FD_DEBUG_SKIP");
    A.debug_skip = (dbg && dbg[0] == '1') ? 1 : 0;
  }
  A.u_zero = L.u_zero;
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
  static int grid_cap = 0;
  if (grid_cap == 0) {
    if (G::SMEM > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(fdt_kernel<P, NO, TX, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)G::SMEM);
      if (e != cudaSuccess) return cuda_fail(e, "fdt_kernel smem attribute");
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fdt_kernel<P, NO, TX, TY>, G::THREADS, G::SMEM);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int ntiles = L.ntx * L.nty;
  launch(fdt_kernel<P, NO, TX, TY>, dim3(ntiles < grid_cap ? ntiles : grid_cap), dim3(G::THREADS), G::SMEM, st, A);
  int rc = check_launch("fdt_kernel");
  if (rc) return rc;
  constexpr long PER = (long)G::BW * (G::OY - G::BW) + (long)(G::OX - G::BW) * G::BW + (long)G::BW * G::BW;
  const long nb = PER * ntiles;
  launch(fdt_fixup<P, NO, TX, TY>, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, st, L.u, L.ws, L.N_x, L.N_y,
         L.ntx, L.nty, L.u_zero);
  return check_launch("fdt_fixup");
}

using FDTLaunchFn = int (*)(const FDTLaunch&, cudaStream_t);
// Tiled kernel for (p, n_o) on an n_x x n_y mesh, or nullptr; sets TX, TY.
// dmma selects the FP64 tensor-core variant (smg_fdm.cuh) of the same tiling.
FDTLaunchFn fdt_dispatch(int p, int n_o, int n_x, int n_y, int* TX, int* TY, bool dmma);

}  // namespace smg
