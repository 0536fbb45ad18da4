// Matrix-free GLL operator apply / residual (subsystem 2).
//
// Reference: PoissonOperator.apply (operators.py:49-54),
// DiffusionOperator.apply (operators.py:86-92), residual (:101-103).
// The reference gathers (p+1)^2 element blocks, applies the element kernel
// by sum factorization and scatter-adds with bincount.  Both operators are
// sums of an x-part (one 1D operator along every node row, per element) and
// a y-part (along every node column):
//   Poisson   : (A u)[Y,X] = (dy/dx) Wy(Y) sum_{e in row}  (u_e L)[b]
//                          + (dx/dy) Wx(X) sum_{e in col}  (L u_e)[a]
//   Diffusion : x-part = (dy/dx) Wy(Y) sum_e sum_j nu w_j (D u_e)_j D[j][b]
//               y-part = (dx/dy) Wx(X) sum_e sum_i D[i][a] nu w_i (D u_e)_i
// where W*(.) is the assembled GLL weight (w_0 + w_p at element vertices).
// This kernel evaluates that form in GATHER order, so every output node is
// written by exactly one thread: no scatter, no atomics, deterministic.
//
// A CTA owns a TY x TX block of elements.  It stages u (and nu) with a halo
// of one element on the low side plus one node on the high side, computes
// the row passes (one thread per (node row, element)) and the column passes
// (one thread per (node column, element)) with the 1D matrices in the
// constant bank, and combines vertex contributions of neighbouring elements
// in shared memory.  Optional fused outputs: r = f - A u, ||r||^2 partials.
#pragma once
#include "smg_common.cuh"

namespace smg {

template <int P>
struct OpArgs {
  const double* __restrict__ u;
  const double* __restrict__ f;      // nullable: out = A u
  double* __restrict__ out;
  const double* __restrict__ nu;     // diffusion only
  double* __restrict__ partials;     // nullable: per-CTA sum of out^2
  int n_x, n_y, N_x, N_y;
  int TX, TY, tiles_x;
  double cx, cy;
  double Mt[(P + 1) * (P + 1)];      // Poisson: stiffness L-hat; diffusion: D (row-major)
  double w[P + 1];
  double wasm[P];                    // assembled weight by local index a in [0,p)
};

__host__ __device__ inline size_t op_smem_doubles(int P, int TX, int TY, bool diff) {
  const size_t OX = (size_t)TX * P, OY = (size_t)TY * P;
  const size_t HX = OX + P + 1, HY = OY + P + 1;
  return HX * HY * (diff ? 2 : 1) + 2 * OX * OY + OY * (TX + 1) + OX * (TY + 1);
}

template <int P, bool DIFF>
__global__ void __launch_bounds__(256)
op_kernel(const __grid_constant__ OpArgs<P> A) {
  constexpr int NP = P + 1;
  extern __shared__ double sm[];
  const int TX = A.TX, TY = A.TY;
  const int OX = TX * P, OY = TY * P, HX = OX + P + 1, HY = OY + P + 1;
  double* U = sm;
  double* NU = U + HX * HY;
  double* AX = NU + (DIFF ? HX * HY : 0);
  double* AY = AX + OX * OY;
  double* VX = AY + OX * OY;          // [y][exl]: right-vertex value of element exl-1
  double* VY = VX + OY * (TX + 1);    // [x][eyl]
  const int tid = threadIdx.x, nt = blockDim.x;
  const int tx = blockIdx.x % A.tiles_x, ty = blockIdx.x / A.tiles_x;
  const int X0 = tx * OX, Y0 = ty * OY;

  // stage u (and nu) with the low-side element halo
  for (int idx = tid; idx < HX * HY; idx += nt) {
    const int hy = idx / HX, hx = idx - hy * HX;
    const int gy = wrapi(Y0 - P + hy, A.N_y), gx = wrapi(X0 - P + hx, A.N_x);
    const size_t g = (size_t)gy * A.N_x + gx;
    U[idx] = __ldg(A.u + g);
    if (DIFF) NU[idx] = __ldg(A.nu + g);
  }
  __syncthreads();

  // row passes: item = (own row y, element exl-1), exl in [0, TX]
  for (int it = tid; it < OY * (TX + 1); it += nt) {
    const int y = it / (TX + 1), exl = it - y * (TX + 1);
    const double* ur = U + (y + P) * HX + exl * P;   // halo col of element exl-1 is exl*P
    double v[NP];
    if (!DIFF) {
      if (exl == 0) {
        double s = A.Mt[P] * ur[0];
#pragma unroll
        for (int k = 1; k < NP; ++k) s = fma(A.Mt[k * NP + P], ur[k], s);
        v[P] = s;
      } else {
        const double x0 = ur[0];
#pragma unroll
        for (int b = 0; b < NP; ++b) v[b] = A.Mt[b] * x0;
#pragma unroll
        for (int k = 1; k < NP; ++k) {
          const double xk = ur[k];
#pragma unroll
          for (int b = 0; b < NP; ++b) v[b] = fma(A.Mt[k * NP + b], xk, v[b]);
        }
      }
    } else {
      const double* nr = NU + (y + P) * HX + exl * P;
      double g[NP];
      double xk[NP];
#pragma unroll
      for (int k = 0; k < NP; ++k) xk[k] = ur[k];
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        double s = A.Mt[j * NP] * xk[0];
#pragma unroll
        for (int k = 1; k < NP; ++k) s = fma(A.Mt[j * NP + k], xk[k], s);
        g[j] = nr[j] * A.w[j] * s;
      }
      if (exl == 0) {
        double s = g[0] * A.Mt[P];
#pragma unroll
        for (int j = 1; j < NP; ++j) s = fma(g[j], A.Mt[j * NP + P], s);
        v[P] = s;
      } else {
#pragma unroll
        for (int b = 0; b < NP; ++b) v[b] = g[0] * A.Mt[b];
#pragma unroll
        for (int j = 1; j < NP; ++j) {
#pragma unroll
          for (int b = 0; b < NP; ++b) v[b] = fma(g[j], A.Mt[j * NP + b], v[b]);
        }
      }
    }
    if (exl > 0) {
      double* ax = AX + y * OX + (exl - 1) * P;
#pragma unroll
      for (int b = 0; b < P; ++b) ax[b] = v[b];
    }
    VX[y * (TX + 1) + exl] = v[P];
  }

  // column passes: item = (own column x, element eyl-1), eyl in [0, TY]
  for (int it = tid; it < OX * (TY + 1); it += nt) {
    const int x = it / (TY + 1), eyl = it - x * (TY + 1);
    const double* uc = U + (eyl * P) * HX + (x + P);
    double v[NP];
    if (!DIFF) {
      if (eyl == 0) {
        double s = A.Mt[P] * uc[0];
#pragma unroll
        for (int k = 1; k < NP; ++k) s = fma(A.Mt[k * NP + P], uc[k * HX], s);
        v[P] = s;
      } else {
        const double x0 = uc[0];
#pragma unroll
        for (int a = 0; a < NP; ++a) v[a] = A.Mt[a] * x0;
#pragma unroll
        for (int k = 1; k < NP; ++k) {
          const double xk = uc[k * HX];
#pragma unroll
          for (int a = 0; a < NP; ++a) v[a] = fma(A.Mt[k * NP + a], xk, v[a]);
        }
      }
    } else {
      const double* nc = NU + (eyl * P) * HX + (x + P);
      double g[NP];
      double xk[NP];
#pragma unroll
      for (int k = 0; k < NP; ++k) xk[k] = uc[k * HX];
#pragma unroll
      for (int i = 0; i < NP; ++i) {
        double s = A.Mt[i * NP] * xk[0];
#pragma unroll
        for (int k = 1; k < NP; ++k) s = fma(A.Mt[i * NP + k], xk[k], s);
        g[i] = nc[i * HX] * A.w[i] * s;
      }
      if (eyl == 0) {
        double s = g[0] * A.Mt[P];
#pragma unroll
        for (int i = 1; i < NP; ++i) s = fma(g[i], A.Mt[i * NP + P], s);
        v[P] = s;
      } else {
#pragma unroll
        for (int a = 0; a < NP; ++a) v[a] = g[0] * A.Mt[a];
#pragma unroll
        for (int i = 1; i < NP; ++i) {
#pragma unroll
          for (int a = 0; a < NP; ++a) v[a] = fma(g[i], A.Mt[i * NP + a], v[a]);
        }
      }
    }
    if (eyl > 0) {
      double* ay = AY + ((eyl - 1) * P) * OX + x;
#pragma unroll
      for (int a = 0; a < P; ++a) ay[a * OX] = v[a];
    }
    VY[x * (TY + 1) + eyl] = v[P];
  }
  __syncthreads();

  // combine + residual + optional norm partial
  double nrm = 0.0;
  for (int idx = tid; idx < OX * OY; idx += nt) {
    const int y = idx / OX, x = idx - y * OX;
    const int a = y % P, b = x % P;
    double ax = AX[idx], ay = AY[idx];
    if (b == 0) ax += VX[y * (TX + 1) + x / P];
    if (a == 0) ay += VY[x * (TY + 1) + y / P];
    const double val = A.cx * A.wasm[a] * ax + A.cy * A.wasm[b] * ay;
    const size_t g = (size_t)(Y0 + y) * A.N_x + (X0 + x);
    const double r = A.f != nullptr ? __ldg(A.f + g) - val : val;
    A.out[g] = r;
    nrm = fma(r, r, nrm);
  }
  if (A.partials != nullptr) {
    __shared__ double red[32];
    double v1[1] = {nrm};
    __syncthreads();
    block_reduce<1>(v1, red);
    if (tid == 0) A.partials[blockIdx.x] = v1[0];
  }
}

struct OpLaunch {
  const double* u;
  const double* f;
  double* out;
  const double* nu;
  double* partials;
  int p, n_x, n_y, TX, TY, diffusion;
  double cx, cy;
  const double* Mt;   // host (p+1)^2
  const double* w;    // host p+1
  const double* wasm; // host p
};

template <int P>
int op_launch(const OpLaunch& L, cudaStream_t st) {
  OpArgs<P> A;
  A.u = L.u; A.f = L.f; A.out = L.out; A.nu = L.nu; A.partials = L.partials;
  A.n_x = L.n_x; A.n_y = L.n_y; A.N_x = L.n_x * P; A.N_y = L.n_y * P;
  A.TX = L.TX; A.TY = L.TY; A.tiles_x = L.n_x / L.TX;
  A.cx = L.cx; A.cy = L.cy;
  for (int i = 0; i < (P + 1) * (P + 1); ++i) A.Mt[i] = L.Mt[i];
  for (int i = 0; i < P + 1; ++i) A.w[i] = L.w[i];
  for (int i = 0; i < P; ++i) A.wasm[i] = L.wasm[i];
  const size_t smem = sizeof(double) * op_smem_doubles(P, L.TX, L.TY, L.diffusion != 0);
  const int grid = (L.n_x / L.TX) * (L.n_y / L.TY);
  if (L.diffusion) {
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(op_kernel<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return cuda_fail(e, "op_kernel smem attribute");
    }
    op_kernel<P, true><<<grid, 256, smem, st>>>(A);
  } else {
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(op_kernel<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return cuda_fail(e, "op_kernel smem attribute");
    }
    op_kernel<P, false><<<grid, 256, smem, st>>>(A);
  }
  return check_launch("op_kernel");
}

using OpLaunchFn = int (*)(const OpLaunch&, cudaStream_t);
OpLaunchFn op_dispatch(int p);
int op_tx_max(int p);

}  // namespace smg
