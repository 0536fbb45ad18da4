// BLAS-1 with device-resident scalars (subsystem 4) and the p=1 coarse
// pseudo-inverse.  All reductions use a fixed grid and a fixed summation
// tree (grid-stride partials -> per-block tree -> last block sums the
// partials in block order), so results are bitwise reproducible run to run
// (the reference's test_krylov.py:73-81 demands identical histories).
#include <cooperative_groups.h>

#include "smg_common.cuh"
#include "smg_tma.cuh"

namespace smg {

// ws layout: [kReduceBlocks * 8 partial doubles][1 counter word]
constexpr int kPartStride = 8;

static int grid_for_reduce(int64_t n) {
  int64_t g = (n + 4 * kReduceThreads - 1) / (4 * kReduceThreads);
  if (g > kReduceBlocks) g = kReduceBlocks;
  return g < 1 ? 1 : (int)g;
}

static int grid_for(int64_t n) {
  int64_t g = (n + kReduceThreads - 1) / kReduceThreads;
  if (g > kReduceBlocks) g = kReduceBlocks;
  return g < 1 ? 1 : (int)g;
}


__device__ __forceinline__ bool last_block_arrive(double* ws) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int* ctr = reinterpret_cast<unsigned int*>(ws + kReduceBlocks * kPartStride);
    const unsigned int t = atomicAdd(ctr, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  return last;
}

__device__ __forceinline__ void reset_counter(double* ws) {
  if (threadIdx.x == 0) *reinterpret_cast<unsigned int*>(ws + kReduceBlocks * kPartStride) = 0u;
}

// Sum NV per-block partials in block order; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void finish(double (&v)[NV], const double* ws, double* red) {
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += ws[b * kPartStride + k];
  }
  block_reduce<NV>(v, red);
}

template <int NV>
__device__ __forceinline__ void publish(double (&v)[NV], double* ws, double* red) {
  block_reduce<NV>(v, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) ws[blockIdx.x * kPartStride + k] = v[k];
  }
}

__global__ void __launch_bounds__(kReduceThreads)
dot_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n, double* out,
           double* ws) {
  SMG_PDL_ENTRY();
  __shared__ double red[32];
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[0] = fma(x[i], y[i], v[0]);
  publish<1>(v, ws, red);
  if (!last_block_arrive(ws)) return;
  finish<1>(v, ws, red);
  if (threadIdx.x == 0) out[0] = v[0];
  reset_counter(ws);
}

__global__ void __launch_bounds__(kReduceThreads)
sum_kernel(const double* __restrict__ x, int64_t n, double* out, double* ws) {
  SMG_PDL_ENTRY();
  __shared__ double red[32];
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[0] += x[i];
  publish<1>(v, ws, red);
  if (!last_block_arrive(ws)) return;
  finish<1>(v, ws, red);
  if (threadIdx.x == 0) out[0] = v[0];
  reset_counter(ws);
}

// out[0] = z.(r - r_old), out[1] = z.r ; also the Polak-Ribiere bookkeeping
// when scal != nullptr: scal[5] = out0 / scal[0] (beta), scal[0] = out1 (delta).
__global__ void __launch_bounds__(kReduceThreads)
dot2_kernel(const double* __restrict__ z, const double* __restrict__ r, const double* __restrict__ ro,
            int64_t n, double* out, double* scal, double* ws) {
  SMG_PDL_ENTRY();
  __shared__ double red[64];
  double v[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double zi = z[i], ri = r[i];
    v[0] = fma(zi, ro != nullptr ? ri - ro[i] : ri, v[0]);
    v[1] = fma(zi, ri, v[1]);
  }
  publish<2>(v, ws, red);
  if (!last_block_arrive(ws)) return;
  finish<2>(v, ws, red);
  if (threadIdx.x == 0) {
    if (out != nullptr) { out[0] = v[0]; out[1] = v[1]; }
    if (scal != nullptr) { scal[5] = v[0] / scal[0]; scal[0] = v[1]; }
  }
  reset_counter(ws);
}

// krylov.py:95-103 as one pass (breakdown check on device).
__global__ void __launch_bounds__(kReduceThreads)
cg_update_kernel(double* __restrict__ u, const double* r_in, double* r_out, const double* __restrict__ p,
                 const double* __restrict__ q, int64_t n, double* scal, int* flag, double* ws) {
  SMG_PDL_ENTRY();
  __shared__ double red[32];
  const double pq = scal[1];
  if (!(pq > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) flag[0] = 1;
    return;
  }
  const double alpha = scal[0] / pq;
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    u[i] = __dadd_rn(u[i], __dmul_rn(alpha, p[i]));
    const double rn = __dsub_rn(r_in[i], __dmul_rn(alpha, q[i]));
    r_out[i] = rn;
    v[0] = fma(rn, rn, v[0]);
  }
  publish<1>(v, ws, red);
  if (!last_block_arrive(ws)) return;
  finish<1>(v, ws, red);
  if (threadIdx.x == 0) { scal[2] = v[0]; scal[6] = alpha; }
  reset_counter(ws);
}

__global__ void cg_direction_kernel(double* __restrict__ p, const double* __restrict__ z, int64_t n,
                                    const double* scal) {
  SMG_PDL_ENTRY();
  const double beta = scal[5];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

// Polak-Ribiere bookkeeping from all-reduced dot2 sums (strip-parallel MGCG):
// scal[5] = scal[3] / scal[0] (beta), scal[0] = scal[4] (delta).
__global__ void cg_beta_finish_kernel(double* scal) {
  SMG_PDL_ENTRY();
  if (threadIdx.x == 0) {
    scal[5] = scal[3] / scal[0];
    scal[0] = scal[4];
  }
}

__global__ void axpby_kernel(double a, const double* __restrict__ x, double b, double* __restrict__ y, int64_t n) {
  SMG_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __dadd_rn(__dmul_rn(a, x[i]), __dmul_rn(b, y[i]));
}

__global__ void sub_mean_kernel(double* __restrict__ f, int64_t n, const double* sum) {
  SMG_PDL_ENTRY();
  const double mean = sum[0] / (double)n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    f[i] -= mean;
}

// Final sum of op_kernel per-CTA partials (fixed order).
__global__ void __launch_bounds__(kReduceThreads) sum_partials_kernel(const double* __restrict__ part, int nb, double* out) {
  SMG_PDL_ENTRY();
  __shared__ double red[32];
  double v[1] = {0.0};
  for (int b = threadIdx.x; b < nb; b += blockDim.x) v[0] += part[b];
  block_reduce<1>(v, red);
  if (threadIdx.x == 0) out[0] = v[0];
}

// ---- small dense GEMM for the coarse pseudo-inverse ------------------------
// C[M,N] = op(A) op(B) (.* S when S != nullptr); op = transpose when tX.
// 16x16 output tile per CTA, one output per thread, K staged in chunks of 64
// (the coarse matrices are 8..512 wide: small tiles keep many CTAs busy and
// the dependent-FMA chain short).
__global__ void __launch_bounds__(256)
gemm_kernel(int M, int N, int K, const double* __restrict__ A, int lda, int tA,
            const double* __restrict__ B, int ldb, int tB, double* __restrict__ C, int ldc,
            const double* __restrict__ S) {
  SMG_PDL_ENTRY();
  __shared__ double As[16][64 + 1];
  __shared__ double Bs[64][16 + 1];
  const int tid = threadIdx.x;
  const int r = tid / 16, cc = tid % 16;
  const int m0 = blockIdx.y * 16, n0 = blockIdx.x * 16;
  double acc0 = 0.0, acc1 = 0.0;
  for (int k0 = 0; k0 < K; k0 += 64) {
    for (int idx = tid; idx < 16 * 64; idx += 256) {
      const int mm = idx / 64, kk = idx % 64;
      const int gm = m0 + mm, gk = k0 + kk;
      As[mm][kk] = (gm < M && gk < K) ? (tA ? A[(size_t)gk * lda + gm] : A[(size_t)gm * lda + gk]) : 0.0;
      const int kb = idx / 16, nn = idx % 16;
      const int gn = n0 + nn, gkb = k0 + kb;
      Bs[kb][nn] = (gn < N && gkb < K) ? (tB ? B[(size_t)gn * ldb + gkb] : B[(size_t)gkb * ldb + gn]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 64; kk += 2) {
      acc0 = fma(As[r][kk], Bs[kk][cc], acc0);
      acc1 = fma(As[r][kk + 1], Bs[kk + 1][cc], acc1);
    }
    __syncthreads();
  }
  const int gm = m0 + r, gn = n0 + cc;
  if (gm < M && gn < N) {
    double v = acc0 + acc1;
    if (S != nullptr) v *= S[(size_t)gm * N + gn];
    C[(size_t)gm * ldc + gn] = v;
  }
}

int gemm(int M, int N, int K, const double* A, int lda, int tA, const double* B, int ldb, int tB,
         double* C, int ldc, const double* S, cudaStream_t st) {
  dim3 grid((N + 15) / 16, (M + 15) / 16);
  launch(gemm_kernel, dim3(grid), dim3(256), 0, st, M, N, K, A, lda, tA, B, ldb, tB, C, ldc, S);
  return check_launch("gemm_kernel");
}

// ---- plain CG of the coarse level (multigrid.py:196-215), device scalars --
// S[0] = ||b||^2, S[1] = p.q, S[2]/S[3] = rho (ping-pong), S[4] = done, S[5] = iterations
__global__ void __launch_bounds__(kReduceThreads)
ccg_update_kernel(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                  const double* __restrict__ q, int64_t n, double* S, int ro, int rn, double tol,
                  int it, double* ws) {
  SMG_PDL_ENTRY();
  __shared__ double red[32];
  if (S[4] != 0.0) return;
  const double alpha = S[ro] / S[1];
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    const double ri = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
    r[i] = ri;
    v[0] = fma(ri, ri, v[0]);
  }
  publish<1>(v, ws, red);
  if (!last_block_arrive(ws)) return;
  finish<1>(v, ws, red);
  if (threadIdx.x == 0) {
    S[rn] = v[0];
    if (sqrt(v[0]) <= tol * sqrt(S[0])) { S[4] = 1.0; S[5] = (double)it; }
  }
  reset_counter(ws);
}

__global__ void ccg_direction_kernel(double* __restrict__ p, const double* __restrict__ r, int64_t n,
                                     const double* S, int ro, int rn) {
  SMG_PDL_ENTRY();
  if (S[4] != 0.0) return;
  const double beta = S[rn] / S[ro];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(r[i], __dmul_rn(beta, p[i]));
}

__global__ void ccg_dot_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                               double* out, const double* S, double* ws) {
  SMG_PDL_ENTRY();
  __shared__ double red[32];
  if (S != nullptr && S[4] != 0.0) return;
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[0] = fma(x[i], y[i], v[0]);
  publish<1>(v, ws, red);
  if (!last_block_arrive(ws)) return;
  finish<1>(v, ws, red);
  if (threadIdx.x == 0) out[0] = v[0];
  reset_counter(ws);
}

// ---- the whole coarse CG in ONE CTA (Poisson, n_x n_y <= 4096) -------------
// The p = 1 Poisson operator is the periodic 5-point stencil
//   (A u)_ij = cx (2 u - u_W - u_E) + cy (2 u - u_S - u_N),  cx = dy/dx, cy = dx/dy
// (PoissonOperator with the GLL p = 1 mass and stiffness, operators.py:30-54,
// assembled).  x, r, p, q live in shared memory; every dot product is a fixed-
// order block reduction (deterministic); the iteration is the reference's
// plain CG (multigrid.py:196-228) with b = f0 - mean(f0), tol on ||r|| /
// ||b||, at most max_iter steps, u0 = x - mean(x).  One launch replaces the
// ~4 launches per iteration and the host polls of the grid-wide path.
__device__ __forceinline__ double cta_sum(double v, double* sred) {
  // fixed tree: warp shuffles, then warp 0 over the per-warp partials; broadcast
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();                  // sred free (previous broadcast consumed)
  if (lane == 0) sred[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < nw ? sred[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) sred[32] = t;
  }
  __syncthreads();
  return sred[32];
}

__global__ void __launch_bounds__(1024) ccg_cta_kernel(int nx, int ny, double cx, double cy,
                                                      const double* __restrict__ f0, double* __restrict__ u0,
                                                      double tol, int max_iter, double* S) {
  SMG_PDL_ENTRY();
  extern __shared__ __align__(16) double csm[];
  const int n = nx * ny, tid = threadIdx.x, NT = blockDim.x;
  double* x = csm;
  double* r = x + n;
  double* p = r + n;
  double* q = p + n;
  double* sred = q + n;   // 33 doubles
  double v = 0.0;
  for (int i = tid; i < n; i += NT) {
    const double fi = f0[i];
    r[i] = fi;
    v += fi;
  }
  const double mean = cta_sum(v, sred) / (double)n;
  v = 0.0;
  for (int i = tid; i < n; i += NT) {
    const double bi = r[i] - mean;
    r[i] = bi;
    p[i] = bi;
    x[i] = 0.0;
    v = fma(bi, bi, v);
  }
  const double bb = cta_sum(v, sred);
  int it = 0;
  bool ok = bb == 0.0;
  double rho = bb;
  const double thr = tol * sqrt(bb);
  while (!ok && it < max_iter) {
    ++it;
    v = 0.0;
    for (int i = tid; i < n; i += NT) {
      const int iy = i / nx, ix = i - iy * nx;
      const double c = p[i];
      const double w = p[iy * nx + (ix == 0 ? nx - 1 : ix - 1)], e = p[iy * nx + (ix == nx - 1 ? 0 : ix + 1)];
      const double so = p[(iy == 0 ? ny - 1 : iy - 1) * nx + ix], no = p[(iy == ny - 1 ? 0 : iy + 1) * nx + ix];
      const double qi = cx * ((c + c) - w - e) + cy * ((c + c) - so - no);
      q[i] = qi;
      v = fma(c, qi, v);
    }
    const double alpha = rho / cta_sum(v, sred);
    v = 0.0;
    for (int i = tid; i < n; i += NT) {
      x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
      const double ri = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
      r[i] = ri;
      v = fma(ri, ri, v);
    }
    const double rr = cta_sum(v, sred);
    if (sqrt(rr) <= thr) { ok = true; break; }
    const double beta = rr / rho;
    rho = rr;
    for (int i = tid; i < n; i += NT) p[i] = __dadd_rn(r[i], __dmul_rn(beta, p[i]));
    __syncthreads();
  }
  v = 0.0;
  for (int i = tid; i < n; i += NT) v += x[i];
  const double xm = cta_sum(v, sred) / (double)n;
  for (int i = tid; i < n; i += NT) u0[i] = x[i] - xm;
  if (tid == 0) {
    S[4] = ok ? 1.0 : 0.0;
    S[5] = (double)it;
  }
}

int ccg_cta_run(int nx, int ny, double cx, double cy, const double* f0, double* u0, double tol, int max_iter,
                double* S, cudaStream_t st) {
  const long n = (long)nx * ny;
  if (n > 4096 || n < 1) return SMG_EUNSUPPORTED;
  const size_t smem = sizeof(double) * (4 * (size_t)n + 33);
  static DeviceFlag attr;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ccg_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(sizeof(double) * (4 * 4096 + 33)));
    if (e != cudaSuccess) return cuda_fail(e, "ccg_cta_kernel smem attribute");
    attr = true;
  }
  launch(ccg_cta_kernel, dim3(1), dim3(1024), smem, st, nx, ny, cx, cy, f0, u0, tol, max_iter, S);
  return check_launch("ccg_cta_kernel");
}

int ccg_update(double* x, double* r, const double* p, const double* q, int64_t n, double* S, int ro,
               int rn, double tol, int it, double* ws, cudaStream_t st) {
  launch(ccg_update_kernel, dim3(grid_for_reduce(n)), dim3(kReduceThreads), 0, st, x, r, p, q, n, S, ro, rn, tol, it, ws);
  return check_launch("ccg_update_kernel");
}
int ccg_direction(double* p, const double* r, int64_t n, const double* S, int ro, int rn, cudaStream_t st) {
  launch(ccg_direction_kernel, dim3(grid_for(n)), dim3(kReduceThreads), 0, st, p, r, n, S, ro, rn);
  return check_launch("ccg_direction_kernel");
}
int ccg_dot(const double* x, const double* y, int64_t n, double* out, const double* S, double* ws, cudaStream_t st) {
  launch(ccg_dot_kernel, dim3(grid_for_reduce(n)), dim3(kReduceThreads), 0, st, x, y, n, out, S, ws);
  return check_launch("ccg_dot_kernel");
}



// ---- fused small-grid coarse pseudo-inverse --------------------------------
// For n_x, n_y <= 128 the four GEMMs u = Q_y (Lp .* (Q_y^T F Q_x)) Q_x^T are
// done as two launches of row blocks (kRB rows per CTA), each chaining two
// products through shared memory:
//   pinv_a: T2[I,:] = ((Q_y^T F)[I,:] Q_x) .* Lp[I,:]
//   pinv_b: U[J,:]  = ((Q_y T2)[J,:]) Q_x^T
constexpr int kRB = 4;
constexpr int kPinvMax = 128;

template <bool FIRST>
__global__ void __launch_bounds__(256) pinv_rows_kernel(int nx, int ny, const double* __restrict__ Qx,
                                                        const double* __restrict__ Qy, const double* __restrict__ Lp,
                                                        const double* __restrict__ in, double* __restrict__ out) {
  SMG_PDL_ENTRY();
  constexpr int KC = 32;
  __shared__ double T[kRB][kPinvMax];
  __shared__ double Xs[KC][kPinvMax + 1];
  __shared__ double Qs[KC][kRB];
  const int r0 = blockIdx.x * kRB;
  const int tid = threadIdx.x;
  // each thread owns outputs (i, x) for idx = tid + 256 j
  double acc[kRB * kPinvMax / 256];
  constexpr int NO = kRB * kPinvMax / 256;
#pragma unroll
  for (int j = 0; j < NO; ++j) acc[j] = 0.0;
  // phase 1: T[i][x] = sum_k Qy'[k][r0+i] in[k][x]   (Qy' = Q_y, used transposed when FIRST)
  for (int k0 = 0; k0 < ny; k0 += KC) {
    const int kc = min(KC, ny - k0);
    for (int idx = tid; idx < kc * nx; idx += 256) {
      const int k = idx / nx, x = idx - k * nx;
      Xs[k][x] = in[(size_t)(k0 + k) * nx + x];
    }
    for (int idx = tid; idx < kc * kRB; idx += 256) {
      const int k = idx / kRB, i = idx - k * kRB;
      const int row = min(r0 + i, ny - 1);
      Qs[k][i] = FIRST ? Qy[(size_t)(k0 + k) * ny + row] : Qy[(size_t)row * ny + (k0 + k)];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NO; ++j) {
      const int idx = tid + 256 * j;
      const int i = idx / kPinvMax, x = idx - i * kPinvMax;
      if (x < nx) {
        double s = acc[j];
        for (int k = 0; k < kc; ++k) s = fma(Qs[k][i], Xs[k][x], s);
        acc[j] = s;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < NO; ++j) {
    const int idx = tid + 256 * j;
    T[idx / kPinvMax][idx % kPinvMax] = acc[j];
    acc[j] = 0.0;
  }
  __syncthreads();
  // phase 2: out[r0+i][x] = sum_j T[i][j] Qx'[j][x]   (Qx' = Q_x when FIRST, else Q_x^T)
  for (int k0 = 0; k0 < nx; k0 += KC) {
    const int kc = min(KC, nx - k0);
    for (int idx = tid; idx < kc * nx; idx += 256) {
      const int k = idx / nx, x = idx - k * nx;
      Xs[k][x] = FIRST ? Qx[(size_t)(k0 + k) * nx + x] : Qx[(size_t)x * nx + (k0 + k)];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NO; ++j) {
      const int idx = tid + 256 * j;
      const int i = idx / kPinvMax, x = idx - i * kPinvMax;
      if (x < nx) {
        double s = acc[j];
        for (int k = 0; k < kc; ++k) s = fma(T[i][k0 + k], Xs[k][x], s);
        acc[j] = s;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < NO; ++j) {
    const int idx = tid + 256 * j;
    const int i = idx / kPinvMax, x = idx - i * kPinvMax;
    const int row = r0 + i;
    if (x < nx && row < ny) {
      double v = acc[j];
      if (FIRST) v *= Lp[(size_t)row * nx + x];
      out[(size_t)row * nx + x] = v;
    }
  }
}

// ---- single-launch coarse pseudo-inverse on a thread-block cluster ----------
// For n_x, n_y <= 64 (the C1/C2 coarse levels) the whole solve
//   u = Q_y (Lp .* ((Q_y^T F) Q_x)) Q_x^T
// runs in ONE launch of a cluster of kCl CTAs (one SM each).  Every CTA
// bulk-copies F, Q_x, Q_y and its Lp rows into shared memory, computes its
// block of rows of T2 = (Q_y^T F) Q_x .* Lp, the cluster exchanges the T2
// blocks through distributed shared memory (after barrier.cluster), and each
// CTA finishes its rows of U = (Q_y T2) Q_x^T.  Same products, same k order
// as the two-launch path.
constexpr int kCl = 8;
constexpr int kClMax = 64;

// K-term dot product with four independent partial sums (fixed order:
// ((s0 + s1) + (s2 + s3))): the shared-memory load latency of one chain is
// overlapped by the other three.
__device__ __forceinline__ double dot4(const double* __restrict__ a, int sa, const double* __restrict__ b, int sb,
                                       int K) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int k = 0;
#pragma unroll 4
  for (; k + 3 < K; k += 4) {
    s0 = fma(a[k * sa], b[k * sb], s0);
    s1 = fma(a[(k + 1) * sa], b[(k + 1) * sb], s1);
    s2 = fma(a[(k + 2) * sa], b[(k + 2) * sb], s2);
    s3 = fma(a[(k + 3) * sa], b[(k + 3) * sb], s3);
  }
  for (; k < K; ++k) s0 = fma(a[k * sa], b[k * sb], s0);
  return (s0 + s1) + (s2 + s3);
}

constexpr int kClThreads = 512;

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kClThreads)
pinv_cluster_kernel(int nx, int ny, const double* __restrict__ Qx, const double* __restrict__ QxT,
                    const double* __restrict__ Qy, const double* __restrict__ Lp, const double* __restrict__ f,
                    double* __restrict__ u) {
  SMG_PDL_ENTRY();
  namespace cgx = cooperative_groups;
  cgx::cluster_group cl = cgx::this_cluster();
  extern __shared__ __align__(16) double smc[];
  const int rank = (int)cl.block_rank();
  const int rb = (ny + kCl - 1) / kCl;          // rows per CTA
  const int i0 = rank * rb, ni = max(0, min(rb, ny - i0));
  double* F = smc;                               // ny x nx
  double* QY = F + ny * nx;                      // ny x ny
  double* QX = QY + ny * ny;                     // nx x nx
  double* QXT = QX + nx * nx;                    // nx x nx, QXT[j][x] = Q_x[x][j]
  double* T2 = QXT + nx * nx;                    // ny x nx (own rows computed, the rest gathered)
  double* T1 = T2 + ny * nx;                     // rb x nx
  double* LP = T1 + rb * nx;                     // rb x nx
  uint64_t* bar = reinterpret_cast<uint64_t*>(LP + rb * nx);
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    const unsigned b = (unsigned)(8 * (ny * nx + ny * ny + 2 * nx * nx)) + (unsigned)(8 * ni * nx);
    mbar_arrive_expect_tx(bar, b);
    bulk_g2s(F, f, (unsigned)(8 * ny * nx), bar);
    bulk_g2s(QY, Qy, (unsigned)(8 * ny * ny), bar);
    bulk_g2s(QX, Qx, (unsigned)(8 * nx * nx), bar);
    bulk_g2s(QXT, QxT, (unsigned)(8 * nx * nx), bar);
    if (ni > 0) bulk_g2s(LP, Lp + (size_t)i0 * nx, (unsigned)(8 * ni * nx), bar);
  }
  __syncthreads();  // nobody polls the mbarrier before thread 0 has initialised it
  mbar_wait(bar, 0);
  // T1[i][x] = sum_k Qy[k][i0+i] F[k][x]
  for (int idx = tid; idx < ni * nx; idx += kClThreads) {
    const int i = idx / nx, x = idx - i * nx;
    T1[idx] = dot4(QY + i0 + i, ny, F + x, nx, ny);
  }
  __syncthreads();
  // T2[i0+i][x] = (sum_j T1[i][j] Qx[j][x]) * Lp[i0+i][x]
  for (int idx = tid; idx < ni * nx; idx += kClThreads) {
    const int i = idx / nx, x = idx - i * nx;
    T2[(i0 + i) * nx + x] = dot4(T1 + i * nx, 1, QX + x, nx, nx) * LP[idx];
  }
  cl.sync();
  // gather the other CTAs' T2 rows through distributed shared memory
  for (int c = 0; c < kCl; ++c) {
    const int c0 = c * rb, cn = max(0, min(rb, ny - c0));
    if (c == rank || cn == 0) continue;
    const double* rem = cl.map_shared_rank(T2, c);
    for (int idx = tid; idx < cn * nx; idx += kClThreads) T2[c0 * nx + idx] = rem[c0 * nx + idx];
  }
  __syncthreads();
  // T1[i][x] = sum_k Qy[i0+i][k] T2[k][x]
  for (int idx = tid; idx < ni * nx; idx += kClThreads) {
    const int i = idx / nx, x = idx - i * nx;
    T1[idx] = dot4(QY + (i0 + i) * ny, 1, T2 + x, nx, ny);
  }
  __syncthreads();
  // u[i0+i][x] = sum_j T1[i][j] Qx[x][j]
  for (int idx = tid; idx < ni * nx; idx += kClThreads) {
    const int i = idx / nx, x = idx - i * nx;
    u[(size_t)(i0 + i) * nx + x] = dot4(T1 + i * nx, 1, QXT + x, nx, nx);
  }
  cl.sync();  // no CTA leaves while its shared memory may still be read
}

// ---- square power-of-two coarse meshes: compile-time cluster kernel ---------
// Same products and k order as pinv_cluster_kernel, specialised on N (n_x =
// n_y = N) so every dot product is fully unrolled with constant strides, and
// spread over CL = N/4 CTAs (a 16-CTA non-portable cluster at N = 64): each
// CTA owns 4 rows, one output per thread per stage.
template <int N>
__device__ __forceinline__ double pc_dot(const double* __restrict__ a, int sa, const double* __restrict__ b, int sb) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
  for (int k = 0; k < N; k += 4) {
    s0 = fma(a[k * sa], b[k * sb], s0);
    s1 = fma(a[(k + 1) * sa], b[(k + 1) * sb], s1);
    s2 = fma(a[(k + 2) * sa], b[(k + 2) * sb], s2);
    s3 = fma(a[(k + 3) * sa], b[(k + 3) * sb], s3);
  }
  return (s0 + s1) + (s2 + s3);
}

template <int N>
__global__ void __launch_bounds__(4 * N) pinv_sq_kernel(const double* __restrict__ Qx, const double* __restrict__ QxT,
                                                       const double* __restrict__ Qy,
                                                       const double* __restrict__ Lp, const double* __restrict__ f,
                                                       double* __restrict__ u) {
  SMG_PDL_TRIGGER();
  namespace cgx = cooperative_groups;
  cgx::cluster_group cl = cgx::this_cluster();
  constexpr int RB = 4, CLN = N / RB, NN = N * N;
  extern __shared__ __align__(16) double smq[];
  const int rank = (int)cl.block_rank();
  const int i0 = rank * RB;
  double* F = smq;          // N x N
  double* QY = F + NN;      // N x N
  double* QX = QY + NN;     // N x N
  double* QXT = QX + NN;    // N x N
  double* T2 = QXT + NN;    // N x N (own rows computed, the rest gathered)
  double* T1 = T2 + NN;     // RB x N
  double* LP = T1 + RB * N; // RB x N
  uint64_t* bar = reinterpret_cast<uint64_t*>(LP + RB * N);
  const int tid = threadIdx.x;
  if (tid == 0) {
    // the eigenbasis tables are per-handle constants: in flight while the
    // preceding grid (which writes f) drains; f itself after the wait
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, (unsigned)(8 * (3 * NN + RB * N)));
    bulk_g2s(QY, Qy, 8u * NN, bar);
    bulk_g2s(QX, Qx, 8u * NN, bar);
    bulk_g2s(QXT, QxT, 8u * NN, bar);
    bulk_g2s(LP, Lp + (size_t)i0 * N, 8u * RB * N, bar);
  }
  SMG_PDL_WAIT();
  if (tid == 0) {
    mbar_arrive_expect_tx(bar + 1, 8u * NN);
    bulk_g2s(F, f, 8u * NN, bar + 1);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  mbar_wait(bar + 1, 0);
  const int i = tid / N, x = tid - i * N;   // one (row, column) output per thread
  // T1[i][x] = sum_k Qy[k][i0+i] F[k][x]
  T1[tid] = pc_dot<N>(QY + i0 + i, N, F + x, N);
  __syncthreads();
  // T2[i0+i][x] = (sum_j T1[i][j] Qx[j][x]) * Lp[i0+i][x]
  T2[(i0 + i) * N + x] = pc_dot<N>(T1 + i * N, 1, QX + x, N) * LP[tid];
  cl.sync();
  {
    // gather the other CTAs' rows: all remote loads in flight, then stores
    double g[CLN];
#pragma unroll
    for (int c = 0; c < CLN; ++c) g[c] = c == rank ? 0.0 : cl.map_shared_rank(T2, c)[c * RB * N + tid];
#pragma unroll
    for (int c = 0; c < CLN; ++c)
      if (c != rank) T2[c * RB * N + tid] = g[c];
  }
  __syncthreads();
  // T1[i][x] = sum_k Qy[i0+i][k] T2[k][x]
  const double t1 = pc_dot<N>(QY + (i0 + i) * N, 1, T2 + x, N);
  __syncthreads();
  T1[tid] = t1;
  __syncthreads();
  // u[i0+i][x] = sum_j T1[i][j] Qx[x][j]
  u[(size_t)(i0 + i) * N + x] = pc_dot<N>(T1 + i * N, 1, QXT + x, N);
  cl.sync();  // no CTA leaves while its shared memory may still be read
}

template <int N>
int pinv_sq_launch(const double* Qx, const double* QxT, const double* Qy, const double* Lp, const double* f,
                   double* u, cudaStream_t st) {
  constexpr int CLN = N / 4;
  const size_t smem = sizeof(double) * (5 * (size_t)N * N + 8 * (size_t)N) + 32;
  static DeviceFlag attr;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(pinv_sq_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && CLN > 8) e = cudaFuncSetAttribute(pinv_sq_kernel<N>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_fail(e, "pinv_sq_kernel attributes");
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CLN);
  cfg.blockDim = dim3(4 * N);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CLN;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, pinv_sq_kernel<N>, Qx, QxT, Qy, Lp, f, u);
  if (e != cudaSuccess) return cuda_fail(e, "pinv_sq_kernel launch");
  return check_launch("pinv_sq_kernel");
}

int pinv_cluster(int nx, int ny, const double* Qx, const double* QxT, const double* Qy, const double* Lp,
                 const double* f, double* u, cudaStream_t st) {
  if (nx > kClMax || ny > kClMax || (nx * ny) % 2 || (nx * nx) % 2 || (ny * ny) % 2) return 1;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al16(f) || !al16(Qx) || !al16(QxT) || !al16(Qy) || !al16(Lp)) return 1;
  static const int sq = env_int("SMG_PINV_SQ", 1);
  if (sq && nx == ny) {
    if (nx == 64) return pinv_sq_launch<64>(Qx, QxT, Qy, Lp, f, u, st);
    if (nx == 32) return pinv_sq_launch<32>(Qx, QxT, Qy, Lp, f, u, st);
    if (nx == 16) return pinv_sq_launch<16>(Qx, QxT, Qy, Lp, f, u, st);
  }
  const int rb = (ny + kCl - 1) / kCl;
  if (((size_t)rb * nx) % 2) return 1;  // keep every row block 16-byte aligned
  const size_t smem = sizeof(double) * (2 * (size_t)ny * nx + (size_t)ny * ny + 2 * (size_t)nx * nx + 2 * (size_t)rb * nx) + 16;
  static DeviceInt attr;   // largest size set so far, per device
  if ((int)smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(pinv_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "pinv_cluster_kernel smem attribute");
    attr = (int)smem;
  }
  launch(pinv_cluster_kernel, dim3(kCl), dim3(kClThreads), smem, st, nx, ny, Qx, QxT, Qy, Lp, f, u);
  return check_launch("pinv_cluster_kernel");
}

int pinv_small(int nx, int ny, const double* Qx, const double* Qy, const double* Lp, const double* f,
               double* tmp, double* u, cudaStream_t st) {
  if (nx > kPinvMax || ny > kPinvMax) return 1;
  const int grid = (ny + kRB - 1) / kRB;
  launch(pinv_rows_kernel<true>, dim3(grid), dim3(256), 0, st, nx, ny, Qx, Qy, Lp, f, tmp);
  int rc = check_launch("pinv_rows_kernel");
  if (rc) return rc;
  launch(pinv_rows_kernel<false>, dim3(grid), dim3(256), 0, st, nx, ny, Qx, Qy, Lp, tmp, u);
  return check_launch("pinv_rows_kernel");
}

// ---- preconditioned CG of the variable-coefficient coarse level -------------
// S[0] = ||b||^2, S[1] = p.q, S[2]/S[3] = r.z (ping-pong), S[4] = done,
// S[5] = iterations, S[6] = ||r||^2
__global__ void __launch_bounds__(kReduceThreads)
pcg_update_kernel(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                  const double* __restrict__ q, int64_t n, double* S, int ro, double tol, int it, double* ws) {
  SMG_PDL_ENTRY();
  __shared__ double red[32];
  if (S[4] != 0.0) return;
  const double alpha = S[ro] / S[1];
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    const double ri = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
    r[i] = ri;
    v[0] = fma(ri, ri, v[0]);
  }
  publish<1>(v, ws, red);
  if (!last_block_arrive(ws)) return;
  finish<1>(v, ws, red);
  if (threadIdx.x == 0) {
    S[6] = v[0];
    if (sqrt(v[0]) <= tol * sqrt(S[0])) { S[4] = 1.0; S[5] = (double)it; }
  }
  reset_counter(ws);
}

// z = scale * z (preconditioner scaling), skipped once converged
__global__ void pcg_scale_kernel(double* __restrict__ z, int64_t n, double scale, const double* S) {
  SMG_PDL_ENTRY();
  if (S[4] != 0.0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] *= scale;
}

// out = in / sqrt(nu) (the diagonal scaling of the coarse PCG preconditioner
// D^-1/2 A_P^+ D^-1/2), skipped once converged
__global__ void pcg_dscale_kernel(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ nu,
                                  int64_t n, const double* S) {
  SMG_PDL_ENTRY();
  if (S[4] != 0.0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i] / sqrt(nu[i]);
}

int pcg_update(double* x, double* r, const double* p, const double* q, int64_t n, double* S, int ro, double tol,
               int it, double* ws, cudaStream_t st) {
  launch(pcg_update_kernel, dim3(grid_for_reduce(n)), dim3(kReduceThreads), 0, st, x, r, p, q, n, S, ro, tol, it, ws);
  return check_launch("pcg_update_kernel");
}
int pcg_scale(double* z, int64_t n, double scale, const double* S, cudaStream_t st) {
  launch(pcg_scale_kernel, dim3(grid_for(n)), dim3(kReduceThreads), 0, st, z, n, scale, S);
  return check_launch("pcg_scale_kernel");
}
int pcg_dscale(const double* in, double* out, const double* nu, int64_t n, const double* S, cudaStream_t st) {
  launch(pcg_dscale_kernel, dim3(grid_for(n)), dim3(kReduceThreads), 0, st, in, out, nu, n, S);
  return check_launch("pcg_dscale_kernel");
}
}  // namespace smg

using namespace smg;

extern "C" {

size_t smg_reduce_ws_doubles(void) { return (size_t)kReduceBlocks * kPartStride + 2; }

int smg_dot(const double* x, const double* y, int64_t n, double* out, double* ws, void* stream) {
  if (!x || !y || !out || !ws || n < 0) { set_error("smg_dot: bad argument"); return SMG_EINVAL; }
  launch(dot_kernel, dim3(grid_for_reduce(n)), dim3(kReduceThreads), 0, as_stream(stream), x, y, n, out, ws);
  return check_launch("dot_kernel");
}

int smg_sum(const double* x, int64_t n, double* out, double* ws, void* stream) {
  if (!x || !out || !ws || n < 0) { set_error("smg_sum: bad argument"); return SMG_EINVAL; }
  launch(sum_kernel, dim3(grid_for_reduce(n)), dim3(kReduceThreads), 0, as_stream(stream), x, n, out, ws);
  return check_launch("sum_kernel");
}

int smg_dot2(const double* x, const double* y, const double* z, int64_t n, double* out, double* ws,
             void* stream) {
  if (!x || !y || !out || !ws || n < 0) { set_error("smg_dot2: bad argument"); return SMG_EINVAL; }
  launch(dot2_kernel, dim3(grid_for_reduce(n)), dim3(kReduceThreads), 0, as_stream(stream), x, y, z, n, out, nullptr, ws);
  return check_launch("dot2_kernel");
}

int smg_cg_beta(const double* z, const double* r, const double* r_old, int64_t n, double* scal,
                double* ws, void* stream) {
  if (!z || !r || !scal || !ws || n < 0) { set_error("smg_cg_beta: bad argument"); return SMG_EINVAL; }
  launch(dot2_kernel, dim3(grid_for_reduce(n)), dim3(kReduceThreads), 0, as_stream(stream), z, r, r_old, n, nullptr, scal, ws);
  return check_launch("dot2_kernel");
}

int smg_axpby(double alpha, const double* x, double beta, double* y, int64_t n, void* stream) {
  if (!x || !y || n < 0) { set_error("smg_axpby: bad argument"); return SMG_EINVAL; }
  launch(axpby_kernel, dim3(grid_for(n)), dim3(kReduceThreads), 0, as_stream(stream), alpha, x, beta, y, n);
  return check_launch("axpby_kernel");
}

int smg_cg_update2(double* u, const double* r_in, double* r_out, const double* p, const double* q,
                   int64_t n, double* scal, int* flag, double* ws, void* stream) {
  if (!u || !r_in || !r_out || !p || !q || !scal || !flag || !ws) {
    set_error("smg_cg_update: bad argument");
    return SMG_EINVAL;
  }
  launch(cg_update_kernel, dim3(grid_for_reduce(n)), dim3(kReduceThreads), 0, as_stream(stream), u, r_in, r_out, p, q, n, scal, flag, ws);
  return check_launch("cg_update_kernel");
}

int smg_cg_update(double* u, double* r, const double* p, const double* q, int64_t n, double* scal,
                  int* flag, double* ws, void* stream) {
  return smg_cg_update2(u, r, r, p, q, n, scal, flag, ws, stream);
}

int smg_cg_beta_finish(double* scal, void* stream) {
  if (!scal) { set_error("smg_cg_beta_finish: bad argument"); return SMG_EINVAL; }
  launch(cg_beta_finish_kernel, dim3(1), dim3(32), 0, as_stream(stream), scal);
  return check_launch("cg_beta_finish_kernel");
}

int smg_cg_direction(double* p, const double* z, int64_t n, double* scal, void* stream) {
  if (!p || !z || !scal) { set_error("smg_cg_direction: bad argument"); return SMG_EINVAL; }
  launch(cg_direction_kernel, dim3(grid_for(n)), dim3(kReduceThreads), 0, as_stream(stream), p, z, n, scal);
  return check_launch("cg_direction_kernel");
}

int smg_project_mean(double* f, int64_t n, double* ws, void* stream) {
  if (!f || !ws || n <= 0) { set_error("smg_project_mean: bad argument"); return SMG_EINVAL; }
  double* s = ws + (size_t)kReduceBlocks * kPartStride + 1;
  launch(sum_kernel, dim3(grid_for_reduce(n)), dim3(kReduceThreads), 0, as_stream(stream), f, n, s, ws);
  int rc = check_launch("sum_kernel");
  if (rc) return rc;
  launch(sub_mean_kernel, dim3(grid_for(n)), dim3(kReduceThreads), 0, as_stream(stream), f, n, s);
  return check_launch("sub_mean_kernel");
}

int smg_sum_partials(const double* part, int nb, double* out, void* stream) {
  launch(sum_partials_kernel, dim3(1), dim3(kReduceThreads), 0, as_stream(stream), part, nb, out);
  return check_launch("sum_partials_kernel");
}

}  // extern "C"
