// Fused additive-Schwarz fast-diagonalization kernel (subsystem 1).
//
// Replaces, for one colour class of elements, the reference sequence
//   r[gy, gx]                           (schwarz.py:271, mesh.py:124-139)
//   S_y^T B S_x ./ (lam_y (+) lam_x)    (schwarz.py:217-218)
//   S_y T S_x^T  * W                    (schwarz.py:219-221)
//   * 1/nu_bar                          (schwarz.py:272-273)
//   u += scatter(...)                   (schwarz.py:274, mesh.py:142-150)
// in one launch.  Elements of one colour have disjoint windows, so the
// scatter-add is a plain read-modify-write: deterministic, no atomics.
//
// This is the fallback / blocks-mode path (FastDiagSolver.solve, factors that
// are not even/odd, TMA-incompatible fields); the tiled kernel (smg_fdt.cuh)
// is the production sweep.  Its outer contraction loops are only partially
// unrolled (compiled for every window size m = 2..41, code size matters more).
//
// Work mapping: a CTA owns E elements; their m x m residual windows are
// staged in shared memory.  The four contractions alternate between
// "column" threads (thread = (element, column)) and "row" threads; every
// thread keeps m accumulators in registers and streams its column/row from
// shared memory, so each DFMA takes one smem operand per m FMAs.  The
// factors S_x, S_y live in the kernel-parameter constant bank (one copy per
// launch => per level, no global symbols) and feed DFMA as uniform operands.
#pragma once
#include "smg_common.cuh"

namespace smg {

template <int M>
struct FDArgs {
  const double* __restrict__ src;      // residual field (N_y,N_x), or blocks (nb,M,M)
  double* __restrict__ dst;            // u field (RMW), or output blocks
  const double* __restrict__ inv_nu;   // (n_y,n_x) 1/nu_bar, or nullptr
  const double* __restrict__ dinv;     // (M,M) 1/(lam_y[i]+lam_x[j])
  int p, n_o, N_x, N_y, n_x;
  int x0, xs, xc, y0, ys, yc;          // colour class: ex = x0 + xs*k (k < xc), same in y
  int nb, blocks_mode, apply_weight;
  double Sy[M * M];                    // Sy[k*M+i] = S_y[k, i]
  double Sx[M * M];                    // Sx[j*M+l] = S_x[j, l]
  double wx[M], wy[M];
};

template <int M>
__host__ __device__ constexpr int fd_elems() { return M <= 23 ? 8 : 4; }
template <int M>
__host__ __device__ constexpr int fd_threads() { return ((fd_elems<M>() * M + 31) / 32) * 32; }
template <int M>
__host__ __device__ constexpr size_t fd_smem() { return sizeof(double) * fd_elems<M>() * M * M; }

template <int M>
__global__ void __launch_bounds__(fd_threads<M>())
fd_kernel(const __grid_constant__ FDArgs<M> A) {
  SMG_PDL_ENTRY();
  constexpr int E = fd_elems<M>();
  constexpr int MM = M * M;
  extern __shared__ double sm[];
  const int tid = threadIdx.x;
  const int nel = A.blocks_mode ? A.nb : A.xc * A.yc;
  const int e0 = blockIdx.x * E;

  // ---- gather the windows (periodic wrap) --------------------------------
  for (int idx = tid; idx < E * MM; idx += blockDim.x) {
    const int e = idx / MM, rem = idx - e * MM;
    const int ge = e0 + e;
    double v = 0.0;
    if (ge < nel) {
      if (A.blocks_mode) {
        v = __ldg(A.src + (size_t)ge * MM + rem);
      } else {
        const int i = rem / M, j = rem - i * M;
        const int ky = ge / A.xc, kx = ge - ky * A.xc;
        const int ex = A.x0 + A.xs * kx, ey = A.y0 + A.ys * ky;
        const int gy = wrapi(ey * A.p - A.n_o + i, A.N_y);
        const int gx = wrapi(ex * A.p - A.n_o + j, A.N_x);
        v = __ldg(A.src + (size_t)gy * A.N_x + gx);
      }
    }
    sm[idx] = v;
  }
  __syncthreads();

  const int e = tid / M, c = tid - e * M;
  const bool act = e < E;
  double* B = sm + e * MM;
  double acc[M];

  // ---- stage 1 (columns): T1[i][c] = sum_k S_y[k][i] R[k][c] --------------
  if (act) {
    double x = B[c];
#pragma unroll
    for (int i = 0; i < M; ++i) acc[i] = A.Sy[i] * x;
#pragma unroll 2
    for (int k = 1; k < M; ++k) {
      x = B[k * M + c];
#pragma unroll
      for (int i = 0; i < M; ++i) acc[i] = fma(A.Sy[k * M + i], x, acc[i]);
    }
#pragma unroll
    for (int i = 0; i < M; ++i) B[i * M + c] = acc[i];
  }
  __syncthreads();

  // ---- stage 2 (rows): T2[c][l] = (sum_j T1[c][j] S_x[j][l]) / (lam_y[c]+lam_x[l]) / nu_bar
  if (act) {
    double x = B[c * M];
#pragma unroll
    for (int l = 0; l < M; ++l) acc[l] = A.Sx[l] * x;
#pragma unroll 2
    for (int j = 1; j < M; ++j) {
      x = B[c * M + j];
#pragma unroll
      for (int l = 0; l < M; ++l) acc[l] = fma(A.Sx[j * M + l], x, acc[l]);
    }
    double s = 1.0;
    if (A.inv_nu != nullptr) {
      const int ge = e0 + e;
      if (ge < nel) {
        const int ky = ge / A.xc, kx = ge - ky * A.xc;
        s = __ldg(A.inv_nu + (size_t)(A.y0 + A.ys * ky) * A.n_x + (A.x0 + A.xs * kx));
      }
    }
#pragma unroll
    for (int l = 0; l < M; ++l) B[c * M + l] = acc[l] * __ldg(A.dinv + c * M + l) * s;
  }
  __syncthreads();

  // ---- stage 3 (columns): T3[i][c] = sum_k S_y[i][k] T2[k][c] -------------
  // (column held in registers so S_y is read along its rows: LDCU.128 pairs)
  if (act) {
    double x[M];
#pragma unroll
    for (int k = 0; k < M; ++k) x[k] = B[k * M + c];
#pragma unroll 2
    for (int i = 0; i < M; ++i) {
      double a = A.Sy[i * M] * x[0];
#pragma unroll
      for (int k = 1; k < M; ++k) a = fma(A.Sy[i * M + k], x[k], a);
      B[i * M + c] = a;
    }
  }
  __syncthreads();

  // ---- stage 4 (rows): out[c][j] = W[c][j] * sum_l T3[c][l] S_x[j][l] ----
  if (act) {
    double x[M];
#pragma unroll
    for (int l = 0; l < M; ++l) x[l] = B[c * M + l];
    const double wyc = A.apply_weight ? A.wy[c] : 1.0;
#pragma unroll 2
    for (int j = 0; j < M; ++j) {
      double a = A.Sx[j * M] * x[0];
#pragma unroll
      for (int l = 1; l < M; ++l) a = fma(A.Sx[j * M + l], x[l], a);
      B[c * M + j] = A.apply_weight ? a * (wyc * A.wx[j]) : a;
    }
  }
  __syncthreads();

  // ---- scatter-add (disjoint windows within a colour) ---------------------
  for (int idx = tid; idx < E * MM; idx += blockDim.x) {
    const int ee = idx / MM, rem = idx - ee * MM;
    const int ge = e0 + ee;
    if (ge >= nel) continue;
    if (A.blocks_mode) {
      A.dst[(size_t)ge * MM + rem] = sm[idx];
    } else {
      const int i = rem / M, j = rem - i * M;
      const int ky = ge / A.xc, kx = ge - ky * A.xc;
      const int ex = A.x0 + A.xs * kx, ey = A.y0 + A.ys * ky;
      const int gy = wrapi(ey * A.p - A.n_o + i, A.N_y);
      const int gx = wrapi(ex * A.p - A.n_o + j, A.N_x);
      double* d = A.dst + (size_t)gy * A.N_x + gx;
      *d = *d + sm[idx];
    }
  }
}

// Host-side launch descriptor filled by the ABI layer.
struct FDLaunch {
  const double* src;
  double* dst;
  const double* inv_nu;
  const double* dinv;
  int p, n_o, N_x, N_y, n_x;
  int x0, xs, xc, y0, ys, yc;
  int nb, blocks_mode, apply_weight;
  const double* Sx;  // host m*m
  const double* Sy;
  const double* wx;
  const double* wy;
};

template <int M>
int fd_launch(const FDLaunch& L, cudaStream_t st) {
  static DeviceFlag attr_done;
  if (!attr_done) {
    if (fd_smem<M>() > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(fd_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)fd_smem<M>());
      if (e != cudaSuccess) return cuda_fail(e, "fd_kernel smem attribute");
    }
    attr_done = true;
  }
  FDArgs<M> A;
  A.src = L.src; A.dst = L.dst; A.inv_nu = L.inv_nu; A.dinv = L.dinv;
  A.p = L.p; A.n_o = L.n_o; A.N_x = L.N_x; A.N_y = L.N_y; A.n_x = L.n_x;
  A.x0 = L.x0; A.xs = L.xs; A.xc = L.xc; A.y0 = L.y0; A.ys = L.ys; A.yc = L.yc;
  A.nb = L.nb; A.blocks_mode = L.blocks_mode; A.apply_weight = L.apply_weight;
  for (int i = 0; i < M * M; ++i) { A.Sx[i] = L.Sx[i]; A.Sy[i] = L.Sy[i]; }
  for (int i = 0; i < M; ++i) { A.wx[i] = L.wx[i]; A.wy[i] = L.wy[i]; }
  const int nel = L.blocks_mode ? L.nb : L.xc * L.yc;
  if (nel <= 0) return SMG_OK;
  const int grid = (nel + fd_elems<M>() - 1) / fd_elems<M>();
  launch(fd_kernel<M>, dim3(grid), dim3(fd_threads<M>()), fd_smem<M>(), st, A);
  return check_launch("fd_kernel");
}

using FDLaunchFn = int (*)(const FDLaunch&, cudaStream_t);
FDLaunchFn fd_dispatch(int m);

}  // namespace smg
