// Coarse pseudo-inverse by 2D FFT (subsystem a10, coarse="pinv").
//
// The p = 1 periodic operator A_0 = (dy/dx) I (x) T_x + (dx/dy) T_y (x) I,
// T = circulant tridiag(-1, 2, -1), is diagonalised by the 2D DFT with
// eigenvalues lam(ky, kx) = (dy/dx) mu_x(kx) + (dx/dy) mu_y(ky),
// mu(k) = 2 - 2 cos(2 pi k / n).  Its pseudo-inverse (zero mode dropped) --
// what the reference's CG approximates to 1e-12 (multigrid.py:196-228) -- is
//   u = IDFT( DFT(f) / lam ),  u_hat(0, 0) = 0,
// i.e. the dense Q_y (Lp .* (Q_y^T f Q_x)) Q_x^T of smg_coarse_pinv's GEMM
// path in O(n^2 log n) instead of 4 n^3 (n = 512 at C5: 0.6 GFLOP per solve,
// once per coarse PCG iteration).  Power-of-two n_x, n_y (every BASELINE
// coarse level); iterative radix-2 complex FFTs in shared memory.
//   larger than 64 x 64 : rows (forward x) -> columns (y, scale, inverse y)
//                         -> rows (inverse x), three launches through a
//                         complex workspace of n_x n_y entries (the coarse ws)
//   up to 64 x 64       : the dense two-launch path is faster; a one-CTA FFT
//                         kernel is kept behind SMG_PINV_FFT=2.
#include <algorithm>
#include <cmath>
#include <vector>

#include <cooperative_groups.h>

#include "smg_common.cuh"

namespace smg {

constexpr int kFftMax = 1024;

struct FftConsts {
  double twx[kFftMax];   // cos, sin of 2 pi k / n_x, k < n_x / 2 (interleaved)
  double twy[kFftMax];
};

__device__ __forceinline__ int brev(int i, int logn) { return (int)(__brev((unsigned)i) >> (32 - logn)); }

// In-place radix-2 DIT FFTs of `lines` lines of n points (input in
// bit-reversed order, output natural), line l at buf + l*ls, point i at
// + i*ps.  inv: conjugate twiddles.  All threads of the CTA participate; ends
// with a barrier.
__device__ __forceinline__ void fft_lines(double2* buf, int n, int logn, int lines, int ls, int ps,
                                          const double* tw, bool inv) {
  const int nh = n >> 1;
  for (int s = 0; s < logn; ++s) {
    const int half = 1 << s, stride = nh >> s;   // twiddle step: W_n^(pos * n / (2 half))
    for (int b = threadIdx.x; b < lines * nh; b += blockDim.x) {
      const int l = b >> (logn - 1), j = b & (nh - 1);
      const int grp = j >> s, pos = j & (half - 1);
      const int i0 = grp * 2 * half + pos, i1 = i0 + half;
      double2* x = buf + (size_t)l * ls;
      const double c = tw[2 * (pos * stride)], sn = inv ? tw[2 * (pos * stride) + 1] : -tw[2 * (pos * stride) + 1];
      const double2 a = x[(size_t)i0 * ps], bb = x[(size_t)i1 * ps];
      const double tr = bb.x * c - bb.y * sn, ti = bb.x * sn + bb.y * c;
      x[(size_t)i0 * ps] = make_double2(a.x + tr, a.y + ti);
      x[(size_t)i1 * ps] = make_double2(a.x - tr, a.y - ti);
    }
    __syncthreads();
  }
}

// Multi-CTA variant: line-local index i stored at i + i/16 (the bit-reversed
// scatter and the strided butterfly stages hit 16 banks otherwise) and
// stage-major complex twiddles SW[half - 1 + pos] = W^(pos n / (2 half))
// (consecutive threads read consecutive entries).  Same butterflies, same
// twiddle values, same order: bitwise-equal results.
__device__ __forceinline__ int fpad(int i) { return i + (i >> 4); }

__device__ __forceinline__ void fft_lines_p(double2* buf, int n, int logn, int lines, int ls, const double2* SW,
                                            bool inv) {
  const int nh = n >> 1;
  for (int s = 0; s < logn; ++s) {
    const int half = 1 << s;
    for (int b = threadIdx.x; b < lines * nh; b += blockDim.x) {
      const int l = b >> (logn - 1), j = b & (nh - 1);
      const int grp = j >> s, pos = j & (half - 1);
      const int i0 = grp * 2 * half + pos, i1 = i0 + half;
      double2* x = buf + (size_t)l * ls;
      const double2 w = SW[half - 1 + pos];
      const double c = w.x, sn = inv ? w.y : -w.y;
      const double2 a = x[fpad(i0)], bb = x[fpad(i1)];
      const double tr = bb.x * c - bb.y * sn, ti = bb.x * sn + bb.y * c;
      x[fpad(i0)] = make_double2(a.x + tr, a.y + ti);
      x[fpad(i1)] = make_double2(a.x - tr, a.y - ti);
    }
    __syncthreads();
  }
}

// Device table of the multi-CTA path (built once per coarse handle,
// fft_table): stage-major twiddles SWx (n_x - 1 complex), SWy (n_y - 1), then
// mu_x (n_x), mu_y (n_y) -- read coalesced instead of as divergent
// parameter-bank loads.
__device__ __forceinline__ void fft_load_sw(const double* __restrict__ tab, int n, double2* SW) {
  const double2* src = reinterpret_cast<const double2*>(tab);
  for (int e = threadIdx.x; e < n - 1; e += blockDim.x) SW[e] = __ldg(src + e);
}

// mu(k) = 2 - 2 cos(2 pi k / n) from the twiddle table (cos is even in k)
__device__ __forceinline__ double mu_of(int k, int n, const double* tw) {
  const int kk = k <= n / 2 ? k : n - k;
  const double c = kk < n / 2 ? tw[2 * kk] : -1.0;   // k = n/2: cos(pi) = -1
  return 2.0 - 2.0 * c;
}

// ---- one CTA: n_x, n_y <= 64 -------------------------------------------------
__global__ void __launch_bounds__(1024) fft_pinv_small_kernel(int nx, int ny, int lx, int ly, double cx, double cy,
                                                              const __grid_constant__ FftConsts C,
                                                              const double* __restrict__ f, double* __restrict__ u) {
  SMG_PDL_TRIGGER();
  extern __shared__ __align__(16) double2 zs[];
  const int PX = nx + 1;      // padded row pitch: column FFTs are bank-conflict free
  double2* Z = zs;            // ny x PX
  double2* Z2 = zs + ny * PX;
  double* TX = reinterpret_cast<double*>(Z2 + ny * PX);   // twiddles in shared memory: the
  double* TY = TX + nx;                                    // param bank serialises divergent reads
  const int n = nx * ny;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) TX[i] = C.twx[i];
  for (int i = threadIdx.x; i < ny; i += blockDim.x) TY[i] = C.twy[i];
  SMG_PDL_WAIT();   // the twiddles (parameters) are staged while the preceding grid drains
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int y = i >> lx, x = i & (nx - 1);
    Z[y * PX + brev(x, lx)] = make_double2(f[i], 0.0);
  }
  __syncthreads();
  fft_lines(Z, nx, lx, ny, PX, 1, TX, false);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int y = i >> lx, x = i & (nx - 1);
    Z2[brev(y, ly) * PX + x] = Z[y * PX + x];
  }
  __syncthreads();
  fft_lines(Z2, ny, ly, nx, 1, PX, TY, false);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int ky = i >> lx, kx = i & (nx - 1);
    const double lam = cx * mu_of(kx, nx, TX) + cy * mu_of(ky, ny, TY);
    const double s = (ky == 0 && kx == 0) ? 0.0 : 1.0 / lam;
    const double2 z = Z2[ky * PX + kx];
    Z[brev(ky, ly) * PX + kx] = make_double2(z.x * s, z.y * s);
  }
  __syncthreads();
  fft_lines(Z, ny, ly, nx, 1, PX, TY, true);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int y = i >> lx, x = i & (nx - 1);
    Z2[y * PX + brev(x, lx)] = Z[y * PX + x];
  }
  __syncthreads();
  fft_lines(Z2, nx, lx, ny, PX, 1, TX, true);
  const double sc = 1.0 / ((double)nx * ny);
  for (int i = threadIdx.x; i < n; i += blockDim.x) u[i] = Z2[(i >> lx) * PX + (i & (nx - 1))].x * sc;
}

// ---- three launches for larger meshes ------------------------------------------
// `lines` FFT lines per CTA, chosen per launch so that the grid has >= 256
// CTAs (8 lines per CTA gave 64 CTAs at 512^2: 72 us per solve on B200)

// rows [r0, r0+lines): forward (inv = false, real input f) or inverse (inv = true,
// complex input W, real output u) FFT along x
__global__ void __launch_bounds__(512) fft_rows_kernel(int nx, int ny, int lx, const double* __restrict__ tab,
                                                       const double* __restrict__ f, double2* __restrict__ W,
                                                       double* __restrict__ u, int inv, int lines) {
  SMG_PDL_ENTRY();
  extern __shared__ __align__(16) double2 zs[];
  const int ls = fpad(nx);
  double2* SX = zs + lines * ls;
  const int r0 = blockIdx.x * lines, nr = min(lines, ny - r0);
  fft_load_sw(tab, nx, SX);
  for (int i = threadIdx.x; i < nr * nx; i += blockDim.x) {
    const int l = i / nx, x = i - l * nx;
    const size_t g = (size_t)(r0 + l) * nx + x;
    zs[l * ls + fpad(brev(x, lx))] = inv ? W[g] : make_double2(f[g], 0.0);
  }
  __syncthreads();
  fft_lines_p(zs, nx, lx, nr, ls, SX, inv != 0);
  if (!inv) {
    for (int i = threadIdx.x; i < nr * nx; i += blockDim.x) {
      const int l = i / nx, x = i - l * nx;
      W[(size_t)r0 * nx + i] = zs[l * ls + fpad(x)];
    }
  } else {
    const double sc = 1.0 / ((double)nx * ny);
    for (int i = threadIdx.x; i < nr * nx; i += blockDim.x) {
      const int l = i / nx, x = i - l * nx;
      u[(size_t)r0 * nx + i] = zs[l * ls + fpad(x)].x * sc;
    }
  }
}

// columns [c0, c0+8): forward FFT along y, divide by lambda, inverse FFT along y
__global__ void __launch_bounds__(512) fft_cols_kernel(int nx, int ny, int ly, double cx, double cy,
                                                       const double* __restrict__ tab, double2* __restrict__ W,
                                                       int lines) {
  SMG_PDL_ENTRY();
  extern __shared__ __align__(16) double2 zs[];   // lines x fpad(ny) (line = column)
  const int ls = fpad(ny);
  double2* Z2 = zs + lines * ls;
  double2* SY = Z2 + lines * ls;
  double* MY = reinterpret_cast<double*>(SY + ny);
  const double* mux = tab + 2 * (nx - 1) + 2 * (ny - 1);
  for (int i = threadIdx.x; i < ny; i += blockDim.x) MY[i] = __ldg(mux + nx + i);
  fft_load_sw(tab + 2 * (nx - 1), ny, SY);
  const int c0 = blockIdx.x * lines, nc = min(lines, nx - c0);
  for (int i = threadIdx.x; i < nc * ny; i += blockDim.x) {
    const int y = i / nc, l = i - y * nc;
    zs[l * ls + fpad(brev(y, ly))] = W[(size_t)y * nx + c0 + l];
  }
  __syncthreads();
  fft_lines_p(zs, ny, ly, nc, ls, SY, false);
  for (int i = threadIdx.x; i < nc * ny; i += blockDim.x) {
    const int l = i / ny, ky = i - l * ny, kx = c0 + l;
    const double lam = cx * __ldg(mux + kx) + cy * MY[ky];
    const double s = (ky == 0 && kx == 0) ? 0.0 : 1.0 / lam;
    const double2 z = zs[l * ls + fpad(ky)];
    Z2[l * ls + fpad(brev(ky, ly))] = make_double2(z.x * s, z.y * s);
  }
  __syncthreads();
  fft_lines_p(Z2, ny, ly, nc, ls, SY, true);
  for (int i = threadIdx.x; i < nc * ny; i += blockDim.x) {
    const int y = i / nc, l = i - y * nc;
    W[(size_t)y * nx + c0 + l] = Z2[l * ls + fpad(y)];
  }
}

static bool pow2(int n, int* lg) {
  if (n < 2 || (n & (n - 1))) return false;
  int l = 0;
  while ((1 << l) < n) ++l;
  *lg = l;
  return true;
}

// 1 = not applicable (caller falls back to the GEMM path)
// The multi-CTA path's device table (see fft_load_sw), or an empty vector
// when the FFT path does not apply to n_x x n_y.
std::vector<double> fft_table(int nx, int ny) {
  int lx = 0, ly = 0;
  std::vector<double> t;
  if (!pow2(nx, &lx) || !pow2(ny, &ly) || nx > kFftMax || ny > 512) return t;
  const double pi = 3.14159265358979323846;
  auto stage = [&](int n) {
    const int nh = n / 2;
    for (int e = 0; e < n - 1; ++e) {
      int half = 1;
      while (2 * half <= e + 1) half *= 2;
      const int k = (e + 1 - half) * (nh / half);
      t.push_back(std::cos(2.0 * pi * k / n));
      t.push_back(std::sin(2.0 * pi * k / n));
    }
  };
  auto mu = [&](int n) {
    for (int k = 0; k < n; ++k) {
      const int kk = k <= n / 2 ? k : n - k;
      const double c = kk < n / 2 ? std::cos(2.0 * pi * kk / n) : -1.0;
      t.push_back(2.0 - 2.0 * c);
    }
  };
  stage(nx);
  stage(ny);
  mu(nx);
  mu(ny);
  return t;
}

int pinv_fft(int nx, int ny, double dx, double dy, const double* f, double* u, double* ws, const double* tab,
             cudaStream_t st) {
  int lx = 0, ly = 0;
  if (!pow2(nx, &lx) || !pow2(ny, &ly) || nx > kFftMax || ny > 512) return 1;
  // SMG_PINV_FFT: 0 never, 1 (default) beyond 64 x 64, 2 always.  Measured
  // (tools/vcycle_breakdown.py): at 64 x 64 the one-CTA FFT takes 36 us vs
  // 16 us for the two-launch dense path; at C4 (256^2) the MGCG solve drops
  // 0.40 -> 0.10 s, at C5 (512^2, coarse PCG) 1.61 -> 0.98 s.
  static const int mode = env_int("SMG_PINV_FFT", 1);
  if (mode == 0 || (mode == 1 && (long)nx * ny <= 64 * 64)) return 1;
  const double cx = dy / dx, cy = dx / dy;
  if (nx <= 64 && ny <= 64) {
    FftConsts C;
    const double pi = 3.14159265358979323846;
    for (int k = 0; k < kFftMax / 2; ++k) {
      C.twx[2 * k] = k < nx / 2 ? std::cos(2.0 * pi * k / nx) : 0.0;
      C.twx[2 * k + 1] = k < nx / 2 ? std::sin(2.0 * pi * k / nx) : 0.0;
      C.twy[2 * k] = k < ny / 2 ? std::cos(2.0 * pi * k / ny) : 0.0;
      C.twy[2 * k + 1] = k < ny / 2 ? std::sin(2.0 * pi * k / ny) : 0.0;
    }
    const size_t smem = sizeof(double2) * 2 * (size_t)(nx + 1) * ny + sizeof(double) * (nx + ny);
    static DeviceFlag attr;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(fft_pinv_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(sizeof(double2) * 2 * 65 * 64 + sizeof(double) * 128));
      if (e != cudaSuccess) return cuda_fail(e, "fft_pinv_small_kernel smem attribute");
      attr = true;
    }
    launch(fft_pinv_small_kernel, dim3(1), dim3(1024), smem, st, nx, ny, lx, ly, cx, cy, C, f, u);
    return check_launch("fft_pinv_small_kernel");
  }
  if (tab == nullptr) return 1;
  double2* W = reinterpret_cast<double2*>(ws);   // the coarse ws holds 2 nx ny doubles
  auto pick = [](int nlines, int n, int* threads) {
    int lines = 8;
    while (lines > 1 && nlines / lines < env_int("SMG_FFT_MINCTAS", 512)) lines >>= 1;
    const int t = lines * (n / 2);
    *threads = t >= 512 ? 512 : (t < 64 ? 64 : ((t + 31) / 32) * 32);
    return lines;
  };
  int tr = 0, tc = 0;
  const int lr = pick(ny, nx, &tr), lc = pick(nx, ny, &tc);
  const size_t smr = sizeof(double2) * ((size_t)lr * (nx + nx / 16) + nx);
  const size_t smc = sizeof(double2) * (2 * (size_t)lc * (ny + ny / 16) + ny) + sizeof(double) * ny;
  static DeviceInt attr_r, attr_c;   // largest dynamic shared-memory size set so far, per device
  if ((int)smr > attr_r) {
    cudaError_t e = cudaFuncSetAttribute(fft_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr);
    if (e != cudaSuccess) return cuda_fail(e, "fft_rows_kernel smem attribute");
    attr_r = (int)smr;
  }
  if ((int)smc > attr_c) {
    cudaError_t e = cudaFuncSetAttribute(fft_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc);
    if (e != cudaSuccess) return cuda_fail(e, "fft_cols_kernel smem attribute");
    attr_c = (int)smc;
  }
  const int gr = (ny + lr - 1) / lr, gc = (nx + lc - 1) / lc;
  launch(fft_rows_kernel, dim3(gr), dim3(tr), smr, st, nx, ny, lx, tab, f, W, static_cast<double*>(nullptr), 0, lr);
  int rc = check_launch("fft_rows_kernel");
  if (rc) return rc;
  launch(fft_cols_kernel, dim3(gc), dim3(tc), smc, st, nx, ny, ly, cx, cy, tab, W, lc);
  rc = check_launch("fft_cols_kernel");
  if (rc) return rc;
  launch(fft_rows_kernel, dim3(gr), dim3(tr), smr, st, nx, ny, lx, tab, static_cast<const double*>(nullptr), W, u, 1, lr);
  return check_launch("fft_rows_kernel");
}


// ---- coarse PCG iterations as ONE cooperative kernel ------------------------------
// The p = 1 diffusion PCG (smg_coarse_pcg: preconditioner D^-1/2 A_P^+ D^-1/2, A_P^+ by
// 2D FFT) ran ten launches per iteration on vectors of n_x n_y <= 512^2 doubles: ~110 us
// per iteration at C5 for ~10 MB of traffic, all launch latency and serial last-block
// reductions, plus iterations wasted between two host reads of the convergence flag.
// Here G CTAs (one per SM, co-resident) each own n_y / G node rows (and n_x / G spectrum
// columns) and run the whole loop with four grid barriers per iteration:
//   EA  p <- z + beta p on the own rows and one halo row each side (p ping-pongs between
//       two buffers), q = A_0 p on the own rows (A_0 at p = 1 is the 5-point stencil with
//       edge coefficients c (nu_a + nu_b) / 2), partial p.q                   | barrier
//   B   alpha; x += alpha p, r -= alpha q (own rows), partial r.r;
//       rows of r / sqrt(nu) -> forward FFT along x -> W                        | barrier
//   C   convergence test on r.r (same bits in every CTA: a uniform exit);
//       own columns of W: FFT along y, / lambda, inverse FFT along y           | barrier
//   D   own rows of W: inverse FFT along x, z = Re / sqrt(nu); partial r.z     | barrier
// Sums are per-CTA tree reductions followed by a fixed-order sum of the G partials
// that every warp repeats for itself: deterministic, no atomics, no host reads.
// Everything another CTA wrote is read with ld.cg (L1 is not coherent across SMs).
namespace cgx = cooperative_groups;

struct PcgCoop {
  int nx, ny, lx, ly, Lr, Lc, max_iter;
  double cx, cy, tol;
  const double* tab;   // fft_table
  const double* nu;    // nodal diffusivity (n_y x n_x)
  double* x;
  double* r;
  double* P0;          // p on entry
  double* P1;
  double* z;
  double2* W;
  double* part;        // 3 * G partial sums
  double* S;           // S[0] = ||b||^2, S[2] = r.z on entry; S[4] = converged, S[5] = iterations, S[6] = ||r||^2
};

__device__ __forceinline__ double pcgc_block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();   // red is free
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += red[w];
  return s;
}

// fixed-order total of G per-CTA partials (G <= 128): warp 0 reads them (every warp of every
// CTA reading the same 1 KB was 21 % of the kernel's stall samples), the CTA shares the sum
__device__ __forceinline__ double pcgc_total(const double* part, int G, double* red) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = lane + 32 * k < G ? __ldcg(part + lane + 32 * k) : 0.0;
    double t = (v[0] + v[1]) + (v[2] + v[3]);
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

__global__ void __launch_bounds__(512) pcg_coop_kernel(const PcgCoop A) {
  cgx::grid_group grid = cgx::this_grid();
  extern __shared__ __align__(16) double2 zs[];
  const int nx = A.nx, ny = A.ny, Lr = A.Lr, Lc = A.Lc, G = gridDim.x;
  const int lsx = fpad(nx), lsy = fpad(ny);
  const int nz = max(Lr * lsx, 2 * Lc * lsy);
  double2* SX = zs + nz;                       // n_x - 1 stage twiddles
  double2* SY = SX + nx;                       // n_y - 1
  double* MX = reinterpret_cast<double*>(SY + ny);   // mu_x (n_x), mu_y (n_y)
  double* MY = MX + nx;
  double* NU = MY + ny;                        // (Lr + 2) x n_x: rows r0 - 1 .. r0 + Lr of nu
  double* ISN = NU + (Lr + 2) * nx;            // Lr x n_x: 1 / sqrt(nu) on the own rows
  double* PS = ISN + Lr * nx;                  // (Lr + 2) x n_x: p on the own rows and the halo rows
  double* QS = PS + (Lr + 2) * nx;             // Lr x n_x: q on the own rows
  double* red = QS + Lr * nx;                  // 64: warp sums, then the grid total
  const int tid = threadIdx.x, NT = blockDim.x;
  const int r0 = blockIdx.x * Lr, c0 = blockIdx.x * Lc;
  const int own = Lr * nx;

  fft_load_sw(A.tab, nx, SX);
  fft_load_sw(A.tab + 2 * (nx - 1), ny, SY);
  {
    const double* mu = A.tab + 2 * (nx - 1) + 2 * (ny - 1);
    for (int i = tid; i < nx; i += NT) MX[i] = __ldg(mu + i);
    for (int i = tid; i < ny; i += NT) MY[i] = __ldg(mu + nx + i);
  }
  for (int i = tid; i < (Lr + 2) * nx; i += NT) {
    const int l = i / nx, xx = i - l * nx;
    const int gy = (r0 - 1 + l + ny) & (ny - 1);
    NU[i] = __ldg(A.nu + (size_t)gy * nx + xx);
  }
  __syncthreads();
  for (int i = tid; i < own; i += NT) ISN[i] = 1.0 / sqrt(NU[nx + i]);
  const double bb = A.S[0];
  double rz_old = A.S[2];
  const double sc = 1.0 / ((double)nx * ny);
  double* part_pq = A.part;
  double* part_rr = A.part + G;
  double* part_rz = A.part + 2 * G;
  int done_it = 0;
  double rr_last = 0.0;
  // a thread's elements are fixed: i = tid + k NT of the own rows (k < KO) and of the own +
  // halo rows (k < KH); x and r of the own rows stay in registers for the whole solve, and
  // every loop that reads global memory issues all of its loads before using any (the
  // phases are latency-bound: one round trip to L2 each instead of one per element)
  constexpr int KO = 4, KH = 6;   // n_x <= 512, L_r <= 4, 512 threads
  const int nhalo = (Lr + 2) * nx;
  double xr[KO], rv[KO];
#pragma unroll
  for (int k = 0; k < KO; ++k) {
    const int i = tid + k * NT;
    xr[k] = i < own ? A.x[(size_t)r0 * nx + i] : 0.0;
    rv[k] = i < own ? A.r[(size_t)r0 * nx + i] : 0.0;
  }
  __syncthreads();

  for (int it = 0; it < A.max_iter; ++it) {
    const double* Pold = (it & 1) ? A.P1 : A.P0;
    double* Pnew = (it & 1) ? A.P0 : A.P1;
    // ---- EA
    double beta = 0.0;
    if (it > 0) {
      const double rz_new = pcgc_total(part_rz, G, red);
      beta = rz_new / rz_old;
      rz_old = rz_new;
    }
    {
      double po[KH], zv[KH];
#pragma unroll
      for (int k = 0; k < KH; ++k) {
        const int i = tid + k * NT;
        po[k] = zv[k] = 0.0;
        if (i < nhalo) {
          const int l = i / nx, xx = i - l * nx;
          const size_t g = (size_t)((r0 - 1 + l + ny) & (ny - 1)) * nx + xx;
          po[k] = __ldcg(Pold + g);
          if (it > 0) zv[k] = __ldcg(A.z + g);
        }
      }
#pragma unroll
      for (int k = 0; k < KH; ++k) {
        const int i = tid + k * NT;
        if (i < nhalo) {
          const int l = i / nx, xx = i - l * nx;
          const double pn = it > 0 ? __dadd_rn(zv[k], __dmul_rn(beta, po[k])) : po[k];
          PS[i] = pn;
          if (l >= 1 && l <= Lr) Pnew[(size_t)(r0 - 1 + l) * nx + xx] = pn;
        }
      }
    }
    __syncthreads();
    double acc = 0.0;
    double qv[KO];
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int i = tid + k * NT;
      qv[k] = 0.0;
      if (i < own) {
        const int l = i / nx + 1, xx = i & (nx - 1);
        const int xe = (xx + 1) & (nx - 1), xw = (xx - 1 + nx) & (nx - 1);
        const double u = PS[l * nx + xx], v = NU[l * nx + xx];
        const double kE = 0.5 * A.cx * (v + NU[l * nx + xe]), kW = 0.5 * A.cx * (v + NU[l * nx + xw]);
        const double kN = 0.5 * A.cy * (v + NU[(l + 1) * nx + xx]), kS = 0.5 * A.cy * (v + NU[(l - 1) * nx + xx]);
        qv[k] = kE * (u - PS[l * nx + xe]) + kW * (u - PS[l * nx + xw]) + kN * (u - PS[(l + 1) * nx + xx]) +
                kS * (u - PS[(l - 1) * nx + xx]);
        acc = fma(u, qv[k], acc);
      }
    }
    {
      const double s = pcgc_block_sum(acc, red);
      if (tid == 0) part_pq[blockIdx.x] = s;
    }
    grid.sync();
    // ---- B
    const double alpha = rz_old / pcgc_total(part_pq, G, red);
    acc = 0.0;
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int i = tid + k * NT;
      if (i < own) {
        const int l = i / nx, xx = i - l * nx;
        xr[k] = __dadd_rn(xr[k], __dmul_rn(alpha, PS[nx + i]));
        rv[k] = __dsub_rn(rv[k], __dmul_rn(alpha, qv[k]));
        acc = fma(rv[k], rv[k], acc);
        zs[l * lsx + fpad(brev(xx, A.lx))] = make_double2(rv[k] * ISN[i], 0.0);
      }
    }
    {
      const double s = pcgc_block_sum(acc, red);   // its barriers also publish zs
      if (tid == 0) part_rr[blockIdx.x] = s;
    }
    fft_lines_p(zs, nx, A.lx, Lr, lsx, SX, false);
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int i = tid + k * NT;
      if (i < own) {
        const int l = i / nx, xx = i - l * nx;
        A.W[(size_t)(r0 + l) * nx + xx] = zs[l * lsx + fpad(xx)];
      }
    }
    grid.sync();
    // ---- C
    rr_last = pcgc_total(part_rr, G, red);
    if (sqrt(rr_last) <= A.tol * sqrt(bb)) {
      done_it = it + 1;
      break;
    }
    {
      double2* Z2 = zs + Lc * lsy;
      double2 wv[KO];
#pragma unroll
      for (int k = 0; k < KO; ++k) {
        const int i = tid + k * NT;
        if (i < Lc * ny) {
          const int y = i / Lc, l = i - y * Lc;
          wv[k] = __ldcg(A.W + (size_t)y * nx + c0 + l);
        }
      }
#pragma unroll
      for (int k = 0; k < KO; ++k) {
        const int i = tid + k * NT;
        if (i < Lc * ny) {
          const int y = i / Lc, l = i - y * Lc;
          zs[l * lsy + fpad(brev(y, A.ly))] = wv[k];
        }
      }
      __syncthreads();
      fft_lines_p(zs, ny, A.ly, Lc, lsy, SY, false);
      for (int i = tid; i < Lc * ny; i += NT) {
        const int l = i / ny, ky = i - l * ny, kx = c0 + l;
        const double lam = A.cx * MX[kx] + A.cy * MY[ky];
        const double s = (ky == 0 && kx == 0) ? 0.0 : 1.0 / lam;
        const double2 zz = zs[l * lsy + fpad(ky)];
        Z2[l * lsy + fpad(brev(ky, A.ly))] = make_double2(zz.x * s, zz.y * s);
      }
      __syncthreads();
      fft_lines_p(Z2, ny, A.ly, Lc, lsy, SY, true);
      for (int i = tid; i < Lc * ny; i += NT) {
        const int y = i / Lc, l = i - y * Lc;
        A.W[(size_t)y * nx + c0 + l] = Z2[l * lsy + fpad(y)];
      }
    }
    grid.sync();
    // ---- D
    {
      double2 wv[KO];
#pragma unroll
      for (int k = 0; k < KO; ++k) {
        const int i = tid + k * NT;
        if (i < own) wv[k] = __ldcg(A.W + (size_t)r0 * nx + i);
      }
#pragma unroll
      for (int k = 0; k < KO; ++k) {
        const int i = tid + k * NT;
        if (i < own) {
          const int l = i / nx, xx = i - l * nx;
          zs[l * lsx + fpad(brev(xx, A.lx))] = wv[k];
        }
      }
    }
    __syncthreads();
    fft_lines_p(zs, nx, A.lx, Lr, lsx, SX, true);
    acc = 0.0;
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int i = tid + k * NT;
      if (i < own) {
        const int l = i / nx, xx = i - l * nx;
        const double zv = zs[l * lsx + fpad(xx)].x * sc * ISN[i];
        A.z[(size_t)r0 * nx + i] = zv;
        acc = fma(rv[k], zv, acc);
      }
    }
    {
      const double s = pcgc_block_sum(acc, red);
      if (tid == 0) part_rz[blockIdx.x] = s;
    }
    grid.sync();
  }
#pragma unroll
  for (int k = 0; k < KO; ++k) {
    const int i = tid + k * NT;
    if (i < own) {
      A.x[(size_t)r0 * nx + i] = xr[k];
      A.r[(size_t)r0 * nx + i] = rv[k];
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    A.S[6] = rr_last;
    if (done_it) { A.S[4] = 1.0; A.S[5] = (double)done_it; }
  }
}

// 1 = not applicable (the caller keeps its launch-per-step loop)
int pcg_coop(int nx, int ny, double dx, double dy, const double* tab, const double* nu, double* x, double* r,
             double* p0, double* p1, double* z, double* W, double* part, double* S, double tol, int max_iter,
             cudaStream_t st) {
  int lx = 0, ly = 0;
  static const int on = env_int("SMG_PCG_COOP", 1);
  if (!on || tab == nullptr || !pow2(nx, &lx) || !pow2(ny, &ly) || nx > 512 || ny > 512 || nx < 128 || ny < 128) return 1;
  int dev = 0, sms = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return 1;
  int G = 128;
  while (G > sms || G > nx || G > ny) G >>= 1;
  if (G < 32) return 1;
  PcgCoop A;
  A.nx = nx; A.ny = ny; A.lx = lx; A.ly = ly; A.Lr = ny / G; A.Lc = nx / G; A.max_iter = max_iter;
  A.cx = dy / dx; A.cy = dx / dy; A.tol = tol;
  A.tab = tab; A.nu = nu; A.x = x; A.r = r; A.P0 = p0; A.P1 = p1; A.z = z;
  A.W = reinterpret_cast<double2*>(W); A.part = part; A.S = S;
  const int lsx = nx + nx / 16, lsy = ny + ny / 16;
  const int nz = std::max(A.Lr * lsx, 2 * A.Lc * lsy);
  const size_t smem = sizeof(double2) * ((size_t)nz + nx + ny) +
                      sizeof(double) * ((size_t)nx + ny + (size_t)(A.Lr + 2) * nx * 2 + (size_t)A.Lr * nx * 2 + 64);
  static DeviceInt attr;   // per device
  if ((int)smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(pcg_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "pcg_coop_kernel smem attribute");
    attr = (int)smem;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg_coop_kernel, 512, smem);
  if (per_sm < 1) return 1;
  void* args[] = {&A};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)pcg_coop_kernel, dim3(G), dim3(512), args, smem, st);
  if (e != cudaSuccess) return cuda_fail(e, "pcg_coop_kernel");
  return check_launch("pcg_coop_kernel");
}

}  // namespace smg
