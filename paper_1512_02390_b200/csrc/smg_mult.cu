// Multiplicative Schwarz sweep (reference
// MultiplicativeSchwarz.smooth, schwarz.py:293-353).
//
// The reference visits the subdomains in lexicographic (e_y, e_x) order
// (reversed on even-numbered sweeps).  For each subdomain it solves the
// unweighted local FD problem on the CURRENT residual window, adds the
// correction to u and refreshes the residual by the element kernels of the
// 3 x 3 elements around the subdomain (schwarz.py:320-334).  On a periodic
// mesh every subdomain depends on its predecessor (neighbouring windows and
// their residual footprints overlap, and the lexicographic chain wraps), so
// the sweep is a strictly sequential chain of n_x * n_y small dense steps.
// It runs as ONE persistent CTA that walks the chain; each step is
//   (1) residual window -> shared memory,
//   (2) du = S_y[(S_y^T B S_x) ./ (l_y (+) l_x)] S_x^T (/ nu_bar): four
//       contractions in shared memory,
//   (3) u[win] += du, and the element kernels of the touched elements into a
//       (3p+1)^2 region buffer,
//   (4) r -= (sum of the element outputs covering each region node), one
//       read-modify-write per node (for meshes with n < 4 elements per side
//       the region wraps onto itself; there the touched elements are applied
//       one after another, as the reference does).
// u and r live in global memory (L2); accesses are L2-coherent (.cg).
#include "smg_common.cuh"
#include "smg_mult.cuh"

namespace smg {

constexpr int kMsThreads = 1024;


__device__ __forceinline__ int ms_mod(int a, int n) {
  int r = a % n;
  return r < 0 ? r + n : r;
}

// C[i][j] = sum_k A(i,k) B(k,j) over shared-memory operands given as
// (row stride, col stride) pairs -- m x m x m, every thread its outputs.
__device__ __forceinline__ void ms_mm(double* C, const double* A, int ai, int ak, const double* B, int bk, int bj,
                                      int m, const double* scale) {
  for (int idx = threadIdx.x; idx < m * m; idx += kMsThreads) {
    const int i = idx / m, j = idx - i * m;
    double s0 = 0.0, s1 = 0.0;
    int k = 0;
    for (; k + 1 < m; k += 2) {
      s0 = fma(A[i * ai + k * ak], B[k * bk + j * bj], s0);
      s1 = fma(A[i * ai + (k + 1) * ak], B[(k + 1) * bk + j * bj], s1);
    }
    if (k < m) s0 = fma(A[i * ai + k * ak], B[k * bk + j * bj], s0);
    double v = s0 + s1;
    if (scale) v *= scale[idx];
    C[idx] = v;
  }
}

__global__ void __launch_bounds__(kMsThreads, 1) mult_sweep_kernel(const __grid_constant__ MsArgs A) {
  // launched with programmatic stream serialization like every libsmg kernel:
  // wait for the residual launch before reading r (and u)
  SMG_PDL_ENTRY();
  extern __shared__ __align__(16) double sms[];
  const int p = A.p, n_o = A.n_o, m = A.m, n_x = A.n_x, n_y = A.n_y;
  const int NP = p + 1, N_x = n_x * p, N_y = n_y * p, mm = m * m;
  const int RG = 3 * p + 1;          // region: elements e-1..e+1
  const int tid = threadIdx.x;
  double* Sx = sms;
  double* Sy = Sx + mm;
  double* Dv = Sy + mm;
  double* B = Dv + mm;               // window / T2
  double* T = B + mm;                // T1 / T3
  double* DU = T + mm;               // correction
  double* L1 = DU + mm;              // Ly (or D)
  double* L2 = L1 + NP * NP;         // Lx
  double* MY = L2 + NP * NP;
  double* MX = MY + NP;
  double* W = MX + NP;
  double* EO = W + NP;               // 9 x (p+1)^2 element outputs
  double* NW = EO + 9 * NP * NP;     // diffusion: 9 x (p+1)^2 nu*w2
  double* DR = NW + 9 * NP * NP;     // (3p+1)^2 du on the element region (wide meshes)
  __shared__ int TL[20];             // touched elements (tx, ty) x 9, count
  for (int i = tid; i < mm; i += kMsThreads) {
    Sx[i] = A.Sx[i];
    Sy[i] = A.Sy[i];
    Dv[i] = A.dinv[i];
  }
  for (int i = tid; i < NP * NP; i += kMsThreads) {
    L1[i] = A.Ly[i];
    if (!A.diffusion) L2[i] = A.Lx[i];
  }
  for (int i = tid; i < NP; i += kMsThreads) {
    if (!A.diffusion) {
      MY[i] = A.my[i];
      MX[i] = A.mx[i];
    } else {
      W[i] = A.w[i];
    }
  }
  __syncthreads();
  const bool wide = n_x >= 4 && n_y >= 4;   // the 3x3 element region does not wrap onto itself
  const int n_el = n_x * n_y;
  for (int s = 0; s < n_el; ++s) {
    const int e = A.forward ? s : n_el - 1 - s;
    const int ey = e / n_x, ex = e - ey * n_x;
    const int wy0 = ey * p - n_o, wx0 = ex * p - n_o;
    // (1) residual window
    for (int idx = tid; idx < mm; idx += kMsThreads) {
      const int i = idx / m, j = idx - i * m;
      B[idx] = __ldcg(A.r + (size_t)ms_mod(wy0 + i, N_y) * N_x + ms_mod(wx0 + j, N_x));
    }
    __syncthreads();
    // (2) T1 = S_y^T B ; B <- (T1 S_x) .* dinv ; T3 = S_y B ; DU = T3 S_x^T (/ nu_bar)
    ms_mm(T, Sy, 1, m, B, m, 1, m, nullptr);
    __syncthreads();
    ms_mm(B, T, m, 1, Sx, m, 1, m, Dv);
    __syncthreads();
    ms_mm(T, Sy, m, 1, B, m, 1, m, nullptr);
    __syncthreads();
    ms_mm(DU, T, m, 1, Sx, 1, m, m, nullptr);
    __syncthreads();
    if (A.nu_bar != nullptr) {
      const double nb = A.nu_bar[e];
      for (int idx = tid; idx < mm; idx += kMsThreads) DU[idx] /= nb;
      __syncthreads();
    }
    // (3) u[win] += du
    for (int idx = tid; idx < mm; idx += kMsThreads) {
      const int i = idx / m, j = idx - i * m;
      double* up = A.u + (size_t)ms_mod(wy0 + i, N_y) * N_x + ms_mod(wx0 + j, N_x);
      __stcg(up, __ldcg(up) + DU[idx]);
    }
    // the touched elements (deduplicated, as the reference's set) and their
    // du blocks: du at a node = DU at its window position, 0 outside the window
    // (thread 0 builds the list in shared memory; everyone reads it after the
    // barrier below)
    if (tid == 0) {
      int nt = 0;
      for (int dyl = -1; dyl <= 1; ++dyl)
        for (int dxl = -1; dxl <= 1; ++dxl) {
          const int tx = ms_mod(ex + dxl, n_x), ty = ms_mod(ey + dyl, n_y);
          bool dup = false;
          for (int q = 0; q < nt; ++q) dup |= (TL[2 * q] == tx && TL[2 * q + 1] == ty);
          if (!dup) {
            TL[2 * nt] = tx;
            TL[2 * nt + 1] = ty;
            ++nt;
          }
        }
      TL[18] = nt;
    }
    __syncthreads();
    const int nt = TL[18];
    const int* tl = TL;
    auto du_glob = [&](int Y, int X) -> double {   // global node -> du value
      const int iy = ms_mod(Y - wy0, N_y), ix = ms_mod(X - wx0, N_x);
      return (iy < m && ix < m) ? DU[iy * m + ix] : 0.0;
    };
    if (wide) {
      // du on the 3x3 element region (region node (ry, rx) = global
      // (ey p - p + ry, ex p - p + rx); the window starts at p - n_o)
      for (int idx = tid; idx < RG * RG; idx += kMsThreads) {
        const int ry = idx / RG, rx = idx - ry * RG;
        const int iy = ry - (p - n_o), ix = rx - (p - n_o);
        DR[idx] = (iy >= 0 && iy < m && ix >= 0 && ix < m) ? DU[iy * m + ix] : 0.0;
      }
      __syncthreads();
    }
    // du at local node (a, k) of touched element q
    auto du_at = [&](int q, int a, int k) -> double {
      if (wide) return DR[((q / 3) * p + a) * RG + (q % 3) * p + k];
      return du_glob(tl[2 * q + 1] * p + a, tl[2 * q] * p + k);
    };
    // element kernel of touched element q at local node (a, b)
    auto ekernel = [&](int q, int a, int b) -> double {
      if (!A.diffusion) {
        // mass_y[a] (block @ stiff_x)[a][b] + (stiff_y @ block)[a][b] mass_x[b]
        double sx = 0.0, sy = 0.0;
        for (int k = 0; k < NP; ++k) {
          sx = fma(du_at(q, a, k), L2[k * NP + b], sx);
          sy = fma(L1[a * NP + k], du_at(q, k, b), sy);
        }
        return MY[a] * sx + sy * MX[b];
      }
      return 0.0;  // diffusion: two-stage, see below
    };
    if (A.diffusion) {
      // cx ((nw .* (block D^T)) D) + cy (D^T (nw .* (D block))): stage the
      // inner products G1 = nw .* (block D^T), G2 = nw .* (D block) in EO/NW
      for (int idx = tid; idx < nt * NP * NP; idx += kMsThreads) {
        const int q = idx / (NP * NP), r2 = idx - q * NP * NP, a = r2 / NP, j = r2 - a * NP;
        const int Y0 = tl[2 * q + 1] * p, X0 = tl[2 * q] * p;
        double g1 = 0.0, g2 = 0.0;
        for (int k = 0; k < NP; ++k) {
          g1 = fma(du_at(q, a, k), L1[j * NP + k], g1);   // (block D^T)[a][j] = sum_k B[a][k] D[j][k]
          g2 = fma(L1[a * NP + k], du_at(q, k, j), g2);   // (D block)[a][j] = sum_k D[a][k] B[k][j]
        }
        const double nwv = A.nu[(size_t)ms_mod(Y0 + a, N_y) * N_x + ms_mod(X0 + j, N_x)] * (W[a] * W[j]);
        EO[idx] = nwv * g1;
        NW[idx] = nwv * g2;
      }
      __syncthreads();
    }
    auto eout = [&](int q, int a, int b) -> double {
      if (!A.diffusion) return ekernel(q, a, b);
      const double* G1 = EO + q * NP * NP;
      const double* G2 = NW + q * NP * NP;
      double s1 = 0.0, s2 = 0.0;
      for (int k = 0; k < NP; ++k) {
        s1 = fma(G1[a * NP + k], L1[k * NP + b], s1);   // (G1 @ D)[a][b]
        s2 = fma(L1[k * NP + a], G2[k * NP + b], s2);   // (D^T @ G2)[a][b]
      }
      return A.cx * s1 + A.cy * s2;
    };
    if (wide) {
      // (4a) the nine element outputs into shared memory (EO; diffusion reads
      //      its staged G1/G2 from EO/NW, so write to DU-free scratch RO)
      double* RO = DR + RG * RG;
      for (int idx = tid; idx < 9 * NP * NP; idx += kMsThreads) {
        const int q = idx / (NP * NP), r2 = idx - q * NP * NP, a = r2 / NP, b = r2 - a * NP;
        RO[idx] = eout(q, a, b);
      }
      __syncthreads();
      // (4b) every region node: subtract the outputs of the elements containing
      //      it (fixed order: element rows, then columns), one RMW per node
      const int ry0 = ey * p - p, rx0 = ex * p - p;
      for (int idx = tid; idx < RG * RG; idx += kMsThreads) {
        const int ry = idx / RG, rx = idx - ry * RG;
        const int by = ry / p, bx = rx / p;          // block of the node (0..3)
        const int ay = ry - by * p, ax = rx - bx * p;
        double acc = 0.0;
        // element rows containing row ry: block by (local a = ay) and, when
        // ay == 0, block by-1 (local a = p); the same for columns
#pragma unroll
        for (int t = 1; t >= 0; --t) {
          const int ey_ = by - t, a = ay + t * p;
          if (ey_ < 0 || ey_ > 2 || (t == 1 && ay != 0)) continue;
#pragma unroll
          for (int u_ = 1; u_ >= 0; --u_) {
            const int ex_ = bx - u_, b = ax + u_ * p;
            if (ex_ < 0 || ex_ > 2 || (u_ == 1 && ax != 0)) continue;
            acc += RO[(ey_ * 3 + ex_) * NP * NP + a * NP + b];
          }
        }
        double* rp = A.r + (size_t)ms_mod(ry0 + ry, N_y) * N_x + ms_mod(rx0 + rx, N_x);
        __stcg(rp, __ldcg(rp) - acc);
      }
    } else {
      for (int q = 0; q < nt; ++q) {
        for (int idx = tid; idx < NP * NP; idx += kMsThreads) {
          const int a = idx / NP, b = idx - a * NP;
          double* rp = A.r + (size_t)ms_mod(tl[2 * q + 1] * p + a, N_y) * N_x + ms_mod(tl[2 * q] * p + b, N_x);
          __stcg(rp, __ldcg(rp) - eout(q, a, b));
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
}

size_t mult_smem_bytes(int p, int m) {
  const size_t NP = p + 1;
  return sizeof(double) * (6 * (size_t)m * m + 2 * NP * NP + 3 * NP + 27 * NP * NP + (3 * NP - 2) * (3 * NP - 2)) + 16;
}

int mult_sweep_launch(const MsArgs& A, cudaStream_t st) {
  const size_t smem = mult_smem_bytes(A.p, A.m);
  if (A.p + 1 > kMsMaxNP || smem > 227 * 1024) { set_error("multiplicative sweep: p=%d, m=%d needs too much shared memory", A.p, A.m); return SMG_EUNSUPPORTED; }
  cudaError_t e = cudaFuncSetAttribute(mult_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_fail(e, "mult_sweep_kernel smem attribute");
  launch(mult_sweep_kernel, dim3(1), dim3(kMsThreads), smem, st, A);
  return check_launch("mult_sweep_kernel");
}

}  // namespace smg
