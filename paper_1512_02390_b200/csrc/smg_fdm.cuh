// Tiled additive-Schwarz kernel, FP64 tensor-core (DMMA) variant.
//
// Same tiles, pipeline, band fixup and math as smg_fdt.cuh (schwarz.py:215-222
// plus the sweep at :268-275) but the four contractions run on the FP64
// tensor cores with mma.sync.aligned.m8n8k4.f64 (SASS DMMA.8x8x4): dense
// factors (no even/odd split), the batch of lines of all elements in the
// tile stacked along the MMA's N (stages 1, 3) or M (stages 2, 4) dimension,
// factor fragments held in registers for the whole stage and the data
// fragments streamed from shared memory.  Each DMMA does 256 FMAs from
// register operands, so instruction issue -- the limit of the DFMA variant --
// drops ~8x; the price is padding of the m-sized factor dimension to
// multiples of 8 (M) and 4 (K): 1.33x the dense flops at m = 19, 1.18x at 35.
#pragma once
#include <vector>

#include "smg_fdt.cuh"

namespace smg {


template <int P, int NO, int TX, int TY>
struct FDMGeom {
  using T = FDTGeom<P, NO, TX, TY>;
  static constexpr int M = T::M, MM = T::MM, E = T::E;
  static constexpr int MT = (M + 7) / 8;     // 8-row tiles of the factor dimension
  static constexpr int KT = (M + 3) / 4;     // 4-deep k steps
  static constexpr int NL = E * M;           // lines (element, row or column) in a tile
  static constexpr int BT = (NL + 7) / 8;    // 8-line batch tiles
  static constexpr int WARPS = 8, THREADS = 32 * WARPS;
  static constexpr int NFRAG = MT * KT;      // factor fragments per stage and lane
  static constexpr size_t SMEM = T::SMEM + sizeof(double) * 4 * NFRAG * 32;
};

struct FDMArgs {
  const double* __restrict__ r;
  double* __restrict__ u;
  const double* __restrict__ inv_nu;
  const double* __restrict__ dinv;   // (M,M) 1/(lam_y[i] + lam_x[j]), natural order
  const double* __restrict__ Sx;     // (M,M) device copies of the factors
  const double* __restrict__ Sy;
  const double* __restrict__ frag;   // [4 stages][MT*KT][32 lanes] factor fragments in lane order
  double* __restrict__ ws;
  int N_x, N_y, n_x, ntx, nty, u_zero;
  double wx[48], wy[48];
};

template <int P, int NO, int TX, int TY>
__global__ void __launch_bounds__(FDMGeom<P, NO, TX, TY>::THREADS, 2)
fdm_kernel(const __grid_constant__ FDMArgs A) {
  SMG_PDL_ENTRY();
  using G = FDMGeom<P, NO, TX, TY>;
  using GT = FDTGeom<P, NO, TX, TY>;
  constexpr int M = G::M, MM = G::MM, MT = G::MT, KT = G::KT, NL = G::NL, BT = G::BT;
  constexpr int OX = GT::OX, OY = GT::OY, RX = GT::RX, RY = GT::RY, BW = GT::BW, STAGE = GT::STAGE;
  constexpr int NT = G::THREADS, WARPS = G::WARPS, E = G::E;
  extern __shared__ double sm[];
  double* EB = sm + 2 * STAGE;
  double* FR = EB + E * MM;  // [4][NFRAG][32] factor fragments, loaded once per CTA
  constexpr int NFRAG = G::NFRAG;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int N_x = A.N_x, N_y = A.N_y, ntx = A.ntx, ntiles = A.ntx * A.nty;

  for (int idx = tid; idx < 4 * NFRAG * 32; idx += NT) cp_async8(FR + idx, A.frag + idx);
  int tile = blockIdx.x;
  if (tile < ntiles) fdt_prefetch<P, NO, TX, TY, NT>(A.r, A.u, N_x, N_y, ntx, tile, sm, A.u_zero != 0);
  cp_async_commit();
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    double* R = sm + (it & 1) * STAGE;
    double* UO = R + RX * RY;
    {
      const int nxt = tile + gridDim.x;
      if (nxt < ntiles)
        fdt_prefetch<P, NO, TX, TY, NT>(A.r, A.u, N_x, N_y, ntx, nxt, sm + ((it + 1) & 1) * STAGE, A.u_zero != 0);
      cp_async_commit();
    }
    const int tx = tile % ntx, ty = tile / ntx;
    const int X0 = tx * OX, Y0 = ty * OY;
    cp_async_wait<1>();
    __syncthreads();

    // ---- stage 1: T1[i][(e,c)] = sum_k S_y[k][i] R_e[k][c]   (batch along N)
    {
      double a[MT][KT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) a[mt][kt] = FR[(0 * NFRAG + mt * KT + kt) * 32 + lane];
      for (int bt = warp; bt < BT; bt += WARPS) {
        const int n = 8 * bt + g;
        const bool vn = n < NL;
        const int e = vn ? n / M : 0, c = vn ? n - e * M : 0;
        const double* col = R + ((e / TX) * P) * RX + (e % TX) * P + c;
        double acc[MT][2];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const int k = 4 * kt + t;
          const double b = (vn && k < M) ? col[k * RX] : 0.0;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) dmma884(acc[mt][0], acc[mt][1], a[mt][kt], b);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int n2 = 8 * bt + 2 * t + j;
          if (n2 < NL) {
            const int e2 = n2 / M, c2 = n2 - e2 * M;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              const int i = 8 * mt + g;
              if (i < M) EB[e2 * MM + i * M + c2] = acc[mt][j];
            }
          }
        }
      }
    }
    __syncthreads();
    for (int idx = tid; idx < RX * RY; idx += NT) R[idx] = 0.0;  // residual consumed

    // ---- stage 2: T2[(e,i)][l] = (sum_j T1[e][i][j] S_x[j][l]) / (lam_y+lam_x) / nu_bar
    {
      double b[KT][MT];
#pragma unroll
      for (int kt = 0; kt < KT; ++kt)
#pragma unroll
        for (int nt = 0; nt < MT; ++nt) b[kt][nt] = FR[(1 * NFRAG + nt * KT + kt) * 32 + lane];
      for (int bt = warp; bt < BT; bt += WARPS) {
        const int m = 8 * bt + g;
        const bool vm = m < NL;
        const double* row = EB + (vm ? m : 0) * M;  // rows (e,i) are contiguous
        double acc[MT][2];
#pragma unroll
        for (int nt = 0; nt < MT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const int k = 4 * kt + t;
          const double av = (vm && k < M) ? row[k] : 0.0;
#pragma unroll
          for (int nt = 0; nt < MT; ++nt) dmma884(acc[nt][0], acc[nt][1], av, b[kt][nt]);
        }
        __syncwarp();
        if (vm) {
          const int e2 = m / M, i2 = m - e2 * M;
          double s = 1.0;
          if (A.inv_nu != nullptr)
            s = __ldg(A.inv_nu + (size_t)(ty * TY + e2 / TX) * A.n_x + (tx * TX + e2 % TX));
#pragma unroll
          for (int nt = 0; nt < MT; ++nt)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int l = 8 * nt + 2 * t + j;
              if (l < M) EB[m * M + l] = acc[nt][j] * (__ldg(A.dinv + i2 * M + l) * s);
            }
        }
      }
    }
    __syncthreads();

    // ---- stage 3: T3[k][(e,l)] = sum_i S_y[k][i] T2[e][i][l]   (batch along N)
    {
      double a[MT][KT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) a[mt][kt] = FR[(2 * NFRAG + mt * KT + kt) * 32 + lane];
      for (int bt = warp; bt < BT; bt += WARPS) {
        const int n = 8 * bt + g;
        const bool vn = n < NL;
        const int e = vn ? n / M : 0, l = vn ? n - e * M : 0;
        const double* col = EB + e * MM + l;
        double acc[MT][2];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const int i = 4 * kt + t;
          const double bv = (vn && i < M) ? col[i * M] : 0.0;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) dmma884(acc[mt][0], acc[mt][1], a[mt][kt], bv);
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int n2 = 8 * bt + 2 * t + j;
          if (n2 < NL) {
            const int e2 = n2 / M, l2 = n2 - e2 * M;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              const int k = 8 * mt + g;
              if (k < M) EB[e2 * MM + k * M + l2] = acc[mt][j];
            }
          }
        }
      }
    }
    __syncthreads();

    // ---- stage 4: out[(e,k)][j] = W[k][j] sum_l T3[e][k][l] S_x[j][l]   (batch along M)
    {
      double b[KT][MT];
#pragma unroll
      for (int kt = 0; kt < KT; ++kt)
#pragma unroll
        for (int nt = 0; nt < MT; ++nt) b[kt][nt] = FR[(3 * NFRAG + nt * KT + kt) * 32 + lane];
      for (int bt = warp; bt < BT; bt += WARPS) {
        const int m = 8 * bt + g;
        const bool vm = m < NL;
        const double* row = EB + (vm ? m : 0) * M;
        double acc[MT][2];
#pragma unroll
        for (int nt = 0; nt < MT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const int l = 4 * kt + t;
          const double av = (vm && l < M) ? row[l] : 0.0;
#pragma unroll
          for (int nt = 0; nt < MT; ++nt) dmma884(acc[nt][0], acc[nt][1], av, b[kt][nt]);
        }
        __syncwarp();
        if (vm) {
          const double wyk = A.wy[m % M];
#pragma unroll
          for (int nt = 0; nt < MT; ++nt)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int jj = 8 * nt + 2 * t + j;
              if (jj < M) EB[m * M + jj] = acc[nt][j] * (wyk * A.wx[jj]);
            }
        }
      }
    }
    __syncthreads();

    // ---- accumulate element windows into the region, colour passes ---------
    {
      constexpr int C = GT::C;
#pragma unroll
      for (int pass = 0; pass < C * C; ++pass) {
        for (int rr = tid; rr < NL; rr += NT) {
          const int e = rr / M, k = rr - e * M;
          const int exl = e % TX, eyl = e / TX;
          if ((eyl % C) * C + (exl % C) != pass) continue;
          const double* src = EB + rr * M;
          double* dst = R + (eyl * P + k) * RX + exl * P;
#pragma unroll
          for (int j = 0; j < M; ++j) dst[j] += src[j];
        }
        __syncthreads();
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
    __syncthreads();
  }
  cp_async_wait<0>();
  (void)E;
}

// Lane-ordered DMMA fragments of the four contraction stages (host side):
//   stage 0: A = S_y^T  (a = S_y[4kt+t][8mt+g])   stage 1: B = S_x   (b = S_x[4kt+t][8nt+g])
//   stage 2: A = S_y    (a = S_y[8mt+g][4kt+t])   stage 3: B = S_x^T (b = S_x[8nt+g][4kt+t])
inline void fdm_fragments(int m, const double* Sx, const double* Sy, std::vector<double>& out) {
  const int MT = (m + 7) / 8, KT = (m + 3) / 4, NF = MT * KT;
  out.assign((size_t)4 * NF * 32, 0.0);
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    for (int ft = 0; ft < MT; ++ft)
      for (int kt = 0; kt < KT; ++kt) {
        const int f = ft * KT + kt, k = 4 * kt + t, r = 8 * ft + g;
        const bool ok = k < m && r < m;
        out[(0 * NF + f) * 32 + lane] = ok ? Sy[k * m + r] : 0.0;
        out[(1 * NF + f) * 32 + lane] = ok ? Sx[k * m + r] : 0.0;
        out[(2 * NF + f) * 32 + lane] = ok ? Sy[r * m + k] : 0.0;
        out[(3 * NF + f) * 32 + lane] = ok ? Sx[r * m + k] : 0.0;
      }
  }
}

template <int P, int NO, int TX, int TY>
int fdm_launch(const FDTLaunch& L, cudaStream_t st) {
  using G = FDMGeom<P, NO, TX, TY>;
  using GT = FDTGeom<P, NO, TX, TY>;
  static_assert(G::M <= 48, "m too large for the DMMA variant's weight arrays");
  FDMArgs A;
  A.r = L.r; A.u = L.u; A.inv_nu = L.inv_nu; A.dinv = L.dinv_dense; A.Sx = L.Sx_dev; A.Sy = L.Sy_dev;
  A.frag = L.frag_dev;
  A.ws = L.ws; A.N_x = L.N_x; A.N_y = L.N_y; A.n_x = L.n_x; A.ntx = L.ntx; A.nty = L.nty; A.u_zero = L.u_zero;
  for (int i = 0; i < 48; ++i) {
    A.wx[i] = i < G::M ? L.wx[i] : 0.0;
    A.wy[i] = i < G::M ? L.wy[i] : 0.0;
  }
  static int grid_cap = 0;
  if (grid_cap == 0) {
    if (G::SMEM > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(fdm_kernel<P, NO, TX, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)G::SMEM);
      if (e != cudaSuccess) return cuda_fail(e, "fdm_kernel smem attribute");
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fdm_kernel<P, NO, TX, TY>, G::THREADS, G::SMEM);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int ntiles = L.ntx * L.nty;
  launch(fdm_kernel<P, NO, TX, TY>, dim3(ntiles < grid_cap ? ntiles : grid_cap), dim3(G::THREADS), G::SMEM, st, A);
  int rc = check_launch("fdm_kernel");
  if (rc) return rc;
  constexpr long PER = (long)GT::BW * (GT::OY - GT::BW) + (long)(GT::OX - GT::BW) * GT::BW + (long)GT::BW * GT::BW;
  const long nb = PER * ntiles;
  launch(fdm_fixup<P, NO, TX, TY>, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, st, L.u, L.ws, L.N_x, L.N_y,
         L.ntx, L.nty, L.u_zero);
  return check_launch("fdm_fixup");
}

}  // namespace smg
