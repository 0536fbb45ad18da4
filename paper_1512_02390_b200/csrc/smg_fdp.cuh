// Paired-line tiled additive-Schwarz kernel (subsystem 1, second engine).
//
// Same math, tiling, ring workspace and fixup pass as the even/odd tiled
// kernel in smg_fdt.cuh (schwarz.py:215-222, 268-275; mesh.py:124-150).  What
// changes is how the four contractions move data through shared memory: ncu
// put fdt_kernel's busiest unit at the shared-memory pipe (74 % at p = 16,
// FP64 pipe 39 %, DRAM 27 %): every half-line thread reads its whole line,
// so each stage reads every staged value twice and writes it once, and the
// 128 B/clk/SM crossbar -- not the DFMA pipe or HBM -- bounds the kernel.
//
//   * A thread owns a MIRRORED PAIR of lines (c, m-1-c) of one element and
//     one parity (warp-uniform).  Stage 1 folds its two box columns in y AND
//     in x before the contraction (a = s_c + s_{m-1-c}, d = s_c - s_{m-1-c}),
//     so what it writes is already the x-folded input of stage 2: stages 2-4
//     read each staged value ONCE (half the loads of fdt_kernel) and every
//     factor entry feeds two accumulators (half the uniform-factor loads).
//   * Stages 2-4 work in place on cells only their thread reads: rows (q,
//     HE+q) or columns (c, HE+c) of the [even | odd] storage order.  By
//     linearity stage 4 runs on the even-y and odd-y half rows and unfolds y
//     on its outputs (row q <- g_q + g_{HE+q}, row HE+q <- g_q - g_{HE+q}:
//     physical row m-1-q lives at storage row HE+q from then on).
//   * One buffer per CTA: the TMA box of the residual region is read by stage
//     1 into registers, then the element windows overwrite it.  u is updated
//     in place in global memory by the gather (coalesced 512-byte rows).  The
//     small footprint (49 KB at p = 16 for a 4x4-element tile) keeps 3 CTAs
//     per SM resident; the other CTAs cover a tile's TMA wait.
//   * Stages 2-4 map lanes to ELEMENTS (element stride odd): every shared
//     memory access of a half-warp hits 16 distinct banks.
#pragma once
#include <cstring>

#include "smg_fdt.cuh"

namespace smg {

// Kernel arguments: as FDTArgs, with every factor row padded to an even
// length and 16-byte aligned so that a uniform load brings two entries
// (LDCU.128: one factor load per four DFMAs with two lines per thread).
constexpr int fdp_pad(int h) { return (h + 1) & ~1; }
template <int M>
struct FDPArgs {
  static constexpr int HE = fdt_he(M), HO = fdt_ho(M), HEP = fdp_pad(HE), HOP = fdp_pad(HO > 0 ? HO : 1);
  CUtensorMap rmap;                   // residual (N_y, N_x), box (BRX, RY)
  CUtensorMap umap;                   // u (N_y, N_x), box (OX, OY): L2 prefetch only
  const double* __restrict__ r;
  double* __restrict__ u;
  const double* __restrict__ inv_nu;  // (n_y, n_x) or nullptr
  const double* __restrict__ dinv;    // (M,M), [even | odd] eigen order in both dims
  double* __restrict__ ws;            // ring workspace: ntiles * NRING
  int N_x, N_y, n_x, ntx, nty;
  int u_zero;
  // analysis factors S[k][i] (row k padded), synthesis factors ST[i][k] times the weight w[k]
  alignas(16) double Sye[HE * HEP];
  alignas(16) double SyeT[HE * HEP];
  alignas(16) double Sxe[HE * HEP];
  alignas(16) double SxeT[HE * HEP];
  alignas(16) double Syo[(HO > 0 ? HO : 1) * HOP];
  alignas(16) double SyoT[(HO > 0 ? HO : 1) * HOP];
  alignas(16) double Sxo[(HO > 0 ? HO : 1) * HOP];
  alignas(16) double SxoT[(HO > 0 ? HO : 1) * HOP];
};

template <int P, int NO, int TX, int TY>
struct FDPK {
  using G = FDTGeom<P, NO, TX, TY>;
  static constexpr int M = G::M, MM = G::MM, HE = G::HE, HO = G::HO, E = G::E;
  static constexpr bool CEN = (M & 1) != 0;   // odd m: the centre line is a single-line role
  static constexpr int NR = E * HE;           // pair roles per parity
  static constexpr int NH = ((NR + 31) / 32) * 32;
  static constexpr int NT = 2 * NH;
  // stages 2-4 map lanes to elements first: a half-warp holds EL elements x LP
  // consecutive lines.  With the window pitch m odd and the element stride
  // ES = LP (mod 2 LP) its 16 accesses fall into 16 distinct 8-byte banks, in
  // the row stages (line offset p m) and the column stages (line offset p)
  static_assert((E & (E - 1)) == 0, "elements per tile must be a power of two");
  static constexpr int EL = E >= 16 ? 16 : E, LP = 16 / EL;
  static constexpr int es_for(int mm) {
    int x = mm;
    while (x % (2 * LP) != LP % (2 * LP)) ++x;
    return x;
  }
  static constexpr int ES = es_for(MM);       // element stride (doubles)
  static constexpr int UB = E * ES > G::RBOX ? E * ES : G::RBOX;
  static constexpr int USZ = (UB + 15) & ~15;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)USZ + MM) + 16;
  static constexpr int by_smem = (int)((227 * 1024) / (SMEM + 1024));
  static constexpr int REGS = 4 * HE + 24 < 64 ? 64 : ((4 * HE + 24 + 7) / 8) * 8;   // two lines of HE accumulators + addressing
  // (two CTAs of 14 full warps at p = 24, 4x4 elements, need 72 registers: allow the cap)
  static constexpr int by_regs = (65536 / (NT * REGS) < 2 && 65536 / (NT * 72) >= 2) ? 2 : 65536 / (NT * REGS);
#ifdef SMG_FDP_MINB
  static constexpr int MINB = SMG_FDP_MINB;   // tuning aid
#else
  static constexpr int MINB = by_smem < 1 ? 1 : (by_smem < by_regs ? by_smem : (by_regs < 1 ? 1 : by_regs));
#endif
  // storage row of physical window row y after stage 4
  __host__ __device__ static constexpr int ry(int y) { return y < HE ? y : HE + (M - 1 - y); }
};

// out1[j], out2[j] = sum_l F[l*H + j] * in{1,2}(l): two lines share every factor entry.
// The l loop stays a loop (the j loop is unrolled: accumulators in registers): the
// fully unrolled kernel was 100 KB of code at p = 32 and ncu's top stall was
// instruction fetch (no_instruction 3.7 warps per issue at p = 32, 1.05 at p = 16).
// Measured on B200 at 256^2 elements (tools/gpu/r2_pair_unr.sh, us per correction, unroll
// 1 / 2 / 3 / 4 / full): p = 8: 66.5 62.5 62.3 60.4 62.5; p = 12: 115.6 111.6 109.6 109.6
// 117.8; p = 16: 191.4 183.3 181.0 185.3 175.0; p = 24: 453.9 441.4 478.1 523.3 513.1;
// p = 32: 1055.8 1204.3 1472.6 1298.4 1303.6.
#ifdef SMG_FDP_UNR
__host__ __device__ constexpr int fdp_unroll(int) { return SMG_FDP_UNR; }   // tuning aid
#else
__host__ __device__ constexpr int fdp_unroll(int H) { return H >= 16 ? 1 : H >= 12 ? 2 : H >= 9 ? H : 4; }
#endif
template <int H, int HP, class In1, class In2>
__device__ __forceinline__ void fdp_contract2(const double* __restrict__ F, In1 in1, In2 in2, double (&o1)[H],
                                              double (&o2)[H]) {
#pragma unroll
  for (int j = 0; j < H; ++j) o1[j] = o2[j] = 0.0;
  constexpr int UNR = fdp_unroll(H);
  // the next step's inputs are loaded before this step's FMAs (a rolled loop is not
  // software-pipelined by the compiler: short-scoreboard stalls at the loop top)
  double x1 = in1(0), x2 = in2(0);
#pragma unroll UNR
  for (int l = 0; l < H; ++l) {
    const double2* __restrict__ F2 = reinterpret_cast<const double2*>(F + l * HP);   // 16-byte aligned rows
    const int ln = l + 1 < H ? l + 1 : l;
    const double n1 = in1(ln), n2 = in2(ln);
#pragma unroll
    for (int j = 0; j < H; j += 2) {
      const double2 fj = F2[j / 2];
      o1[j] = fma(fj.x, x1, o1[j]);
      o2[j] = fma(fj.x, x2, o2[j]);
      if (j + 1 < H) {
        o1[j + 1] = fma(fj.y, x1, o1[j + 1]);
        o2[j + 1] = fma(fj.y, x2, o2[j + 1]);
      }
    }
    x1 = n1;
    x2 = n2;
  }
}

template <int P, int NO, int TX, int TY>
__global__ void __launch_bounds__(FDPK<P, NO, TX, TY>::NT, FDPK<P, NO, TX, TY>::MINB)
fdp_kernel(const __grid_constant__ FDPArgs<P + 1 + 2 * NO> A) {
  SMG_PDL_TRIGGER();
  using G = FDTGeom<P, NO, TX, TY>;
  using K = FDPK<P, NO, TX, TY>;
  constexpr int M = G::M, MM = G::MM, E = G::E, OX = G::OX, OY = G::OY, RX = G::RX, RY = G::RY;
  constexpr int HE = G::HE, HO = G::HO, HOX = G::HOX, BRX = G::BRX, NRING = G::NRING;
  constexpr int NT = K::NT, NH = K::NH, NR = K::NR, ES = K::ES;
  constexpr bool CEN = K::CEN;
  constexpr int HEP = fdp_pad(HE), HOP = fdp_pad(HOX);
  static_assert(K::SMEM <= 227 * 1024, "tile does not fit in shared memory");
  extern __shared__ __align__(1024) double sm[];
  double* U = sm;                  // residual box (row pitch BRX), then E element windows (stride ES, pitch M)
  double* SD = sm + K::USZ;        // 1/(lam_y + lam_x), [even | odd] order in both dimensions
  uint64_t* bar = reinterpret_cast<uint64_t*>(SD + MM);
  const double* FSye = A.Sye;
  const double* FSyeT = A.SyeT;
  const double* FSxe = A.Sxe;
  const double* FSxeT = A.SxeT;
  const double* FSyo = A.Syo;
  const double* FSyoT = A.SyoT;
  const double* FSxo = A.Sxo;
  const double* FSxoT = A.SxoT;
  const int tid = threadIdx.x;
  const int N_x = A.N_x, N_y = A.N_y, ntx = A.ntx, nty = A.nty, ntiles = ntx * nty;
  const bool u_zero = A.u_zero != 0;

  const bool odd = tid >= NH;      // warp-uniform parity
  const int role = odd ? tid - NH : tid;
  const bool act = role < NR;
  const int rr = act ? role : 0;
  // stage 1 reads the box: lanes walk the window columns of one element
  const int e1 = rr / HE, p1 = rr - e1 * HE;
  const bool sg1 = CEN && p1 == HO;
  // stages 2-4 work on the element windows: lanes walk the elements first
  // (bank-conflict-free, see FDPK::ES)
  const int e2 = rr % E, p2 = rr / E;
  const bool sg2 = CEN && p2 == HO;
  double* B = U + e2 * ES;
  const int q2 = sg2 ? p2 : HE + p2;   // second line of the pair (the single role repeats its line; never stored)

  if (tid == 0) {
    if (smem_u32(sm) & 127) __trap();
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  for (int idx = tid; idx < MM; idx += NT) SD[idx] = A.dinv[idx];
  __syncthreads();
  SMG_PDL_WAIT();

  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int tx = tile % ntx, ty = tile / ntx;
    const int X0 = tx * OX, Y0 = ty * OY;
    const bool seam = tx == 0 || ty == 0 || tx == ntx - 1 || ty == nty - 1;
    const int shift = fdt_box_shift(X0, NO);
    // ---- residual box -> U (every thread is past the previous tile's reads of U)
    if (tid == 0) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(bar, seam ? 0u : (unsigned)(G::RBOX * 8));
      if (!seam) tma_load_2d(U, &A.rmap, (X0 - NO) & ~1, Y0 - NO, bar);
      // L2 prefetch: this tile's block of u (read by the gather) and the next tile's box
      if (!u_zero) tma_prefetch_2d(&A.umap, X0, Y0);
      const int nxt = tile + gridDim.x;
      if (nxt < ntiles) {
        const int nx = nxt % ntx, ny = nxt / ntx;
        if (!(nx == 0 || ny == 0 || nx == ntx - 1 || ny == nty - 1))
          tma_prefetch_2d(&A.rmap, (nx * OX - NO) & ~1, ny * OY - NO);
      }
    }
    if (seam) {
      fdt_region_cpasync<P, NO, TX, TY, NT>(A.r, N_x, N_y, X0, Y0, U + shift);
      cp_async_commit();
      cp_async_wait<0>();
    }
    double s = 1.0;   // 1 / nu_bar of this thread's stage-2 element
    if (A.inv_nu != nullptr) s = __ldg(A.inv_nu + (size_t)(ty * TY + e2 / TX) * A.n_x + (tx * TX + e2 % TX));
    mbar_wait(bar, (unsigned)it & 1u);
    if (seam) __syncthreads();   // the cp.async pieces of the other threads

    // ---- stage 1 (box columns c, m-1-c): y-fold by parity, x-fold of the pair, then
    //      [tA; tD][i] = sum_k S[k][i] (a_k; d_k); results stay in registers until
    //      every thread has read the box
    double tA[HE], tD[HE];
    {
      constexpr int UNR1 = fdp_unroll(HE);
      const int exl = e1 % TX, eyl = e1 / TX;
      const double* c1 = U + shift + (eyl * P) * BRX + exl * P + p1;
      const double* c2 = U + shift + (eyl * P) * BRX + exl * P + (M - 1 - p1);
      // one step = the four box values of rows k and m-1-k in the two columns; the next
      // step's values are loaded before this step's FMAs (software pipelining by hand)
      double v1a = c1[0], v1b = c1[(M - 1) * BRX], v2a = c2[0], v2b = c2[(M - 1) * BRX];
      if (!odd) {
#pragma unroll
        for (int i = 0; i < HE; ++i) tA[i] = tD[i] = 0.0;
#pragma unroll UNR1
        for (int k = 0; k < HO; ++k) {
          const int kn = k + 1 < HO ? k + 1 : k;
          const double n1a = c1[kn * BRX], n1b = c1[(M - 1 - kn) * BRX];
          const double n2a = c2[kn * BRX], n2b = c2[(M - 1 - kn) * BRX];
          const double s1 = v1a + v1b;
          double s2 = v2a + v2b;
          if (sg1) s2 = 0.0;
          const double a = s1 + s2, d = s1 - s2;
          const double2* __restrict__ F2 = reinterpret_cast<const double2*>(FSye + k * HEP);
#pragma unroll
          for (int i = 0; i < HE; i += 2) {
            const double2 fi = F2[i / 2];
            tA[i] = fma(fi.x, a, tA[i]);
            tD[i] = fma(fi.x, d, tD[i]);
            if (i + 1 < HE) {
              tA[i + 1] = fma(fi.y, a, tA[i + 1]);
              tD[i + 1] = fma(fi.y, d, tD[i + 1]);
            }
          }
          v1a = n1a; v1b = n1b; v2a = n2a; v2b = n2b;
        }
        if (CEN) {   // centre row of the window
          const double s1 = c1[HO * BRX];
          double s2 = c2[HO * BRX];
          if (sg1) s2 = 0.0;
          const double a = s1 + s2, d = s1 - s2;
#pragma unroll
          for (int i = 0; i < HE; ++i) {
            tA[i] = fma(FSye[HO * HEP + i], a, tA[i]);
            tD[i] = fma(FSye[HO * HEP + i], d, tD[i]);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < HO; ++i) tA[i] = tD[i] = 0.0;
#pragma unroll UNR1
        for (int k = 0; k < HO; ++k) {
          const int kn = k + 1 < HO ? k + 1 : k;
          const double n1a = c1[kn * BRX], n1b = c1[(M - 1 - kn) * BRX];
          const double n2a = c2[kn * BRX], n2b = c2[(M - 1 - kn) * BRX];
          const double s1 = v1a - v1b;
          double s2 = v2a - v2b;
          if (sg1) s2 = 0.0;
          const double a = s1 + s2, d = s1 - s2;
          const double2* __restrict__ F2 = reinterpret_cast<const double2*>(FSyo + k * HOP);
#pragma unroll
          for (int i = 0; i < HO; i += 2) {
            const double2 fi = F2[i / 2];
            tA[i] = fma(fi.x, a, tA[i]);
            tD[i] = fma(fi.x, d, tD[i]);
            if (i + 1 < HO) {
              tA[i + 1] = fma(fi.y, a, tA[i + 1]);
              tD[i + 1] = fma(fi.y, d, tD[i + 1]);
            }
          }
          v1a = n1a; v1b = n1b; v2a = n2a; v2b = n2b;
        }
      }
    }
    __syncthreads();   // the box is consumed
    if (act) {
      double* W = U + e1 * ES + (odd ? HE * M : 0);
      if (!odd) {
#pragma unroll
        for (int i = 0; i < HE; ++i) {
          W[i * M + p1] = tA[i];
          if (!sg1) W[i * M + HE + p1] = tD[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < HO; ++i) {
          W[i * M + p1] = tA[i];
          if (!sg1) W[i * M + HE + p1] = tD[i];
        }
      }
    }
    __syncthreads();

    // ---- stage 2 (storage rows p2, HE+p2; x parity = this warp's): in place,
    //      T2[r][j] = (sum_l Sx[l][j] F1[r][l]) / (lam_y[r] + lam_x[j]) / nu_bar
    if (act) {
      double* r1 = B + p2 * M + (odd ? HE : 0);
      double* r2 = B + q2 * M + (odd ? HE : 0);
      const double* d1 = SD + p2 * M + (odd ? HE : 0);
      const double* d2 = SD + q2 * M + (odd ? HE : 0);
      if (!odd) {
        double t1[HE], t2[HE];
        fdp_contract2<HE, HEP>(FSxe, [&](int l) { return r1[l]; }, [&](int l) { return r2[l]; }, t1, t2);
#pragma unroll
        for (int j = 0; j < HE; ++j) {
          r1[j] = t1[j] * (d1[j] * s);
          if (!sg2) r2[j] = t2[j] * (d2[j] * s);
        }
      } else {
        double t1[HOX], t2[HOX];
        fdp_contract2<HOX, HOP>(FSxo, [&](int l) { return r1[l]; }, [&](int l) { return r2[l]; }, t1, t2);
#pragma unroll
        for (int j = 0; j < HO; ++j) {
          r1[j] = t1[j] * (d1[j] * s);
          if (!sg2) r2[j] = t2[j] * (d2[j] * s);
        }
      }
    }
    __syncthreads();

    // ---- stage 3 (storage columns p2, HE+p2; y parity = this warp's): in place,
    //      e[k] = sum_i SyeT[i][k] T2[i][c] (rows [0,HE)), o[k] from the rows [HE, m)
    if (act) {
      double* c1 = B + p2 + (odd ? HE * M : 0);
      double* c2 = B + q2 + (odd ? HE * M : 0);
      if (!odd) {
        double o1[HE], o2[HE];
        fdp_contract2<HE, HEP>(FSyeT, [&](int i) { return c1[i * M]; }, [&](int i) { return c2[i * M]; }, o1, o2);
#pragma unroll
        for (int k = 0; k < HE; ++k) {
          c1[k * M] = o1[k];
          if (!sg2) c2[k * M] = o2[k];
        }
      } else {
        double o1[HOX], o2[HOX];
        fdp_contract2<HOX, HOP>(FSyoT, [&](int i) { return c1[i * M]; }, [&](int i) { return c2[i * M]; }, o1, o2);
#pragma unroll
        for (int k = 0; k < HO; ++k) {
          c1[k * M] = o1[k];
          if (!sg2) c2[k * M] = o2[k];
        }
      }
    }
    __syncthreads();

    // ---- stage 4 (storage rows p2 = e-row k, HE+p2 = o-row k): x synthesis of both
    //      half rows, y unfold on the outputs: row k <- g_e + g_o, row HE+k <- g_e - g_o
    //      (= physical row m-1-k)
    if (act) {
      double* r1 = B + p2 * M + (odd ? HE : 0);
      double* r2 = B + q2 * M + (odd ? HE : 0);
      if (!odd) {
        double g1[HE], g2[HE];
        fdp_contract2<HE, HEP>(FSxeT, [&](int j) { return r1[j]; }, [&](int j) { return r2[j]; }, g1, g2);
#pragma unroll
        for (int l = 0; l < HE; ++l) {
          if (sg2) {
            r1[l] = g1[l];
          } else {
            r1[l] = g1[l] + g2[l];
            r2[l] = g1[l] - g2[l];
          }
        }
      } else {
        double g1[HOX], g2[HOX];
        fdp_contract2<HOX, HOP>(FSxoT, [&](int j) { return r1[j]; }, [&](int j) { return r2[j]; }, g1, g2);
#pragma unroll
        for (int l = 0; l < HO; ++l) {
          if (sg2) {
            r1[l] = g1[l];
          } else {
            r1[l] = g1[l] + g2[l];
            r2[l] = g1[l] - g2[l];
          }
        }
      }
    }
    __syncthreads();

    // ---- x unfold of every storage row (out[l] = ex[l] + ox[l], out[m-1-l] = ex[l] - ox[l];
    //      centre of odd m: ex) fused with the x fold of the overlaps: the row's home
    //      cells P..P+NO-1 take the right neighbour's cells 0..NO-1, its home cells
    //      NO..2NO the left neighbour's cells P+NO..P+2NO, both unfolded on the fly
    //      from the neighbours' half-form rows; every read precedes every write
    {
      const int w = tid;                 // E*M <= NT: one storage row per thread
      const bool on = w < E * M;
      const int e = on ? w % E : 0, row = on ? w / E : 0, exl = e % TX;
      double* br = U + e * ES + row * M;
      double out[M];
      {
        double ev[HE], ov[HOX];
#pragma unroll
        for (int j = 0; j < HE; ++j) ev[j] = br[j];
#pragma unroll
        for (int j = 0; j < HO; ++j) ov[j] = br[HE + j];
#pragma unroll
        for (int j = 0; j < HO; ++j) {
          out[j] = ev[j] + ov[j];
          out[M - 1 - j] = ev[j] - ov[j];
        }
        if (CEN) out[HO] = ev[HO];
      }
      if (exl + 1 < TX) {
#pragma unroll
        for (int k = 0; k < NO; ++k) out[P + k] += br[ES + k] + br[ES + HE + k];
      }
      if (exl > 0) {
#pragma unroll
        for (int k = NO; k <= 2 * NO; ++k) out[k] += br[2 * NO - k - ES] - br[HE + 2 * NO - k - ES];
      }
      __syncthreads();
      if (on) {
#pragma unroll
        for (int j = 0; j < M; ++j) br[j] = out[j];
      }
    }
    __syncthreads();

    // ---- gather with the y fold on the fly: a node of a home row cy takes its own
    //      element's cell plus, for cy >= P, the upper neighbour's row cy - P and, for
    //      cy <= 2 NO, the lower neighbour's row cy + P (fixed order).  Own nodes update
    //      u in global memory (rows of OX doubles, coalesced); region nodes owned by
    //      neighbour tiles (the ring) go to the workspace
    auto node = [&](const double* colp, int ey, int cy) {
      // colp: column cx of element (0, ex); ey: element row; cy: window row
      const double* c = colp + ey * (TX * ES);
      double v = c[K::ry(cy) * M];
      if (cy >= P && ey + 1 < TY) v += c[TX * ES + (cy - P) * M];
      if (cy <= 2 * NO && ey > 0) v += c[K::ry(cy + P) * M - TX * ES];
      return v;
    };
    {
      // thread = (tile column ox, element row eyl): the P rows of the element row are
      // compile-time steps, so the window row, its storage row and the fold
      // conditions are constants and every shared-memory offset is an immediate
      constexpr int NG = NT / OX;
      static_assert(NG >= 1, "fewer threads than tile columns");
      const int ox = tid % OX, g = tid / OX;
      const double* colp = U + (ox / P) * ES + (ox % P + NO);
      if (g < NG) {
        for (int eyl = g; eyl < TY; eyl += NG) {
          const double* c = colp + eyl * (TX * ES);
          const bool up = eyl + 1 < TY, dn = eyl > 0;
          double* ug = A.u + (size_t)(Y0 + eyl * P) * N_x + (X0 + ox);
          constexpr int CH = P % 8 == 0 ? 8 : P;   // rows in flight per thread
#pragma unroll
          for (int q0 = 0; q0 < P; q0 += CH) {
            double uv[CH];
#pragma unroll
            for (int q = 0; q < CH; ++q) uv[q] = u_zero ? 0.0 : ug[(size_t)(q0 + q) * N_x];
#pragma unroll
            for (int q = 0; q < CH; ++q) {
              const int cy = q0 + q + NO;
              double v = c[K::ry(cy) * M];
              if (cy >= P && up) v += c[TX * ES + (cy - P) * M];
              if (cy <= 2 * NO && dn) v += c[K::ry(cy + P) * M - TX * ES];
              ug[(size_t)(q0 + q) * N_x] = uv[q] + v;
            }
          }
        }
      }
    }
    {
      double* Wr = A.ws + (size_t)tile * NRING;
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
        Wr[k] = node(U + ex * ES + (x - ex * P), ey, y - ey * P);
      }
    }
    __syncthreads();   // U is free for the next tile's box
  }
}

template <int P, int NO, int TX, int TY>
int fdp_launch_k(const FDTLaunch& L, cudaStream_t st) {
  using G = FDTGeom<P, NO, TX, TY>;
  using K = FDPK<P, NO, TX, TY>;
  constexpr int M = G::M, HE = fdt_he(M), HO = fdt_ho(M);
  FDPArgs<M> A;
  constexpr int HEP = FDPArgs<M>::HEP, HOP = FDPArgs<M>::HOP;
  // umap only feeds the L2 prefetch of the tile's block of u (updated in place in global memory)
  if (!tmap_2d(&A.rmap, L.r, L.N_x, L.N_y, G::BRX, G::RY) || !tmap_2d(&A.umap, L.u, L.N_x, L.N_y, G::OX, G::OY))
    return SMG_EUNSUPPORTED;
  A.r = L.r; A.u = L.u; A.inv_nu = L.inv_nu; A.dinv = L.dinv; A.ws = L.ws;
  A.N_x = L.N_x; A.N_y = L.N_y; A.n_x = L.n_x; A.ntx = L.ntx; A.nty = L.nty;
  A.u_zero = L.u_zero;
  std::memset(A.Sye, 0, sizeof(A.Sye)); std::memset(A.SyeT, 0, sizeof(A.SyeT));
  std::memset(A.Sxe, 0, sizeof(A.Sxe)); std::memset(A.SxeT, 0, sizeof(A.SxeT));
  std::memset(A.Syo, 0, sizeof(A.Syo)); std::memset(A.SyoT, 0, sizeof(A.SyoT));
  std::memset(A.Sxo, 0, sizeof(A.Sxo)); std::memset(A.SxoT, 0, sizeof(A.SxoT));
  // synthesis factors carry the (mirror-symmetric) weight of their output node
  for (int k = 0; k < HE; ++k)
    for (int i = 0; i < HE; ++i) {
      A.Sye[k * HEP + i] = L.Sye[k * HE + i]; A.SyeT[i * HEP + k] = L.Sye[k * HE + i] * L.wy[k];
      A.Sxe[k * HEP + i] = L.Sxe[k * HE + i]; A.SxeT[i * HEP + k] = L.Sxe[k * HE + i] * L.wx[k];
    }
  for (int k = 0; k < HO; ++k)
    for (int i = 0; i < HO; ++i) {
      A.Syo[k * HOP + i] = L.Syo[k * HO + i]; A.SyoT[i * HOP + k] = L.Syo[k * HO + i] * L.wy[k];
      A.Sxo[k * HOP + i] = L.Sxo[k * HO + i]; A.SxoT[i * HOP + k] = L.Sxo[k * HO + i] * L.wx[k];
    }
  static DeviceInt grid_cap;
  if (grid_cap == 0) {
    if (K::SMEM > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(fdp_kernel<P, NO, TX, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)K::SMEM);
      if (e != cudaSuccess) return cuda_fail(e, "fdp_kernel smem attribute");
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fdp_kernel<P, NO, TX, TY>, K::NT, K::SMEM);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int ntiles = L.ntx * L.nty;
  const int grid = ntiles < grid_cap ? ntiles : grid_cap;
  launch(fdp_kernel<P, NO, TX, TY>, dim3(grid), dim3(K::NT), K::SMEM, st, A);
  int rc = check_launch("fdp_kernel");
  if (rc) return rc;
  const long nb = fdt_fixup_per_tile<P, NO, TX, TY>() * ntiles;
  launch(fdt_fixup<P, NO, TX, TY>, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, st, L.u, L.ws, L.N_x, L.ntx,
         L.nty);
  return check_launch("fdt_fixup");
}

// Paired-line kernel for (p, n_o) on an n_x x n_y mesh, or nullptr; sets TX, TY.
FDTLaunchFn fdp_dispatch(int p, int n_o, int n_x, int n_y, int* TX, int* TY);

}  // namespace smg
