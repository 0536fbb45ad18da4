// Poisson residual r = f - A u with one WARP per element (p = 8, 16).
//
// Same operator and gather form as op_kernel (smg_op.cuh; reference
// PoissonOperator.apply, operators.py:49-54, residual :101-103), organised
// so that no block-level barrier separates the passes:
//   * the CTA stages the u window of its TX x TY element tile (one-element
//     halo on the low side, one node on the high side) by bulk row copies;
//   * in every warp, lanes 0..p-1 run the even/odd row line of element row a
//     (and the left neighbour's vertex-only line), lanes 16..16+p-1 the column
//     line of element column b (and the lower neighbour's vertex-only line) --
//     the same code path on both halves (runtime stride), so the warp does not
//     diverge, and the 1D operator entries are uniform parameter-bank operands;
//   * x- and y-parts meet in two per-warp 16 x 17 shared buffers; each lane
//     then writes p/2 outputs of its column: coalesced rows of r.
// Deterministic: every output node has one writer, fixed summation order.
#include <cstring>

#include "smg_common.cuh"
#include "smg_op.cuh"
#include "smg_tma.cuh"

namespace smg {

template <int P>
struct OpwArgs {
  const double* __restrict__ u;
  const double* __restrict__ f;
  double* __restrict__ out;
  double* __restrict__ dotp;   // DOT kernels: per-CTA partials of sum(u * out)
  double* __restrict__ fc;     // RESTR kernels: the coarse field and the restriction ring (smg_rw.cu layout)
  double* __restrict__ rring;
  int N_x, N_y, tiles_x;
  double cx, cy;
  double Le[((P + 1) / 2 + 1) * ((P + 1) / 2 + 1)];
  double Lo[((P + 1) / 2) * ((P + 1) / 2) + 1];
  double wasm[P];
  // opl_kernel: the same halves transposed ([k][b], rows padded to an even length and 16-byte
  // aligned) so that the b loop at a fixed k reads consecutive entries (128-bit uniform loads)
  static constexpr int kH = (P + 1) / 2, kHC = kH + ((P + 1) & 1), kHCP = (kHC + 1) & ~1, kHP = (kH + 1) & ~1;
  alignas(16) double LeT[(kH + 1) * kHCP];
  alignas(16) double LoT[(kH > 0 ? kH : 1) * kHP];
  double J[P * (P / 2 + 1)];   // RESTR: interpolation rows a < P (p_c = P/2), J[a * (p_c + 1) + ac]
};

// Even/odd 1D line: v[b] = sum_k L[k][b] x[k st] (L centro-symmetric); with
// ONLY_LAST just v[P].
template <int P, bool ONLY_LAST>
__device__ __forceinline__ void opw_line(const OpwArgs<P>& A, const double* x, int st, double (&v)[P + 1]) {
  constexpr int NP = P + 1, H = NP / 2;
  constexpr bool MID = (NP & 1) != 0;
  constexpr int HC = H + (MID ? 1 : 0);
  double a[H], d[H];
#pragma unroll
  for (int k = 0; k < H; ++k) {
    const double xk = x[k * st], xm = x[(P - k) * st];
    a[k] = xk + xm;
    d[k] = xk - xm;
  }
  const double c = MID ? x[H * st] : 0.0;
  if (ONLY_LAST) {
    double e = MID ? A.Le[H] * c : 0.0, o = 0.0;
#pragma unroll
    for (int k = 0; k < H; ++k) {
      e = fma(A.Le[k], a[k], e);
      o = fma(A.Lo[k], d[k], o);
    }
    v[P] = e - o;
  } else {
    double e[HC], o[H];
#pragma unroll
    for (int b = 0; b < HC; ++b) e[b] = MID ? A.Le[b * HC + H] * c : 0.0;
#pragma unroll
    for (int b = 0; b < H; ++b) o[b] = 0.0;
#pragma unroll
    for (int k = 0; k < H; ++k) {
#pragma unroll
      for (int b = 0; b < HC; ++b) e[b] = fma(A.Le[b * HC + k], a[k], e[b]);
#pragma unroll
      for (int b = 0; b < H; ++b) o[b] = fma(A.Lo[b * H + k], d[k], o[b]);
    }
#pragma unroll
    for (int b = 0; b < H; ++b) {
      v[b] = e[b] + o[b];
      v[P - b] = e[b] - o[b];
    }
    if (MID) v[H] = e[H];
  }
}

template <int P, int TX, int TY>
struct OpwGeom {
  // elements per warp: the row lines of an element take P of a half-warp's 16 lanes, so at
  // p = 8 a warp carries two elements (one per 8-lane group of each half) -- 8 idle lanes of
  // 16 made the p = 8 residual latency-bound at twice the warps (C4 level 8: 51 us for 4.2 M DOF)
  static constexpr int EW = P <= 8 ? 16 / P : 1;
  static_assert((TX * TY) % EW == 0, "whole warps");
  static constexpr int NW = TX * TY / EW;
  static constexpr int OX = TX * P, OY = TY * P;
  static constexpr int HX = OX + P + 1, HY = OY + P + 1;
  static constexpr int DP = (HX + 2) & ~1;
  static constexpr int LDA = P + 1;   // per-warp AX row stride
  static constexpr size_t SMEM = sizeof(double) * ((size_t)DP * HY + (size_t)TX * TY * P * LDA) + 16;
};

// DOT: also the per-CTA partial of sum(u * out) over the CTA's nodes (MGCG's p . A p without
// re-reading p and q: the node's u is in the staged window); fixed shuffle / warp order.
// RESTR (with f: r = f - A u): r is not written; the column lanes restrict their column of the
// element's own nodes in registers (y pass), the row lanes finish the x pass from the warp's
// buffer, own coarse nodes are written and the high-side coarse row / column go to the
// restriction ring -- restrict_warp_kernel's passes and summation order (smg_rw.cu), fed from
// registers instead of from a stored residual; restrict_fixup follows.
template <int P, int TX, int TY, bool DOT = false, bool RESTR = false>
__global__ void __launch_bounds__(32 * OpwGeom<P, TX, TY>::NW,
                                  OpwGeom<P, TX, TY>::NW == 4 ? (RESTR ? 6 : 7) : (OpwGeom<P, TX, TY>::NW == 2 ? 12 : 1))
opw_kernel(const __grid_constant__ OpwArgs<P> A) {
  SMG_PDL_TRIGGER();
  using G = OpwGeom<P, TX, TY>;
  constexpr int NW = G::NW, EW = G::EW, OX = G::OX, OY = G::OY, HX = G::HX, HY = G::HY, DP = G::DP, LDA = G::LDA;
  static_assert(2 * P <= 32, "row and column lines share one warp");
  extern __shared__ __align__(16) double smw[];
  double* U = smw;                          // HY x DP, origin (Y0-P, X0-P) at column sh
  double* AXb = U + DP * HY;                // (TX TY) x P x LDA: x-part [a][b] per element
  uint64_t* bar = reinterpret_cast<uint64_t*>(AXb + TX * TY * P * LDA);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tx = blockIdx.x % A.tiles_x, ty = blockIdx.x / A.tiles_x;
  const int X0 = tx * OX, Y0 = ty * OY;
  const int N_x = A.N_x, N_y = A.N_y;
  const int sh = pwin_shift(X0 - P, N_x);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, pwin_bytes(HX, HY, sh));
  }
  SMG_PDL_WAIT();   // barrier set up while the preceding grid drains; u after it
  __syncthreads();
  if (warp == 0) pwin_issue_warp(A.u, N_x, N_y, X0 - P, Y0 - P, HX, HY, U, DP, bar);
  // this lane's element: lane group (lane & 15) / P of the warp's EW elements
  const int sub = (lane & 15) / P;
  const bool lact = sub < EW;
  const int eidx = warp * EW + (lact ? sub : 0);
  const int exl = eidx % TX, eyl = eidx / TX;
  // the first chunk of f rows of the column lanes, requested while the window is in flight
  // (ncu: 16 % of the stall samples sat on the first use of f after the lines)
  // (RESTR only: the plain and DOT variants at p = 16 spill with eight more live doubles)
  constexpr int CHF = P / 2;
  [[maybe_unused]] double f0[CHF];
  if constexpr (RESTR) {
    const bool cl = lane >= 16 && lact && A.f != nullptr;
    const size_t gf = (size_t)(Y0 + eyl * P) * N_x + (X0 + exl * P + (lane & 15) % P);
#pragma unroll
    for (int i = 0; i < CHF; ++i) f0[i] = cl ? __ldg(A.f + gf + (size_t)i * N_x) : 0.0;
  }
  mbar_wait(bar, 0);
  // element origin in U
  const int ur0 = P + eyl * P, uc0 = sh + P + exl * P;
  double* AX = AXb + eidx * P * LDA;
  // lanes [0,16): row a = li (stride 1); lanes [16,32): column b = li (stride DP)
  const int li = (lane & 15) % P;
  const bool col = lane >= 16;
  const int st = col ? DP : 1;
  const double* xl = col ? U + ur0 * DP + uc0 + li : U + (ur0 + li) * DP + uc0;
  const double* xv = col ? xl - P * DP : xl - P;   // the neighbour element's line (vertex term)
  double v[P + 1], vv[P + 1];
  if (lact) {
    opw_line<P, false>(A, xl, st, v);
    opw_line<P, true>(A, xv, st, vv);
    // raw line values; the combination below is op_kernel's, operation for
    // operation (bitwise-equal results)
    if (!col) {
      double* dst = AX + li * LDA;      // x-sum of row a = li at column b (+ left vertex at b = 0)
      dst[0] = v[0] + vv[P];
#pragma unroll
      for (int k = 1; k < P; ++k) dst[k] = v[k];
    }
  }
  __syncwarp();
  // the column lane b keeps the y-part of its column in registers and writes
  // the column's outputs (each row of r coalesced across the half-warp)
  [[maybe_unused]] double dacc = 0.0;
  if (col && lact) {
    const int b = li;
    const double wyb = A.cy * A.wasm[b];
    const size_t g0 = (size_t)(Y0 + eyl * P) * N_x + (X0 + exl * P + b);
    constexpr int CH = P / 2;          // f loads in flight per chunk
    constexpr int PCr = P / 2, NCr = PCr + 1;
    [[maybe_unused]] double tr[NCr];
    if constexpr (RESTR) {
#pragma unroll
      for (int ay = 0; ay < NCr; ++ay) tr[ay] = 0.0;
    }
#pragma unroll
    for (int a0 = 0; a0 < P; a0 += CH) {
      double fv[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i)
        fv[i] = (RESTR && a0 == 0) ? f0[i] : (A.f != nullptr ? __ldg(A.f + g0 + (size_t)(a0 + i) * N_x) : 0.0);
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int a = a0 + i;
        double val = fma(A.cx * A.wasm[a], AX[a * LDA + b], wyb * v[a]);
        if (a == 0) val = fma(wyb, vv[P], val);
        const double o = A.f != nullptr ? fv[i] - val : val;
        if constexpr (RESTR) {
#pragma unroll
          for (int ay = 0; ay < NCr; ++ay) tr[ay] = fma(A.J[a * NCr + ay], o, tr[ay]);
        } else {
          A.out[g0 + (size_t)a * N_x] = o;
        }
        if constexpr (DOT) dacc = fma(U[(ur0 + a) * DP + uc0 + b], o, dacc);
      }
    }
    if constexpr (RESTR) {
      // T[ay][b] over the x-parts of this column (no other lane reads column b)
#pragma unroll
      for (int ay = 0; ay < NCr; ++ay) AX[ay * LDA + b] = tr[ay];
    }
  }
  if constexpr (RESTR) {
    constexpr int PCr = P / 2, NCr = PCr + 1;
    __syncwarp();
    if (!col && lact && li < NCr) {
      const double* trow = AX + li * LDA;
      double c[NCr];
#pragma unroll
      for (int ax = 0; ax < NCr; ++ax) c[ax] = 0.0;
#pragma unroll
      for (int b = 0; b < P; ++b) {
        const double tb = trow[b];
#pragma unroll
        for (int ax = 0; ax < NCr; ++ax) c[ax] = fma(A.J[b * NCr + ax], tb, c[ax]);
      }
      const int ex = tx * TX + exl, ey = ty * TY + eyl, n_x = A.tiles_x * TX;
      double* R = A.rring + (size_t)(ey * n_x + ex) * (2 * PCr + 1);
      if (li < PCr) {
        double* d = A.fc + (size_t)(ey * PCr + li) * ((size_t)n_x * PCr) + ex * PCr;
#pragma unroll
        for (int ax = 0; ax < PCr; ++ax) d[ax] = c[ax];
        R[PCr + 1 + li] = c[PCr];            // right column
      } else {
#pragma unroll
        for (int ax = 0; ax < NCr; ++ax) R[ax] = c[ax];   // top row, corner last
      }
    }
  }
  if constexpr (DOT) {
    // the column lanes hold their columns' sums, every other lane an exact zero: fixed
    // xor tree over the whole warp (outside the divergent branches), then the warps in order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
    if (lane == 0) AX[0] = dacc;   // the x-part buffer of the warp's first element is consumed
  }
  if constexpr (DOT) {
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) s += AXb[w * EW * P * LDA];
      A.dotp[blockIdx.x] = s;
    }
  }
}

// Host: 1 = not applicable (caller uses op_kernel).
template <int P, int TX, int TY>
int opw_launch_t(const OpLaunch& L, cudaStream_t st, double* dotp = nullptr, const double* J = nullptr,
                 double* fc = nullptr, double* rring = nullptr) {
  using G = OpwGeom<P, TX, TY>;
  if (L.diffusion || L.partials != nullptr || L.n_x % TX || L.n_y % TY) return 1;
  // the periodic window loader wraps once: the staged window must not exceed the mesh
  if (L.n_x * P < G::HX || L.n_y * P < G::HY) return 1;
  const int N_x = L.n_x * P;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (N_x % 2 || !al16(L.u)) return 1;
  OpwArgs<P> A;
  A.u = L.u; A.f = L.f; A.out = L.out; A.dotp = dotp; A.fc = fc; A.rring = rring;
  if (J != nullptr) std::memcpy(A.J, J, sizeof(A.J));
  A.N_x = N_x; A.N_y = L.n_y * P; A.tiles_x = L.n_x / TX;
  A.cx = L.cx; A.cy = L.cy;
  {
    // even/odd halves of L-hat (host-checked centro-symmetry, as op_fill_consts)
    constexpr int NP = P + 1, H = NP / 2, HC = H + (NP & 1);
    auto Lbk = [&](int bb, int k) { return L.Mt[k * NP + bb]; };
    double asym = 0.0, mx = 0.0;
    for (int bb = 0; bb < NP; ++bb)
      for (int k = 0; k < NP; ++k) {
        asym = std::fmax(asym, std::fabs(Lbk(bb, k) - Lbk(P - bb, P - k)));
        mx = std::fmax(mx, std::fabs(Lbk(bb, k)));
      }
    if (asym > 1e-14 * mx) return 1;
    for (int bb = 0; bb < HC; ++bb) {
      for (int k = 0; k < H; ++k) A.Le[bb * HC + k] = 0.5 * (Lbk(bb, k) + Lbk(bb, P - k));
      if (NP & 1) A.Le[bb * HC + H] = Lbk(bb, H);
    }
    for (int bb = 0; bb < H; ++bb)
      for (int k = 0; k < H; ++k) A.Lo[bb * H + k] = 0.5 * (Lbk(bb, k) - Lbk(bb, P - k));
    A.Lo[H * H] = 0.0;
  }
  for (int i = 0; i < P; ++i) A.wasm[i] = L.wasm[i];
  static DeviceFlag attr;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(opw_kernel<P, TX, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)G::SMEM);
    if (e != cudaSuccess) return cuda_fail(e, "opw_kernel smem attribute");
    attr = true;
  }
  if (dotp != nullptr) {
    static DeviceFlag attr2;
    if (!attr2) {
      cudaError_t e = cudaFuncSetAttribute(opw_kernel<P, TX, TY, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)G::SMEM);
      if (e != cudaSuccess) return cuda_fail(e, "opw_kernel smem attribute");
      attr2 = true;
    }
    launch(opw_kernel<P, TX, TY, true>, dim3((L.n_x / TX) * (L.n_y / TY)), dim3(32 * G::NW), G::SMEM, st, A);
    return check_launch("opw_kernel");
  }
  if (J != nullptr) {
    static DeviceFlag attr3;
    if (!attr3) {
      cudaError_t e = cudaFuncSetAttribute(opw_kernel<P, TX, TY, false, true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
      if (e != cudaSuccess) return cuda_fail(e, "opw_kernel smem attribute");
      attr3 = true;
    }
    launch(opw_kernel<P, TX, TY, false, true>, dim3((L.n_x / TX) * (L.n_y / TY)), dim3(32 * G::NW), G::SMEM, st, A);
    return check_launch("opw_kernel");
  }
  launch(opw_kernel<P, TX, TY>, dim3((L.n_x / TX) * (L.n_y / TY)), dim3(32 * G::NW), G::SMEM, st, A);
  return check_launch("opw_kernel");
}

// fc (+ ring) = restriction of r = f - A u to p_c = p / 2 without storing r (p = 8, 16; J: rows a < p of
// the (p+1) x (p_c+1) interpolation matrix); the caller runs restrict_fixup next.  1 = not applicable.
int opw_residual_restrict(const OpLaunch& L, const double* J, double* fc, double* rring, cudaStream_t st) {
  static const int on = env_int("SMG_RR_OPW", 1);
  if (!on || L.f == nullptr || J == nullptr || fc == nullptr || rring == nullptr) return 1;
  if (L.p == 16) return opw_launch_t<16, 2, 2>(L, st, nullptr, J, fc, rring);
  if (L.p == 8) {   // 4x2-element tiles (four warps) where they fit: C4 level-8 pair 35.8 -> 33.1 us
    const int rc = opw_launch_t<8, 4, 2>(L, st, nullptr, J, fc, rring);
    return rc != 1 ? rc : opw_launch_t<8, 2, 2>(L, st, nullptr, J, fc, rring);
  }
  if (L.p == 4) {   // four elements per warp; 4 x 4-element tiles where the mesh allows
    const int rc = opw_launch_t<4, 4, 4>(L, st, nullptr, J, fc, rring);
    return rc != 1 ? rc : opw_launch_t<4, 2, 2>(L, st, nullptr, J, fc, rring);
  }
  return 1;
}

// out = A u and per-CTA partials of u . out (n_ctas of them); 1 = not applicable.
int opw_apply_dot(const OpLaunch& L, double* partials, int* n_ctas, cudaStream_t st) {
  static const int on = env_int("SMG_OP_WARP", 1);
  if (!on || L.f != nullptr || partials == nullptr) return 1;
  *n_ctas = (L.n_x / 2) * (L.n_y / 2);
  if (L.p == 16) return opw_launch_t<16, 2, 2>(L, st, partials);
  if (L.p == 8) return opw_launch_t<8, 2, 2>(L, st, partials);
  return 1;
}

// ---- p = 32: one element per CTA, a row warp and a column warp, halo-free -----------
// The tensor-core kernel (opdh_kernel, smg_opd.cu) pads the even/odd halves of L-hat
// (17 x 17, 16 x 16) to 20 x 24 DMMA slots -- 57 % useful -- and the DMMA and DFMA pipes
// are one datapath (profiles/r2_fp64_mixed_pipes.txt), so at p = 32 the exact DFMA form is
// the cheaper one per line (34 vs 60 pipe cycles).  A CTA stages its element's own
// (p+1)^2 window (odd pitch: rows and columns are both conflict-free); warp 0 runs the p
// row lines (lane = row a, k-streamed even/odd line, L-hat entries as uniform operands),
// warp 1 the p column lines; the x-parts meet warp 1 in shared memory, which writes the
// coalesced rows of r.  Node-p values go to the ring of opdh_kernel's layout ([0,p) rows,
// [p,2p) columns per element); opl_fixup applies them.
template <int P>
__device__ __forceinline__ void opl_line(const OpwArgs<P>& A, const double* x, int st, double (&v)[P + 1]) {
  constexpr int NP = P + 1, H = NP / 2;
  constexpr bool MID = (NP & 1) != 0;
  constexpr int HC = H + (MID ? 1 : 0);
  constexpr int HCP = OpwArgs<P>::kHCP, HP = OpwArgs<P>::kHP;
  double e[HC], o[H];
  {
    const double c = MID ? x[H * st] : 0.0;
    const double2* __restrict__ Lc = reinterpret_cast<const double2*>(A.LeT + H * HCP);
#pragma unroll
    for (int b = 0; b < HC; b += 2) {
      const double2 l2 = Lc[b / 2];
      e[b] = MID ? l2.x * c : 0.0;
      if (b + 1 < HC) e[b + 1] = MID ? l2.y * c : 0.0;
    }
#pragma unroll
    for (int b = 0; b < H; ++b) o[b] = 0.0;
  }
  // the inputs of the next PF steps are requested before this step's FMAs
  constexpr int PF = 4;
  double xk[PF], xm[PF];
#pragma unroll
  for (int q = 0; q < PF; ++q) {
    xk[q] = q < H ? x[q * st] : 0.0;
    xm[q] = q < H ? x[(P - q) * st] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < H; ++k) {
    const double a = xk[k % PF] + xm[k % PF], d = xk[k % PF] - xm[k % PF];
    if (k + PF < H) {
      xk[k % PF] = x[(k + PF) * st];
      xm[k % PF] = x[(P - k - PF) * st];
    }
    const double2* __restrict__ Le2 = reinterpret_cast<const double2*>(A.LeT + k * HCP);
    const double2* __restrict__ Lo2 = reinterpret_cast<const double2*>(A.LoT + k * HP);
#pragma unroll
    for (int b = 0; b < HC; b += 2) {
      const double2 l2 = Le2[b / 2];
      e[b] = fma(l2.x, a, e[b]);
      if (b + 1 < HC) e[b + 1] = fma(l2.y, a, e[b + 1]);
    }
#pragma unroll
    for (int b = 0; b < H; b += 2) {
      const double2 l2 = Lo2[b / 2];
      o[b] = fma(l2.x, d, o[b]);
      if (b + 1 < H) o[b + 1] = fma(l2.y, d, o[b + 1]);
    }
  }
#pragma unroll
  for (int b = 0; b < H; ++b) {
    v[b] = e[b] + o[b];
    v[P - b] = e[b] - o[b];
  }
  if (MID) v[H] = e[H];
}

template <int P>
struct OplGeom {
  static constexpr int NP = P + 1, DPW = NP | 1, LDA = P | 1;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)NP * DPW + (size_t)P * LDA);
};

template <int P>
__global__ void __launch_bounds__(64, 10) opl_kernel(const __grid_constant__ OpwArgs<P> A, double* __restrict__ ring) {
  SMG_PDL_ENTRY();
  using G = OplGeom<P>;
  constexpr int NP = G::NP, DPW = G::DPW, LDA = G::LDA;
  static_assert(P <= 32, "one lane per line");
  extern __shared__ __align__(16) double smw[];
  double* U = smw;                 // NP x DPW window of u, origin (Y0, X0)
  double* AX = U + NP * DPW;       // P x LDA x-parts [a][b]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int el = blockIdx.x;
  const int ex = el % A.tiles_x, ey = el / A.tiles_x;
  const int X0 = ex * P, Y0 = ey * P;
  const int N_x = A.N_x, N_y = A.N_y;
  // window rows: coalesced row segments, periodic wrap on the high side
  // (8-byte cp.async: every value in flight at once, no register round trip; the odd
  // pitch rules out 16-byte bulk rows)
  {
    const int xw = X0 + P == N_x ? 0 : X0 + P;     // the high-side column (periodic)
    for (int i = tid; i < NP * NP; i += 64) {
      const int y = i / NP, x = i - y * NP;
      const int gy = Y0 + y == N_y ? 0 : Y0 + y;
      const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(U + y * DPW + x));
      const double* g = A.u + (size_t)gy * N_x + (x == P ? xw : X0 + x);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(g));
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }
  __syncthreads();
  double* R = ring + (size_t)el * (2 * P);
  double v[P + 1];
  if (lane < P) {
    if (warp == 0) {
      opl_line<P>(A, U + lane * DPW, 1, v);          // row a = lane
#pragma unroll
      for (int b = 0; b < P; ++b) AX[lane * LDA + b] = v[b];
      R[lane] = v[P];
    } else {
      opl_line<P>(A, U + lane, DPW, v);              // column b = lane
      R[P + lane] = v[P];
    }
  }
  __syncthreads();
  if (warp == 1 && lane < P) {
    const int b = lane;
    const double wyb = A.cy * A.wasm[b];
    const size_t g0 = (size_t)Y0 * N_x + (X0 + b);
    constexpr int CH = 8;
#pragma unroll
    for (int a0 = 0; a0 < P; a0 += CH) {
      double fv[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) fv[i] = A.f != nullptr ? __ldg(A.f + g0 + (size_t)(a0 + i) * N_x) : 0.0;
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int a = a0 + i;
        const double val = fma(A.cx * A.wasm[a], AX[a * LDA + b], wyb * v[a]);
        A.out[g0 + (size_t)a * N_x] = A.f != nullptr ? fv[i] - val : val;
      }
    }
  }
}

// One thread per low-side node of an element (as opdh_fixup, smg_opd.cu): (a, 0) takes the
// left element's row-line value, then at the corner the lower element's column-line value;
// (0, b), b >= 1, the lower element's.
template <int P>
__global__ void __launch_bounds__(256) opl_fixup(double* __restrict__ out, const double* __restrict__ ring, int n_x,
                                                 int n_y, double sign, const __grid_constant__ OpwArgs<P> A) {
  SMG_PDL_ENTRY();
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long)n_x * n_y * 2 * P) return;
  const int e = (int)(gid / (2 * P)), k = (int)(gid - (long)e * (2 * P));
  if (k == P) return;
  const int ey = e / n_x, ex = e - ey * n_x;
  const int el = ey * n_x + wrapi(ex - 1, n_x), ed = wrapi(ey - 1, n_y) * n_x + ex;
  const int a = k < P ? k : 0, b = k < P ? 0 : k - P;
  double* o = out + (size_t)(ey * P + a) * ((size_t)n_x * P) + ex * P + b;
  double v = *o;
  if (k < P) v = fma(sign * A.cx * A.wasm[a], ring[(size_t)el * (2 * P) + a], v);
  if (k > P) v = fma(sign * A.cy * A.wasm[b], ring[(size_t)ed * (2 * P) + P + b], v);
  if (k == 0) v = fma(sign * A.cy * A.wasm[0], ring[(size_t)ed * (2 * P) + P], v);
  *o = v;
}

// Host: 1 = not applicable.
template <int P>
int opl_launch_t(const OpLaunch& L, double* ring, cudaStream_t st) {
  using G = OplGeom<P>;
  if (L.diffusion || L.partials != nullptr || ring == nullptr) return 1;
  OpwArgs<P> A;
  A.u = L.u; A.f = L.f; A.out = L.out; A.dotp = nullptr;
  A.N_x = L.n_x * P; A.N_y = L.n_y * P; A.tiles_x = L.n_x;
  A.cx = L.cx; A.cy = L.cy;
  {
    constexpr int NP = P + 1, H = NP / 2, HC = H + (NP & 1);
    auto Lbk = [&](int bb, int k) { return L.Mt[k * NP + bb]; };
    double asym = 0.0, mx = 0.0;
    for (int bb = 0; bb < NP; ++bb)
      for (int k = 0; k < NP; ++k) {
        asym = std::fmax(asym, std::fabs(Lbk(bb, k) - Lbk(P - bb, P - k)));
        mx = std::fmax(mx, std::fabs(Lbk(bb, k)));
      }
    if (asym > 1e-14 * mx) return 1;
    for (int bb = 0; bb < HC; ++bb) {
      for (int k = 0; k < H; ++k) A.Le[bb * HC + k] = 0.5 * (Lbk(bb, k) + Lbk(bb, P - k));
      if (NP & 1) A.Le[bb * HC + H] = Lbk(bb, H);
    }
    for (int bb = 0; bb < H; ++bb)
      for (int k = 0; k < H; ++k) A.Lo[bb * H + k] = 0.5 * (Lbk(bb, k) - Lbk(bb, P - k));
    A.Lo[H * H] = 0.0;
    constexpr int HCP = OpwArgs<P>::kHCP, HP = OpwArgs<P>::kHP;
    std::memset(A.LeT, 0, sizeof(A.LeT));
    std::memset(A.LoT, 0, sizeof(A.LoT));
    for (int bb = 0; bb < HC; ++bb)
      for (int k = 0; k < HC; ++k) A.LeT[k * HCP + bb] = A.Le[bb * HC + k];
    for (int bb = 0; bb < H; ++bb)
      for (int k = 0; k < H; ++k) A.LoT[k * HP + bb] = A.Lo[bb * H + k];
  }
  for (int i = 0; i < P; ++i) A.wasm[i] = L.wasm[i];
  static DeviceFlag attr;
  if (!attr) {
    if (G::SMEM > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(opl_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
      if (e != cudaSuccess) return cuda_fail(e, "opl_kernel smem attribute");
    }
    attr = true;
  }
  const int n_el = L.n_x * L.n_y;
  static const int pdl_big = env_int("SMG_OPL_PDL", 0);
  const bool pdl = n_el < kPdlMaxElements || pdl_big;
  launch_pdl(pdl, opl_kernel<P>, dim3(n_el), dim3(64), G::SMEM, st, A, ring);
  int rc = check_launch("opl_kernel");
  if (rc) return rc;
  const long nb = (long)n_el * 2 * P;
  launch_pdl(pdl, opl_fixup<P>, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, st, L.out, (const double*)ring, L.n_x,
             L.n_y, L.f != nullptr ? -1.0 : 1.0, A);
  return check_launch("opl_fixup");
}

// Poisson p = 32 with a ring workspace; 1 = not applicable (SMG_OPL=0 keeps opdh_kernel)
int opl_launch(const OpLaunch& L, cudaStream_t st) {
  static const int on = env_int("SMG_OPL", 1);
  if (!on || L.p != 32) return 1;
  return opl_launch_t<32>(L, L.ring, st);
}

int opw_launch(const OpLaunch& L, cudaStream_t st) {
  static const int on = env_int("SMG_OP_WARP", 1);
  if (!on) return 1;
  if (L.p == 16) return opw_launch_t<16, 2, 2>(L, st);
  if (L.p == 8) return opw_launch_t<8, 2, 2>(L, st);
  return 1;
}

}  // namespace smg
