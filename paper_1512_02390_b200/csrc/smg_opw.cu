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
  int N_x, N_y, tiles_x;
  double cx, cy;
  double Le[((P + 1) / 2 + 1) * ((P + 1) / 2 + 1)];
  double Lo[((P + 1) / 2) * ((P + 1) / 2) + 1];
  double wasm[P];
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
  static constexpr int NW = TX * TY;
  static constexpr int OX = TX * P, OY = TY * P;
  static constexpr int HX = OX + P + 1, HY = OY + P + 1;
  static constexpr int DP = (HX + 2) & ~1;
  static constexpr int LDA = P + 1;   // per-warp AX row stride
  static constexpr size_t SMEM = sizeof(double) * ((size_t)DP * HY + (size_t)NW * P * LDA) + 16;
};

// DOT: also the per-CTA partial of sum(u * out) over the CTA's nodes (MGCG's p . A p without
// re-reading p and q: the node's u is in the staged window); fixed shuffle / warp order.
template <int P, int TX, int TY, bool DOT = false>
__global__ void __launch_bounds__(32 * TX * TY, TX * TY == 4 ? 7 : 1) opw_kernel(const __grid_constant__ OpwArgs<P> A) {
  SMG_PDL_TRIGGER();
  using G = OpwGeom<P, TX, TY>;
  constexpr int NW = G::NW, OX = G::OX, OY = G::OY, HX = G::HX, HY = G::HY, DP = G::DP, LDA = G::LDA;
  static_assert(2 * P <= 32, "row and column lines share one warp");
  extern __shared__ __align__(16) double smw[];
  double* U = smw;                          // HY x DP, origin (Y0-P, X0-P) at column sh
  double* AXb = U + DP * HY;                // NW x P x LDA: x-part [a][b]
  uint64_t* bar = reinterpret_cast<uint64_t*>(AXb + NW * P * LDA);
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
  // this warp's element
  const int exl = warp % TX, eyl = warp / TX;
  mbar_wait(bar, 0);
  // element origin in U
  const int ur0 = P + eyl * P, uc0 = sh + P + exl * P;
  double* AX = AXb + warp * P * LDA;
  // lanes 0..P-1: row a = lane (stride 1); lanes 16..16+P-1: column b (stride DP)
  const int li = lane & 15;
  const bool lact = li < P;
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
#pragma unroll
    for (int a0 = 0; a0 < P; a0 += CH) {
      double fv[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) fv[i] = A.f != nullptr ? __ldg(A.f + g0 + (size_t)(a0 + i) * N_x) : 0.0;
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int a = a0 + i;
        double val = fma(A.cx * A.wasm[a], AX[a * LDA + b], wyb * v[a]);
        if (a == 0) val = fma(wyb, vv[P], val);
        const double o = A.f != nullptr ? fv[i] - val : val;
        A.out[g0 + (size_t)a * N_x] = o;
        if constexpr (DOT) dacc = fma(U[(ur0 + a) * DP + uc0 + b], o, dacc);
      }
    }
  }
  if constexpr (DOT) {
    // the column lanes hold their columns' sums, every other lane an exact zero: fixed
    // xor tree over the whole warp (outside the divergent branches), then the warps in order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
    if (lane == 0) AX[0] = dacc;   // the warp's x-part buffer is consumed
  }
  if constexpr (DOT) {
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) s += AXb[w * P * LDA];
      A.dotp[blockIdx.x] = s;
    }
  }
}

// Host: 1 = not applicable (caller uses op_kernel).
template <int P, int TX, int TY>
int opw_launch_t(const OpLaunch& L, cudaStream_t st, double* dotp = nullptr) {
  using G = OpwGeom<P, TX, TY>;
  if (L.diffusion || L.partials != nullptr || L.n_x % TX || L.n_y % TY) return 1;
  const int N_x = L.n_x * P;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (N_x % 2 || !al16(L.u)) return 1;
  OpwArgs<P> A;
  A.u = L.u; A.f = L.f; A.out = L.out; A.dotp = dotp;
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
  launch(opw_kernel<P, TX, TY>, dim3((L.n_x / TX) * (L.n_y / TY)), dim3(32 * G::NW), G::SMEM, st, A);
  return check_launch("opw_kernel");
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

int opw_launch(const OpLaunch& L, cudaStream_t st) {
  static const int on = env_int("SMG_OP_WARP", 1);
  if (!on) return 1;
  if (L.p == 16) return opw_launch_t<16, 2, 2>(L, st);
  if (L.p == 8) return opw_launch_t<8, 2, 2>(L, st);
  return 1;
}

}  // namespace smg
