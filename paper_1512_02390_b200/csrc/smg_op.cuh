// Matrix-free GLL operator apply / residual (subsystem 2).
//
// Reference: PoissonOperator.apply (operators.py:49-54),
// DiffusionOperator.apply (operators.py:86-92), residual (:101-103).
// The reference gathers (p+1)^2 element blocks, applies the element kernel
// by sum factorization and scatter-adds with bincount.  Both operators are
// sums of an x-part (a 1D operator along every node row, element by element)
// and a y-part (along every node column):
//   Poisson   : (A u)[Y,X] = (dy/dx) Wy(Y) sum_{e in row}  (u_e L)[b]
//                          + (dx/dy) Wx(X) sum_{e in col}  (L u_e)[a]
//   Diffusion : x-part = (dy/dx) Wy(Y) sum_e sum_j nu w_j (D u_e)_j D[j][b]
//               y-part = (dx/dy) Wx(X) sum_e sum_i D[i][a] nu w_i (D u_e)_i
// with W*(.) the assembled GLL weight (w_0 + w_p at element vertices).  The
// kernel evaluates that form in GATHER order -- every output node is written
// by exactly one thread: no scatter, no atomics, deterministic.
//
// A CTA owns a TY x TX block of elements (compile-time).  It stages u (and
// nu) with a one-element halo on the low side plus one node on the high
// side, and f, with cp.async; runs the row passes (thread = (node row,
// element)) and column passes (thread = (node column, element)) with the 1D
// matrices in the parameter constant bank; and combines the two vertex
// contributions of neighbouring elements in shared memory.  Fused outputs:
// r = f - A u (f may be absent) and per-CTA partials of ||r||^2.
#pragma once
#include <cmath>
#include <vector>
#include "smg_common.cuh"
#include "smg_tma.cuh"

namespace smg {

template <int P>
struct OpArgs {
  const double* __restrict__ u;
  const double* __restrict__ f;      // nullable: out = A u
  double* __restrict__ out;
  const double* __restrict__ nu;     // diffusion only
  double* __restrict__ partials;     // nullable: per-CTA sum of out^2
  int N_x, N_y, tiles_x;
  int bulk;                          // 1: bulk row copies (N_x even, 16-byte aligned fields)
  double cx, cy;
  double Mt[(P + 1) * (P + 1)];      // Poisson: stiffness L-hat; diffusion: D (row-major)
  // Poisson even/odd halves of L-hat (centro-symmetric): row b, pair k
  //   Le[b][k] = (L[b][k] + L[b][P-k]) / 2 (k < H), Le[b][H] = L[b][H] (odd P+1)
  //   Lo[b][k] = (L[b][k] - L[b][P-k]) / 2
  double Le[((P + 1) / 2 + 1) * ((P + 1) / 2 + 1)];
  double Lo[((P + 1) / 2) * ((P + 1) / 2) + 1];
  int eo;                            // 1: use the even/odd halves (host-checked symmetry)
  double w[P + 1];
  double wasm[P];                    // assembled weight by local index a in [0,p)
};

// Optional (-DSMG_DIFF_SMEM): diffusion with the derivative matrix D staged in
// shared memory (D and D^T, rows padded to an even pitch, read as double2
// broadcasts) instead of the parameter constant bank.  Measured on B200 at
// C5's p = 24 level (151M DOF residual): constant bank 7.9 ms, shared memory
// 13.7 ms (one CTA fewer per SM, shared-memory bandwidth), so the constant
// bank stays the default.
template <int P>
struct DiffTab {
#ifdef SMG_DIFF_SMEM
  static constexpr bool ON = P >= 3;
#else
  static constexpr bool ON = false;
#endif
  static constexpr int NP = P + 1, NPP = (NP + 1) & ~1;
  static constexpr int DOUBLES = ON ? 2 * NP * NPP : 0;
};

template <int P, int TX, int TY, bool DIFF>
struct OpGeom {
  static constexpr int NP = P + 1;
  static constexpr int OX = TX * P, OY = TY * P;
  static constexpr int HX = OX + P + 1, HY = OY + P + 1;
  static constexpr int DP = (HX + 2) & ~1;     // staged row pitch (room for the bulk-copy shift)
  static constexpr int ROWJ = OY * (TX + 1), COLJ = OX * (TY + 1);
  static constexpr int THREADS = (ROWJ > COLJ ? ROWJ : COLJ) >= 256 ? 256 : (((ROWJ > COLJ ? ROWJ : COLJ) + 31) / 32) * 32;
  static constexpr int DTAB = DIFF ? DiffTab<P>::DOUBLES : 0;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)DP * HY * (DIFF ? 2 : 1) + (size_t)OX * OY +
                                                   (size_t)OY * (TX + 1) + (size_t)OX * (TY + 1) + P + DTAB + 2) + 16;
};

// DS[j][b] = D[j][b], DT[k][j] = D[j][k] (pitch NPP, zero padding), from the
// row-major D in the parameter bank; all threads of the CTA call.
template <int P>
__device__ __forceinline__ void diff_tab_fill(const double* Mt, double* DS, int tid, int nt) {
  constexpr int NP = P + 1, NPP = DiffTab<P>::NPP;
  double* DT = DS + NP * NPP;
  for (int i = tid; i < NP * NPP; i += nt) {
    const int r = i / NPP, c = i - r * NPP;
    DS[i] = c < NP ? Mt[r * NP + c] : 0.0;
    DT[i] = c < NP ? Mt[c * NP + r] : 0.0;
  }
}

// 16-byte aligned start for the tables after `after` doubles.
__device__ __forceinline__ double* diff_tab_ptr(double* after) {
  return reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(after) + 15) & ~uintptr_t(15));
}

__device__ __forceinline__ void op_cp_async8(double* smem, const double* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}

// One 1D pass over a line of NP nodes x[0..P] (stride ST in smem):
//   Poisson  : v[b] = sum_k L[k][b] x_k                    (v = L^T x = L x)
//   Diffusion: v[b] = sum_j (nu_j w_j (D x)_j) D[j][b]
// ONLY_LAST: just v[P] (the neighbour element's vertex contribution).
template <int P, bool DIFF, bool ONLY_LAST, int ST>
__device__ __forceinline__ void line_op(const OpArgs<P>& A, const double* x, const double* nu, double (&v)[P + 1]) {
  constexpr int NP = P + 1;
  if (!DIFF && A.eo) {
    // x = sym + antisym: L maps each onto itself (JLJ = L), so with
    // a_k = x_k + x_{P-k}, d_k = x_k - x_{P-k} (and the centre c):
    //   E_b = sum_k Le[b][k] a_k (+ Le[b][H] c),  O_b = sum_k Lo[b][k] d_k,
    //   v_b = E_b + O_b,  v_{P-b} = E_b - O_b   -- half the FMAs
    constexpr int H = NP / 2;
    constexpr bool MID = (NP & 1) != 0;
    constexpr int HC = H + (MID ? 1 : 0);
    double a[H], d[H];
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const double xk = x[k * ST], xm = x[(P - k) * ST];
      a[k] = xk + xm;
      d[k] = xk - xm;
    }
    const double c = MID ? x[H * ST] : 0.0;
    if (ONLY_LAST) {
      double e = MID ? A.Le[H] * c : 0.0, o = 0.0;
#pragma unroll
      for (int k = 0; k < H; ++k) {
        e = fma(A.Le[k], a[k], e);
        o = fma(A.Lo[k], d[k], o);
      }
      v[P] = e - o;
    } else {
      double e[HC], o[H > 0 ? H : 1];
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
  } else if (!DIFF) {
    if (ONLY_LAST) {
      double s = A.Mt[P] * x[0];
#pragma unroll
      for (int k = 1; k < NP; ++k) s = fma(A.Mt[k * NP + P], x[k * ST], s);
      v[P] = s;
    } else {
      const double x0 = x[0];
#pragma unroll
      for (int b = 0; b < NP; ++b) v[b] = A.Mt[b] * x0;
#pragma unroll
      for (int k = 1; k < NP; ++k) {
        const double xk = x[k * ST];
#pragma unroll
        for (int b = 0; b < NP; ++b) v[b] = fma(A.Mt[k * NP + b], xk, v[b]);
      }
    }
  } else {
    double xk[NP], g[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) xk[k] = x[k * ST];
#pragma unroll
    for (int j = 0; j < NP; ++j) g[j] = A.Mt[j * NP] * xk[0];
#pragma unroll
    for (int k = 1; k < NP; ++k)
#pragma unroll
      for (int j = 0; j < NP; ++j) g[j] = fma(A.Mt[j * NP + k], xk[k], g[j]);
#pragma unroll
    for (int j = 0; j < NP; ++j) g[j] *= nu[j * ST] * A.w[j];
    if (ONLY_LAST) {
      double s = g[0] * A.Mt[P];
#pragma unroll
      for (int j = 1; j < NP; ++j) s = fma(g[j], A.Mt[j * NP + P], s);
      v[P] = s;
    } else {
#pragma unroll
      for (int b = 0; b < NP; ++b) v[b] = g[0] * A.Mt[b];
#pragma unroll
      for (int j = 1; j < NP; ++j)
#pragma unroll
        for (int b = 0; b < NP; ++b) v[b] = fma(g[j], A.Mt[j * NP + b], v[b]);
    }
  }
}

// Diffusion line op with the shared-memory tables (same operation order as
// line_op's diffusion branch: bitwise-equal results).  g = D x runs as a
// loop over k (x_k from shared memory, the D^T row as double2 pairs), so only
// the output contraction v = g D is unrolled.
template <int P, bool ONLY_LAST, int ST>
__device__ __forceinline__ void line_op_dsm(const double* __restrict__ w, const double* x, const double* nu,
                                            const double* DS, double (&v)[P + 1]) {
  constexpr int NP = P + 1, NPP = DiffTab<P>::NPP, NH = NP / 2;
  const double* DT = DS + NP * NPP;
  double g[NP];
  {
    const double x0 = x[0];
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      const double2 d = *reinterpret_cast<const double2*>(DT + 2 * j);
      g[2 * j] = d.x * x0;
      g[2 * j + 1] = d.y * x0;
    }
    if (NP & 1) g[NP - 1] = DT[NP - 1] * x0;
  }
#pragma unroll 2
  for (int k = 1; k < NP; ++k) {
    const double xk = x[k * ST];
    const double* dr = DT + k * NPP;
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      const double2 d = *reinterpret_cast<const double2*>(dr + 2 * j);
      g[2 * j] = fma(d.x, xk, g[2 * j]);
      g[2 * j + 1] = fma(d.y, xk, g[2 * j + 1]);
    }
    if (NP & 1) g[NP - 1] = fma(dr[NP - 1], xk, g[NP - 1]);
  }
#pragma unroll
  for (int j = 0; j < NP; ++j) g[j] *= nu[j * ST] * w[j];
  if (ONLY_LAST) {
    const double* dc = DT + P * NPP;   // D[j][P] = DT[P][j]
    double s = g[0] * dc[0];
#pragma unroll
    for (int j = 1; j < NP; ++j) s = fma(g[j], dc[j], s);
    v[P] = s;
  } else {
#pragma unroll
    for (int b = 0; b < NH; ++b) {
      const double2 d = *reinterpret_cast<const double2*>(DS + 2 * b);
      v[2 * b] = g[0] * d.x;
      v[2 * b + 1] = g[0] * d.y;
    }
    if (NP & 1) v[NP - 1] = g[0] * DS[NP - 1];
#pragma unroll
    for (int j = 1; j < NP; ++j) {
      const double* dr = DS + j * NPP;
#pragma unroll
      for (int b = 0; b < NH; ++b) {
        const double2 d = *reinterpret_cast<const double2*>(dr + 2 * b);
        v[2 * b] = fma(g[j], d.x, v[2 * b]);
        v[2 * b + 1] = fma(g[j], d.y, v[2 * b + 1]);
      }
      if (NP & 1) v[NP - 1] = fma(g[j], dr[NP - 1], v[NP - 1]);
    }
  }
}

// line_op, with the diffusion tables from shared memory when DS != nullptr
template <int P, bool DIFF, bool ONLY_LAST, int ST>
__device__ __forceinline__ void line_op_any(const OpArgs<P>& A, const double* x, const double* nu, const double* DS,
                                            double (&v)[P + 1]) {
  if constexpr (DIFF && DiffTab<P>::ON) line_op_dsm<P, ONLY_LAST, ST>(A.w, x, nu, DS, v);
  else line_op<P, DIFF, ONLY_LAST, ST>(A, x, nu, v);
}

template <int P, int TX, int TY, bool DIFF>
__global__ void __launch_bounds__(OpGeom<P, TX, TY, DIFF>::THREADS)
op_kernel(const __grid_constant__ OpArgs<P> A) {
  SMG_PDL_TRIGGER();   // the tables and barrier below are set up while the preceding grid drains
  using G = OpGeom<P, TX, TY, DIFF>;
  constexpr int NP = G::NP, OX = G::OX, OY = G::OY, HX = G::HX, HY = G::HY, NT = G::THREADS;
  extern __shared__ __align__(16) double smo[];
  constexpr int DP = G::DP;
  constexpr int KO = (OX * OY + NT - 1) / NT;     // output nodes per thread
  double* U = smo;                                  // HY x DP, origin (Y0-P, X0-P) at column sh
  double* NU = U + DP * HY;                        // diffusion only
  double* AX = NU + (DIFF ? DP * HY : 0);          // OY x OX: row-pass values, then x+y parts
  double* VX = AX + OX * OY;                       // OY x (TX+1): right-vertex value of element exl-1
  double* VY = VX + OY * (TX + 1);                 // OX x (TY+1)
  double* WS = VY + OX * (TY + 1);                 // P assembled weights (indexed per thread)
  double* DS = diff_tab_ptr(WS + P);               // diffusion: D, D^T tables (G::DTAB doubles)
  uint64_t* bar = reinterpret_cast<uint64_t*>(DS + G::DTAB);
  const int tid = threadIdx.x;
  const int tx = blockIdx.x % A.tiles_x, ty = blockIdx.x / A.tiles_x;
  const int X0 = tx * OX, Y0 = ty * OY;
  const int N_x = A.N_x, N_y = A.N_y;
  if constexpr (G::DTAB > 0) diff_tab_fill<P>(A.Mt, DS, tid, NT);

  int sh = 0;
  if (A.bulk) {
    // bulk row copies issued by warp 0 (periodic wrap handled per row)
    sh = pwin_shift(X0 - P, N_x);
    if (tid == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(bar, pwin_bytes(HX, HY, sh) * (DIFF ? 2u : 1u));
    }
    SMG_PDL_WAIT();
    __syncthreads();
    if (tid < 32) {
      pwin_issue_warp(A.u, N_x, N_y, X0 - P, Y0 - P, HX, HY, U, DP, bar);
      if (DIFF) pwin_issue_warp(A.nu, N_x, N_y, X0 - P, Y0 - P, HX, HY, NU, DP, bar);
    }
  } else {
    SMG_PDL_WAIT();
    for (int idx = tid; idx < HX * HY; idx += NT) {
      const int hy = idx / HX, hx = idx - hy * HX;
      const size_t g = (size_t)wrapi(Y0 - P + hy, N_y) * N_x + wrapi(X0 - P + hx, N_x);
      op_cp_async8(U + hy * DP + hx, A.u + g);
      if (DIFF) op_cp_async8(NU + hy * DP + hx, A.nu + g);
    }
  }
  // f of this thread's output nodes: in flight while the window lands and
  // the line passes run
  double fv[KO];
#pragma unroll
  for (int k = 0; k < KO; ++k) {
    const int idx = tid + k * NT;
    fv[k] = (A.f != nullptr && idx < OX * OY) ? __ldg(A.f + (size_t)(Y0 + idx / OX) * N_x + (X0 + idx % OX)) : 0.0;
  }
  for (int i = tid; i < P; i += NT) WS[i] = A.wasm[i];
  if (A.bulk) mbar_wait(bar, 0);
  else asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();

  // row passes: item = (own row y, element exl-1), exl in [0, TX]
  // full lines (exl >= 1) first, the vertex-only lines (exl == 0) last, so
  // that warps do not diverge between the two
  // one-element tiles (p >= 24): full lines on warp 0, the neighbour's
  // vertex-only lines on warp 1 -- no warp runs both paths one after the
  // other (C5 p = 24 diffusion residual 11.4 -> 7.9 ms on B200)
  constexpr bool SPLIT = TX == 1 && TY == 1 && P <= 32 && NT == 64;
  for (int it0 = tid; it0 < (SPLIT ? NT : OY * (TX + 1)); it0 += NT) {
    const int it = SPLIT ? (tid < 32 ? tid : OY + tid - 32) : it0;
    if (SPLIT && (tid & 31) >= P) continue;
    const bool full = it < OY * TX;
    const int y = full ? it / TX : it - OY * TX, exl = full ? 1 + (it - (it / TX) * TX) : 0;
    const double* ur = U + (y + P) * DP + sh + exl * P;
    const double* nr = NU + (y + P) * DP + sh + exl * P;
    double v[NP];
    if (exl == 0) {
      line_op_any<P, DIFF, true, 1>(A, ur, nr, DS, v);
    } else {
      line_op_any<P, DIFF, false, 1>(A, ur, nr, DS, v);
      double* ax = AX + y * OX + (exl - 1) * P;
#pragma unroll
      for (int b = 0; b < P; ++b) ax[b] = v[b];
    }
    VX[y * (TX + 1) + exl] = v[P];
  }
  __syncthreads();
  // column passes: item = (own column x, element eyl-1), eyl in [0, TY]; each
  // node of the item's column gets its full x-part (with the vertex term of
  // the left element) and its own y-part; the y-vertex term of the element
  // below (a == 0) is added in the output pass
  for (int it0 = tid; it0 < (SPLIT ? NT : OX * (TY + 1)); it0 += NT) {
    const int it = SPLIT ? (tid < 32 ? tid : OX + tid - 32) : it0;
    if (SPLIT && (tid & 31) >= P) continue;
    const bool full = it < OX * TY;
    const int x = full ? it / TY : it - OX * TY, eyl = full ? 1 + (it - (it / TY) * TY) : 0;
    const double* uc = U + (eyl * P) * DP + sh + (x + P);
    const double* nc = NU + (eyl * P) * DP + sh + (x + P);
    double v[NP];
    if (eyl == 0) {
      line_op_any<P, DIFF, true, DP>(A, uc, nc, DS, v);
    } else {
      line_op_any<P, DIFF, false, DP>(A, uc, nc, DS, v);
      const int exl = x / P, b = x - exl * P;
      const double wyb = A.cy * WS[b];
      double* axc = AX + ((eyl - 1) * P) * OX + x;
      const double* vx = VX + ((eyl - 1) * P) * (TX + 1) + exl;
#pragma unroll
      for (int a = 0; a < P; ++a) {
        double ax = axc[a * OX];
        if (b == 0) ax += vx[a * (TX + 1)];
        axc[a * OX] = fma(A.cx * A.wasm[a], ax, wyb * v[a]);
      }
    }
    VY[x * (TY + 1) + eyl] = v[P];
  }
  __syncthreads();

  double nrm = 0.0;
#pragma unroll
  for (int k = 0; k < KO; ++k) {
    const int idx = tid + k * NT;
    if (idx < OX * OY) {
      const int y = idx / OX, x = idx - y * OX;
      const int a = y % P, b = x % P;
      double val = AX[idx];
      if (a == 0) val = fma(A.cy * WS[b], VY[x * (TY + 1) + y / P], val);
      const double r = A.f != nullptr ? fv[k] - val : val;
      A.out[(size_t)(Y0 + y) * N_x + (X0 + x)] = r;
      nrm = fma(r, r, nrm);
    }
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
  int p, n_x, n_y, diffusion;
  double cx, cy;
  const double* Mt;   // host (p+1)^2
  const double* w;    // host p+1
  const double* wasm; // host p
  double* ring = nullptr;   // optional: 2 p doubles per element (halo-free opdh_kernel, smg_opd.cu)
};

// Host: operator constants of OpArgs (everything but the pointers / tiling).
template <int P>
void op_fill_consts(OpArgs<P>& A, const OpLaunch& L, bool diff) {
  A.N_x = L.n_x * P; A.N_y = L.n_y * P;
  A.cx = L.cx; A.cy = L.cy;
  for (int i = 0; i < (P + 1) * (P + 1); ++i) A.Mt[i] = L.Mt[i];
  {
    // even/odd halves of the Poisson stiffness when it is centro-symmetric
    constexpr int NP = P + 1, H = NP / 2, HC = H + (NP & 1);
    auto Lbk = [&](int b, int k) { return L.Mt[k * NP + b]; };
    double asym = 0.0, mx = 0.0;
    for (int b = 0; b < NP; ++b)
      for (int k = 0; k < NP; ++k) {
        asym = std::fmax(asym, std::fabs(Lbk(b, k) - Lbk(P - b, P - k)));
        mx = std::fmax(mx, std::fabs(Lbk(b, k)));
      }
    A.eo = (!diff && asym <= 1e-14 * mx) ? 1 : 0;
    for (int b = 0; b < HC; ++b) {
      for (int k = 0; k < H; ++k) A.Le[b * HC + k] = 0.5 * (Lbk(b, k) + Lbk(b, P - k));
      if (NP & 1) A.Le[b * HC + H] = Lbk(b, H);
    }
    for (int b = 0; b < H; ++b)
      for (int k = 0; k < H; ++k) A.Lo[b * H + k] = 0.5 * (Lbk(b, k) - Lbk(b, P - k));
    A.Lo[H * H] = 0.0;
  }
  for (int i = 0; i < P + 1; ++i) A.w[i] = L.w[i];
  for (int i = 0; i < P; ++i) A.wasm[i] = L.wasm[i];
}

template <int P, int TX, int TY, bool DIFF>
int op_launch_t(const OpLaunch& L, cudaStream_t st) {
  using G = OpGeom<P, TX, TY, DIFF>;
  OpArgs<P> A;
  A.u = L.u; A.f = L.f; A.out = L.out; A.nu = L.nu; A.partials = L.partials;
  op_fill_consts<P>(A, L, DIFF);
  A.tiles_x = L.n_x / TX;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  A.bulk = (A.N_x % 2 == 0) && al16(L.u) && (!DIFF || al16(L.nu)) ? 1 : 0;
  static DeviceFlag attr;
  if (!attr) {
    {  // always: static shared memory adds to the dynamic size
      cudaError_t e = cudaFuncSetAttribute(op_kernel<P, TX, TY, DIFF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)G::SMEM);
      if (e != cudaSuccess) return cuda_fail(e, "op_kernel smem attribute");
    }
    attr = true;
  }
  launch(op_kernel<P, TX, TY, DIFF>, dim3((L.n_x / TX) * (L.n_y / TY)), dim3(G::THREADS), G::SMEM, st, A);
  return check_launch("op_kernel");
}

// FP64 tensor-core diffusion residual for p = 24 (smg_opd.cu) without norm
// partials; returns 1 when not applicable.  frag: device table built from D
// by opd_fragments.
int opd_launch(const OpLaunch& L, const double* frag, cudaStream_t st);
bool opd_applies(int p, bool diffusion);
void opd_fragments(int p, bool diffusion, const double* D, const double* w, std::vector<double>& out);

using OpLaunchFn = int (*)(const OpLaunch&, cudaStream_t);
// Warp-per-element Poisson residual (smg_opw.cu) for p = 8, 16 without norm
// partials; returns 1 when not applicable.
int opw_launch(const OpLaunch& L, cudaStream_t st);
// Poisson p = 32, row warp + column warp per element, halo-free with L.ring (smg_opw.cu)
int opl_launch(const OpLaunch& L, cudaStream_t st);
// out = A u with per-CTA partials of u . out (smg_opw.cu); 1 = not applicable
int opw_apply_dot(const OpLaunch& L, double* partials, int* n_ctas, cudaStream_t st);
int opw_residual_restrict(const OpLaunch& L, const double* J, double* fc, double* rring, cudaStream_t st);
int opdh_apply_dot(const OpLaunch& L, const double* frag, double* ring, double* partials, int* n_ctas,
                   cudaStream_t st);
// Launcher for order p and mesh n_x x n_y (largest compiled tile dividing the
// mesh); *ctas = grid size (number of partials).
OpLaunchFn op_dispatch(int p, bool diffusion, int n_x, int n_y, int* ctas);

}  // namespace smg
