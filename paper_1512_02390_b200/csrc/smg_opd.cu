// Operator residuals on FP64 tensor cores (DMMA), one element per CTA:
// diffusion at p = 24 (C5's top level) and Poisson at p = 32 (C3's).
//
// Poisson lines are the single product V = X . L-hat (no nu, one DMMA
// chain); the rest of this description is the diffusion case.
//
// Reference: DiffusionOperator.apply (operators.py:86-92), residual (:101-103).
// Same gather form as op_kernel (smg_op.cuh): every node row of the element
// (and of its left neighbour, whose vertex value the element's b = 0 column
// needs) is a line x -> v = D^T (nu w . (D x)) along x, every node column a
// line along y, and the two parts meet in shared memory.  Here the lines are
// batched 8 at a time into m8n8k4 DMMAs:
//   G (8 x NP) = X (8 x NP) . D^T      (k padded to 4 KT, n to 8 NTL)
//   G         *= nu(line, node) w(node)
//   V (8 x NP) = G . D                 (G moved from accumulator to operand
//                                        layout by quad shuffles)
// The constant-coefficient-free line op stays FP64-exact per product; the
// summation order differs from op_kernel's, so results agree to rounding
// (the parity tests pin 1e-12 against the reference).  The row/column line
// batches of a pass are split over three warps so that each warp holds one
// batch of full lines and one batch of vertex-only lines.
#include <cstdlib>
#include <vector>

#include "smg_common.cuh"
#include "smg_op.cuh"
#include "smg_tma.cuh"

namespace smg {

template <int P, bool DIFF>
struct OpdGeom {
  static constexpr int NP = P + 1;
  static constexpr int KT = (NP + 3) / 4, NTL = (NP + 7) / 8;
  static constexpr int HX = 2 * P + 1, HY = 2 * P + 1, DP = (HX + 2) & ~1;
  static constexpr int LINES = 2 * P;            // P full lines + P vertex-only lines per pass
  static constexpr int BATCHES = LINES / 8;
  static constexpr int WARPS = BATCHES / 2;
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int FRAG = (DIFF ? 2 : 1) * KT * NTL * 32;   // lane-ordered B fragments: D^T then D (or L)
  static constexpr size_t SMEM =
      sizeof(double) * ((size_t)(DIFF ? 2 : 1) * DP * HY + (size_t)P * P + 2 * (size_t)P + 2 * (size_t)P + P + NP) + 16;
  static_assert(P % 4 == 0 && BATCHES % 2 == 0, "lines must fill whole batches");
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// One batch of 8 lines: line g (lane / 4) starts at x0 (stride ST); its nu at
// n0.  Returns, per n-tile j, V[g][8j + 2t], V[g][8j + 2t + 1] (t = lane % 4).
// ONLY_LAST: only the n-tile holding node P is formed in the second product.
template <int P, bool DIFF, bool ONLY_LAST>
__device__ __forceinline__ void opd_batch(const double* x0, const double* n0, int st, const double* WT,
                                          const double* __restrict__ frag, double (&V)[OpdGeom<P, DIFF>::NTL][2]) {
  using G = OpdGeom<P, DIFF>;
  constexpr int NP = G::NP, KT = G::KT, NTL = G::NTL;
  const int lane = threadIdx.x & 31, t = lane & 3;
  if constexpr (!DIFF) {
    // Poisson: V = X . L (B[k][n] = L[k][n]); vertex lines only the n-tile of node P
    constexpr int J0 = ONLY_LAST ? P / 8 : 0;
#pragma unroll
    for (int j = J0; j < NTL; ++j) V[j][0] = V[j][1] = 0.0;
#pragma unroll
    for (int q = 0; q < KT; ++q) {
      const int k = 4 * q + t;
      const double a = k < NP ? x0[k * st] : 0.0;
#pragma unroll
      for (int j = J0; j < NTL; ++j) dmma(V[j][0], V[j][1], a, __ldg(frag + (q * NTL + j) * 32 + lane));
    }
    return;
  }
  double C[NTL][2];
#pragma unroll
  for (int j = 0; j < NTL; ++j) C[j][0] = C[j][1] = 0.0;
#pragma unroll
  for (int q = 0; q < KT; ++q) {
    const int k = 4 * q + t;
    const double a = k < NP ? x0[k * st] : 0.0;
#pragma unroll
    for (int j = 0; j < NTL; ++j) dmma(C[j][0], C[j][1], a, __ldg(frag + (q * NTL + j) * 32 + lane));
  }
  // G *= nu w (columns n = 8j + 2t + e of line g)
#pragma unroll
  for (int j = 0; j < NTL; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int n = 8 * j + 2 * t + e;
      C[j][e] = n < NP ? C[j][e] * (n0[n * st] * WT[n]) : 0.0;
    }
  constexpr int J0 = ONLY_LAST ? P / 8 : 0;
#pragma unroll
  for (int j = J0; j < NTL; ++j) V[j][0] = V[j][1] = 0.0;
#pragma unroll
  for (int q = 0; q < KT; ++q) {
    // operand A[g][t] = G[g][4q + t], held by lane (g, 2 (q & 1) + t / 2) at element t & 1
    const int src = (lane & ~3) | (2 * (q & 1) + (t >> 1));
    const double v0 = __shfl_sync(0xffffffffu, C[q >> 1][0], src);
    const double v1 = __shfl_sync(0xffffffffu, C[q >> 1][1], src);
    const double a = (t & 1) ? v1 : v0;
#pragma unroll
    for (int j = J0; j < NTL; ++j) dmma(V[j][0], V[j][1], a, __ldg(frag + ((KT + q) * NTL + j) * 32 + lane));
  }
}

// Diffusion batch with the symmetry of the GLL derivative matrix,
// D[P-i][P-j] = -D[i][j]: in terms of a_k = x_k + x_{P-k}, d_k = x_k - x_{P-k}
// (k < H = P/2) and the centre c = x_H,
//   G[n]   = (E a + D[n][H] c) + O d,   G[P-n] = O d - (E a + D[n][H] c),
//   E[n][k] = (D[n][k] + D[n][P-k]) / 2,  O[n][k] = (D[n][k] - D[n][P-k]) / 2
// for n <= H -- two (H+1) x (H+1) products instead of one (P+1) x (P+1), i.e.
// 2 x 16 x 16 instead of 32 x 28 DMMA slots at p = 24; the second product
// (V = g D) splits the same way with a' = g_j + g_{P-j}, d' = g_j - g_{P-j}.
// Returns, for node n = 8j + 2t + e <= H of line g, Vb = V[n] and Vm = V[P-n].
// ONLY_LAST: only the n-tile holding n = 0 (V[P] = Vm[0][0] at t = 0).
template <int P, bool ONLY_LAST>
__device__ __forceinline__ void opd_batch_eo(const double* x0, const double* n0, int st, const double* WT,
                                             const double* __restrict__ frag, double (&Vb)[(P / 2 + 8) / 8][2],
                                             double (&Vm)[(P / 2 + 8) / 8][2]) {
  constexpr int H = P / 2, KH = (H + 1 + 3) / 4, NH = (H + 1 + 7) / 8;
  static_assert(P % 2 == 0, "even order");
  const int lane = threadIdx.x & 31, t = lane & 3;
  const double* BE = frag;
  const double* BO = frag + KH * NH * 32;
  const double* BE2 = frag + 2 * KH * NH * 32;
  const double* BO2 = BE2 + 2 * NH * NH * 32;
  double W[NH][2], U[NH][2];
#pragma unroll
  for (int j = 0; j < NH; ++j) W[j][0] = W[j][1] = U[j][0] = U[j][1] = 0.0;
#pragma unroll
  for (int q = 0; q < KH; ++q) {
    const int k = 4 * q + t;
    const double xa = k <= H ? x0[k * st] : 0.0;
    const double xb = k < H ? x0[(P - k) * st] : 0.0;
    const double a = xa + xb, d = k < H ? xa - xb : 0.0;
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      dmma(W[j][0], W[j][1], a, __ldg(BE + (q * NH + j) * 32 + lane));
      dmma(U[j][0], U[j][1], d, __ldg(BO + (q * NH + j) * 32 + lane));
    }
  }
  // g = G nu w at nodes n and P - n, then a' (centre: g_H) and d'
#pragma unroll
  for (int j = 0; j < NH; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int n = 8 * j + 2 * t + e;
      double ga = 0.0, gd = 0.0;
      if (n <= H) {
        // the GLL weight w[n] = w[P-n] is folded into column n of the first tables
        const double gn = (U[j][e] + W[j][e]) * n0[n * st];
        const double gm = (U[j][e] - W[j][e]) * n0[(P - n) * st];
        ga = n < H ? gn + gm : gn;
        gd = n < H ? gn - gm : 0.0;
      }
      W[j][e] = ga;
      U[j][e] = gd;
    }
  constexpr int J0 = 0, J1 = ONLY_LAST ? 1 : NH;
  double W2[NH][2], U2[NH][2];
#pragma unroll
  for (int j = J0; j < J1; ++j) W2[j][0] = W2[j][1] = U2[j][0] = U2[j][1] = 0.0;
  // k-step q = (n-tile q / 2, slot q % 2): lane t feeds ITS accumulator (node 8 (q/2) + 2t + q%2)
  // as the A operand -- the sum over k is order-free, so the second product's fragment
  // tables are stored in this node order (opd_fragments) and no quad shuffle is needed
#pragma unroll
  for (int q = 0; q < 2 * NH; ++q) {
    const double a = W[q >> 1][q & 1], d = U[q >> 1][q & 1];
#pragma unroll
    for (int j = J0; j < J1; ++j) {
      dmma(W2[j][0], W2[j][1], a, __ldg(BE2 + (q * NH + j) * 32 + lane));
      dmma(U2[j][0], U2[j][1], d, __ldg(BO2 + (q * NH + j) * 32 + lane));
    }
  }
#pragma unroll
  for (int j = J0; j < J1; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      Vb[j][e] = U2[j][e] + W2[j][e];
      Vm[j][e] = U2[j][e] - W2[j][e];
    }
}

// The vertex-only batch (the neighbour's node P) and the full batch of one
// warp in lockstep: their DMMA chains interleave (8 independent accumulator
// chains in the first product instead of 4 -- ncu put the opd warps on
// DMMA-dependency and fragment-load stalls), each fragment load feeds both.
// Same arithmetic as two opd_batch_eo calls.
template <int P>
__device__ __forceinline__ void opd_batch_eo_pair(const double* xv, const double* nv, const double* xf,
                                                  const double* nf, int st, const double* WT,
                                                  const double* __restrict__ frag, double& vlast,
                                                  double (&Vb)[2][2], double (&Vm)[2][2]);

// Compact tables of the halo-free p = 24 kernel (H = P/2 = 12 = 3 x 4): doubles in the
// fragment buffer before them (the opd_batch_eo tables) and their own size.
constexpr int opd_two_offset(int p) {
  const int H = p / 2, KH = (H + 1 + 3) / 4, NH = (H + 1 + 7) / 8;
  return 2 * (KH + 2 * NH) * NH * 32;
}
constexpr int opd_two_doubles(int p) { return 4 * ((p / 2) / 4) * 2 * 32 + 32; }

// Two FULL batches in lockstep (the halo-free kernel: a warp's row batch, stride 1, and
// its column batch, stride stc), every fragment load feeds both.  Returns V[n] (Vb) and
// V[P-n] (Vm) of both batches, n = 8j + 2t + e <= H.
//
// The four half products are 13 x 12 / 12 x 13 (the even halves have the centre as a 13th
// input and no centre output, D[H][H] = 0 and E[.][H] = 0; the odd halves the reverse).
// Padding k to 16 wasted a quarter of the DMMA slots, so here every product runs H / 4 = 3
// k-steps over k < H and the centre input enters as a rank-1 DFMA update.  The first
// product's outputs are placed (by the column order of its tables) where the second
// product wants its k operand: n-tile 0 holds nodes 2t + e, n-tile 1 holds node 8 + t in
// its even columns and the centre output (odd half only) in column 1 -- k-steps
// (0,0), (0,1), (1,0) of the second product are then exactly the nodes < H, no shuffle;
// the centre g_H is broadcast in the quad for the second rank-1 update.
// fr: BE | BO | BE2 | BO2 (3 x 2 x 32 each) | CE1[16] | CE2[16]  (opd_fragments).
template <int P>
__device__ __forceinline__ void opd_batch_eo_two(const double* xr, const double* nr, const double* xc,
                                                 const double* nc, int stc, const double* fr,
                                                 double (&Vb)[2][2][2], double (&Vm)[2][2][2]) {
  constexpr int H = P / 2, KQ = H / 4, NH = 2;
  static_assert(H % 4 == 0 && H + 1 > 8 && H + 1 <= 16, "p = 24 layout");
  const int lane = threadIdx.x & 31, t = lane & 3;
  const double* BE = fr;
  const double* BO = BE + KQ * NH * 32;
  const double* BE2 = BO + KQ * NH * 32;
  const double* BO2 = BE2 + KQ * NH * 32;
  const double* CE1 = BO2 + KQ * NH * 32;
  const double* CE2 = CE1 + 16;
  double W[2][NH][2], U[2][NH][2];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int j = 0; j < NH; ++j) W[s][j][0] = W[s][j][1] = U[s][j][0] = U[s][j][1] = 0.0;
#pragma unroll
  for (int q = 0; q < KQ; ++q) {
    const int k = 4 * q + t;   // < H
    double a[2], d[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const double* x0 = s ? xc : xr;
      const int st = s ? stc : 1;
      const double xa = x0[k * st], xb = x0[(P - k) * st];
      a[s] = xa + xb;
      d[s] = xa - xb;
    }
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      const double be = BE[(q * NH + j) * 32 + lane], bo = BO[(q * NH + j) * 32 + lane];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        dmma(W[s][j][0], W[s][j][1], a[s], be);
        dmma(U[s][j][0], U[s][j][1], d[s], bo);
      }
    }
  }
  // centre input x_H into the even half (slot (1,1) has no even output)
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const double c = (s ? xc : xr)[H * (s ? stc : 1)];
    W[s][0][0] = fma(c, CE1[t], W[s][0][0]);
    W[s][0][1] = fma(c, CE1[4 + t], W[s][0][1]);
    W[s][1][0] = fma(c, CE1[8 + t], W[s][1][0]);
  }
  // g = G nu (w is in the tables) at nodes n and P - n -> a', d'; the centre g_H from slot (1,1) of lane t = 0
  double cp[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const double* n0 = s ? nc : nr;
    const int st = s ? stc : 1;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int j = q >> 1, e = q & 1;
      const int n = j == 0 ? 2 * t + e : 8 + t;
      const double gn = (U[s][j][e] + W[s][j][e]) * n0[n * st];
      const double gm = (U[s][j][e] - W[s][j][e]) * n0[(P - n) * st];
      W[s][j][e] = gn + gm;
      U[s][j][e] = gn - gm;
    }
    cp[s] = __shfl_sync(0xffffffffu, U[s][1][1] * n0[H * st], lane & ~3);
  }
  double W2[2][NH][2], U2[2][NH][2];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int j = 0; j < NH; ++j) W2[s][j][0] = W2[s][j][1] = U2[s][j][0] = U2[s][j][1] = 0.0;
#pragma unroll
  for (int q = 0; q < KQ; ++q) {   // k-step q: the nodes of slot (q / 2, q % 2)
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      const double be = BE2[(q * NH + j) * 32 + lane], bo = BO2[(q * NH + j) * 32 + lane];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        dmma(W2[s][j][0], W2[s][j][1], W[s][q >> 1][q & 1], be);
        dmma(U2[s][j][0], U2[s][j][1], U[s][q >> 1][q & 1], bo);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NH; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const double c2 = CE2[(2 * j + e) * 4 + t];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double w2 = fma(cp[s], c2, W2[s][j][e]);
        Vb[s][j][e] = U2[s][j][e] + w2;
        Vm[s][j][e] = U2[s][j][e] - w2;
      }
    }
}

template <int P>
__device__ __forceinline__ void opd_batch_eo_pair(const double* xv, const double* nv, const double* xf,
                                                  const double* nf, int st, const double* WT,
                                                  const double* __restrict__ frag, double& vlast,
                                                  double (&Vb)[2][2], double (&Vm)[2][2]) {
  constexpr int H = P / 2, KH = (H + 1 + 3) / 4, NH = (H + 1 + 7) / 8;
  static_assert(NH == 2 && P % 2 == 0, "p = 24 layout");
  const int lane = threadIdx.x & 31, t = lane & 3;
  const double* BE = frag;
  const double* BO = frag + KH * NH * 32;
  const double* BE2 = frag + 2 * KH * NH * 32;
  const double* BO2 = BE2 + 2 * NH * NH * 32;
  double W[2][NH][2], U[2][NH][2];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int j = 0; j < NH; ++j) W[s][j][0] = W[s][j][1] = U[s][j][0] = U[s][j][1] = 0.0;
#pragma unroll
  for (int q = 0; q < KH; ++q) {
    const int k = 4 * q + t;
    double a[2], d[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const double* x0 = s ? xf : xv;
      const double xa = k <= H ? x0[k * st] : 0.0;
      const double xb = k < H ? x0[(P - k) * st] : 0.0;
      a[s] = xa + xb;
      d[s] = k < H ? xa - xb : 0.0;
    }
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      const double be = __ldg(BE + (q * NH + j) * 32 + lane), bo = __ldg(BO + (q * NH + j) * 32 + lane);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        dmma(W[s][j][0], W[s][j][1], a[s], be);
        dmma(U[s][j][0], U[s][j][1], d[s], bo);
      }
    }
  }
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const double* n0 = s ? nf : nv;
#pragma unroll
    for (int j = 0; j < NH; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = 8 * j + 2 * t + e;
        double ga = 0.0, gd = 0.0;
        if (n <= H) {
          const double gn = (U[s][j][e] + W[s][j][e]) * n0[n * st];
          const double gm = (U[s][j][e] - W[s][j][e]) * n0[(P - n) * st];
          ga = n < H ? gn + gm : gn;
          gd = n < H ? gn - gm : 0.0;
        }
        W[s][j][e] = ga;
        U[s][j][e] = gd;
      }
  }
  double W2[2][NH][2], U2[2][NH][2];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int j = 0; j < NH; ++j) W2[s][j][0] = W2[s][j][1] = U2[s][j][0] = U2[s][j][1] = 0.0;
#pragma unroll
  for (int q = 0; q < 2 * NH; ++q) {   // node-ordered k-steps (see opd_batch_eo): no quad shuffle
    double a[2], d[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      a[s] = W[s][q >> 1][q & 1];
      d[s] = U[s][q >> 1][q & 1];
    }
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      const double be = __ldg(BE2 + (q * NH + j) * 32 + lane), bo = __ldg(BO2 + (q * NH + j) * 32 + lane);
      if (j == 0) {   // the vertex batch needs only the n-tile holding node 0 (its V[P])
        dmma(W2[0][j][0], W2[0][j][1], a[0], be);
        dmma(U2[0][j][0], U2[0][j][1], d[0], bo);
      }
      dmma(W2[1][j][0], W2[1][j][1], a[1], be);
      dmma(U2[1][j][0], U2[1][j][1], d[1], bo);
    }
  }
  vlast = U2[0][0][0] - W2[0][0][0];
#pragma unroll
  for (int j = 0; j < NH; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      Vb[j][e] = U2[1][j][e] + W2[1][j][e];
      Vm[j][e] = U2[1][j][e] - W2[1][j][e];
    }
}

// Poisson batch with the centro-symmetry L[P-i][P-j] = L[i][j] of L-hat:
//   v[n] = (Ee a + L[H][n] c) + Oo d,   v[P-n] = (Ee a + L[H][n] c) - Oo d,
//   Ee[k][n] = (L[k][n] + L[P-k][n]) / 2,  Oo[k][n] = (L[k][n] - L[P-k][n]) / 2
// (n <= H = P/2): 2 x 20 x 24 DMMA slots per batch instead of 36 x 40 at p = 32.
template <int P, bool ONLY_LAST>
__device__ __forceinline__ void opd_batch_pe(const double* x0, int st, const double* __restrict__ frag,
                                             double (&Vb)[(P / 2 + 8) / 8][2], double (&Vm)[(P / 2 + 8) / 8][2]) {
  constexpr int H = P / 2, KH = (H + 1 + 3) / 4, NH = (H + 1 + 7) / 8;
  const int lane = threadIdx.x & 31, t = lane & 3;
  const double* BE = frag;
  const double* BO = frag + KH * NH * 32;
  constexpr int J1 = ONLY_LAST ? 1 : NH;
  double W[NH][2], U[NH][2];
#pragma unroll
  for (int j = 0; j < J1; ++j) W[j][0] = W[j][1] = U[j][0] = U[j][1] = 0.0;
#pragma unroll
  for (int q = 0; q < KH; ++q) {
    const int k = 4 * q + t;
    const double xa = k <= H ? x0[k * st] : 0.0;
    const double xb = k < H ? x0[(P - k) * st] : 0.0;
    const double a = xa + xb, d = k < H ? xa - xb : 0.0;
#pragma unroll
    for (int j = 0; j < J1; ++j) {
      dmma(W[j][0], W[j][1], a, __ldg(BE + (q * NH + j) * 32 + lane));
      dmma(U[j][0], U[j][1], d, __ldg(BO + (q * NH + j) * 32 + lane));
    }
  }
#pragma unroll
  for (int j = 0; j < J1; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      Vb[j][e] = W[j][e] + U[j][e];
      Vm[j][e] = W[j][e] - U[j][e];
    }
}

template <int P, bool DIFF>
__global__ void __launch_bounds__(OpdGeom<P, DIFF>::THREADS, 5) opd_kernel(const __grid_constant__ OpArgs<P> A,
                                                                        const double* __restrict__ frag) {
  SMG_PDL_TRIGGER();   // barrier + weight tables overlap the preceding grid; wait before u / nu / f
  using G = OpdGeom<P, DIFF>;
  constexpr int NP = G::NP, KT = G::KT, NTL = G::NTL, DP = G::DP, HX = G::HX, HY = G::HY;
  constexpr int OX = P, OY = P, NT = G::THREADS;
  extern __shared__ __align__(16) double smd[];
  double* U = smd;                  // HY x DP window of u (column shift sh)
  double* NU = U + DP * HY;         // same window of nu (diffusion)
  double* AX = NU + (DIFF ? DP * HY : 0);   // OY x OX x-parts, then x+y parts
  double* VX = AX + OX * OY;        // OY x 2: vertex value of the left element's row lines
  double* VY = VX + 2 * OY;         // OX x 2
  double* WS = VY + 2 * OX;         // P assembled weights
  double* WT = WS + P;              // NP GLL weights
  uint64_t* bar = reinterpret_cast<uint64_t*>(WT + NP);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int tx = blockIdx.x % A.tiles_x, ty = blockIdx.x / A.tiles_x;
  const int X0 = tx * OX, Y0 = ty * OY;
  const int N_x = A.N_x, N_y = A.N_y;

  const int sh = pwin_shift(X0 - P, N_x);
  for (int i = tid; i < P; i += NT) WS[i] = A.wasm[i];
  for (int i = tid; i < NP; i += NT) WT[i] = A.w[i];
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, (DIFF ? 2u : 1u) * pwin_bytes(HX, HY, sh));
  }
  SMG_PDL_WAIT();
  __syncthreads();
  if (tid < 32) {
    pwin_issue_warp(A.u, N_x, N_y, X0 - P, Y0 - P, HX, HY, U, DP, bar);
    if (DIFF) pwin_issue_warp(A.nu, N_x, N_y, X0 - P, Y0 - P, HX, HY, NU, DP, bar);
  }
  // f while the window lands (the B fragments stream from the lane-ordered
  // table through L1 inside the batches: 14 KB, shared by the SM's CTAs --
  // held in registers they cost two resident CTAs per SM)
  constexpr int KO = (OX * OY + NT - 1) / NT;
  double fv[KO];
#pragma unroll
  for (int k = 0; k < KO; ++k) {
    const int idx = tid + k * NT;
    fv[k] = (A.f != nullptr && idx < OX * OY) ? __ldg(A.f + (size_t)(Y0 + idx / OX) * N_x + (X0 + idx % OX)) : 0.0;
  }
  mbar_wait(bar, 0);
  __syncthreads();

  // ---- row pass: warp w takes full-line batch w (rows 8w..8w+7 of the
  //      element) and vertex batch w (the same rows of the left neighbour)
  {
    double V[NTL][2];
    const int y = 8 * warp + g;
    const double* ur = U + (y + P) * DP + sh;
    const double* nr = NU + (y + P) * DP + sh;
    if constexpr (DIFF) {
      double Vb[2][2], Vm[2][2], vl;
      // left neighbour (its node P only) and the element's own row lines
      opd_batch_eo_pair<P>(ur, nr, ur + P, nr + P, 1, WT, frag, vl, Vb, Vm);
      if (t == 0) VX[y * 2] = vl;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int b = 8 * j + 2 * t + e;
          if (b <= P / 2) {
            AX[y * OX + b] = Vb[j][e];
            if (b == 0) VX[y * 2 + 1] = Vm[j][e];
            else if (b < P / 2) AX[y * OX + (P - b)] = Vm[j][e];
          }
        }
    } else {
      constexpr int NHO = (P / 2 + 8) / 8;
      double Vb[NHO][2], Vm[NHO][2];
      opd_batch_pe<P, true>(ur, 1, frag, Vb, Vm);   // left neighbour: its node P only
      if (t == 0) VX[y * 2] = Vm[0][0];
      opd_batch_pe<P, false>(ur + P, 1, frag, Vb, Vm);
#pragma unroll
      for (int j = 0; j < NHO; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int b = 8 * j + 2 * t + e;
          if (b <= P / 2) {
            AX[y * OX + b] = Vb[j][e];
            if (b == 0) VX[y * 2 + 1] = Vm[j][e];
            else if (b < P / 2) AX[y * OX + (P - b)] = Vm[j][e];
          }
        }
    }
  }
  __syncthreads();
  // ---- column pass (x-part of the left element added at b == 0) -----------
  {
    double V[NTL][2];
    const int x = 8 * warp + g;
    const double* uc = U + sh + (x + P);
    const double* nc = NU + sh + (x + P);
    const double wyb = A.cy * WS[x];
    auto put = [&](int a, double v) {   // y-part v at node a of column x
      if (a < P) {
        double ax = AX[a * OX + x];
        if (x == 0) ax += VX[a * 2];
        AX[a * OX + x] = fma(A.cx * WS[a], ax, wyb * v);
      } else {
        VY[x * 2 + 1] = v;
      }
    };
    if constexpr (DIFF) {
      double Vb[2][2], Vm[2][2], vl;
      // lower neighbour (its node P only) and the element's own column lines
      opd_batch_eo_pair<P>(uc, nc, uc + P * DP, nc + P * DP, DP, WT, frag, vl, Vb, Vm);
      if (t == 0) VY[x * 2] = vl;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int a = 8 * j + 2 * t + e;
          if (a <= P / 2) {
            put(a, Vb[j][e]);
            if (a < P / 2) put(P - a, Vm[j][e]);
          }
        }
    } else {
      constexpr int NHO = (P / 2 + 8) / 8;
      double Vb[NHO][2], Vm[NHO][2];
      opd_batch_pe<P, true>(uc, DP, frag, Vb, Vm);   // lower neighbour: its node P only
      if (t == 0) VY[x * 2] = Vm[0][0];
      opd_batch_pe<P, false>(uc + P * DP, DP, frag, Vb, Vm);
#pragma unroll
      for (int j = 0; j < NHO; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int a = 8 * j + 2 * t + e;
          if (a <= P / 2) {
            put(a, Vb[j][e]);
            if (a < P / 2) put(P - a, Vm[j][e]);
          }
        }
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KO; ++k) {
    const int idx = tid + k * NT;
    if (idx < OX * OY) {
      const int y = idx / OX, x = idx - y * OX;
      double val = AX[idx];
      if (y == 0) val = fma(A.cy * WS[x], VY[x * 2], val);
      A.out[(size_t)(Y0 + y) * N_x + (X0 + x)] = A.f != nullptr ? fv[k] - val : val;
    }
  }
}

// ---- halo-free variant ------------------------------------------------------
// opd_kernel stages a (2P+1)^2 window (the element and its left / lower /
// corner neighbours) and recomputes the neighbours' row and column lines for
// their node-P vertex value: every u and nu value is read four times from L2
// and the vertex batches cost 75 % of a full batch.  Here a CTA stages only
// its own (P+1)^2 window, runs its P row lines and P column lines (a warp's
// row batch and column batch in lockstep), and hands the node-P value of
// every line to the right / upper neighbour through a ring workspace of 2P
// doubles per element; opdh_fixup subtracts them (adds them for out = A u) at
// the neighbours' low-side nodes with the weights the fused kernel applied,
// in a fixed order (x term, then y term at the corner).
template <int P, bool DIFF>
struct OpdhGeom {
  static constexpr int NP = P + 1;
  // window pitch: even (16-byte rows for the bulk copies); = 12 (mod 16) at p = 24, where the
  // row batch (8 lines x 4 consecutive k) AND the column batch (4 rows k apart x 8 columns) both
  // touch every bank pair exactly twice (pitch 26: three times for the columns; 1592 -> 1554 us)
  static constexpr int DP = P == 24 ? 28 : (NP + 2) & ~1;
  static constexpr int WARPS = P / 8;
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int WIN = ((DP * NP + 15) & ~15);          // one window (doubles), 128-byte multiple
  static constexpr int NWIN = DIFF ? 2 : 1;                    // u (and nu)
  // x-part buffer pitch = 2 (mod 8): the column-wise combine (fixed column, rows 2 t apart
  // across the quad lanes) hits 16 distinct banks per half-warp (pitch P gave 4-way conflicts)
  static constexpr int OXP = P + 2;
  // diffusion: the four fragment tables staged in shared memory (the persistent CTA reads
  // them once per element; as L1-cached global loads they shared the LSU with everything else)
  static constexpr int NFR = DIFF ? opd_two_doubles(P) : 0;
  static constexpr size_t SMEM =
      sizeof(double) * ((size_t)2 * NWIN * WIN + (size_t)P * OXP + (size_t)P + NP + NFR) + 32;
  static_assert(P % 8 == 0, "lines must fill whole batches");
};

// Persistent: a CTA walks elements e = blockIdx.x, + gridDim.x, ... with the NEXT element's
// window in flight (two window buffers, two mbarriers) while the current one is computed --
// one element per CTA spent 35-45 % of its stall samples waiting for its own window.
// DOT (out = A u only): the CTA also accumulates u . (A u) over its elements -- the own
// nodes' parts times the window's u, and the ring values it hands on times u at the
// neighbours' nodes they are destined for (its own window's node-P column and row), with
// the weights opdh_fixup applies -- into A.partials[blockIdx.x] (summed in block order by
// the caller: deterministic for a given grid).
template <int P, bool DIFF, bool DOT = false>
__global__ void __launch_bounds__(OpdhGeom<P, DIFF>::THREADS, DIFF ? 6 : 4)
opdh_kernel(const __grid_constant__ OpArgs<P> A, const double* __restrict__ frag, double* __restrict__ ring,
            int n_el) {
  SMG_PDL_TRIGGER();
  using G = OpdhGeom<P, DIFF>;
  constexpr int NP = G::NP, DP = G::DP, OX = P, OY = P, NT = G::THREADS, WIN = G::WIN, NWIN = G::NWIN, OXP = G::OXP;
  extern __shared__ __align__(128) double smd[];
  double* WB = smd;                          // [2][NWIN] windows: NP x DP of u (and nu), column shift sh
  double* AX = WB + 2 * NWIN * WIN;          // OY x OXP x-parts, then x+y parts
  double* WS = AX + OY * OXP;                // P assembled weights
  double* WT = WS + P;                       // NP GLL weights
  double* FR = WT + NP;                      // NFR fragment doubles (diffusion)
  uint64_t* bar = reinterpret_cast<uint64_t*>(FR + G::NFR);   // [2]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int N_x = A.N_x, N_y = A.N_y;

  for (int i = tid; i < G::NFR; i += NT) FR[i] = frag[opd_two_offset(P) + i];
  for (int i = tid; i < P; i += NT) WS[i] = A.wasm[i];
  for (int i = tid; i < NP; i += NT) WT[i] = A.w[i];
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  SMG_PDL_WAIT();
  __syncthreads();
  // window of element e into buffer b: warp 0 posts the byte count and issues the rows of u,
  // warp 1 those of nu (a copy may complete before the count is posted: the phase cannot end
  // before thread 0's arrival); the buffer's previous readers are past a barrier
  auto issue = [&](int e, int b) {
    const int tx = e % A.tiles_x, ty = e / A.tiles_x;
    const int X0 = tx * OX, Y0 = ty * OY;
    if (tid == 0) mbar_arrive_expect_tx(bar + b, (unsigned)NWIN * pwin_bytes(NP, NP, pwin_shift(X0, N_x)));
    if (warp == 0) pwin_issue_warp(A.u, N_x, N_y, X0, Y0, NP, NP, WB + (b * NWIN) * WIN, DP, bar + b);
    if (DIFF && warp == 1) pwin_issue_warp(A.nu, N_x, N_y, X0, Y0, NP, NP, WB + (b * NWIN + 1) * WIN, DP, bar + b);
  };
  if (warp < 2 && (int)blockIdx.x < n_el) issue(blockIdx.x, 0);

  int it = 0;
  double dacc = 0.0;
  for (int el = blockIdx.x; el < n_el; el += gridDim.x, ++it) {
    const int bsel = it & 1;
    const int tx = el % A.tiles_x, ty = el / A.tiles_x;
    const int X0 = tx * OX, Y0 = ty * OY;
    const int sh = pwin_shift(X0, N_x);
    double* R = ring + (size_t)el * (2 * P);   // [0,P): node-P values of the row lines; [P,2P): column lines
    if (warp < 2 && el + (int)gridDim.x < n_el) issue(el + gridDim.x, bsel ^ 1);
    constexpr int KO = (OX * OY + NT - 1) / NT;
    double fv[KO];
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int idx = tid + k * NT;
      fv[k] = (A.f != nullptr && idx < OX * OY) ? __ldg(A.f + (size_t)(Y0 + idx / OX) * N_x + (X0 + idx % OX)) : 0.0;
    }
    const double* U = WB + (bsel * NWIN) * WIN;
    const double* NU = U + WIN;
    mbar_wait(bar + bsel, (unsigned)(it >> 1) & 1u);

    // warp w: row lines y = 8w..8w+7 and column lines x = 8w..8w+7 of the element
    const int li = 8 * warp + g;          // this lane group's row AND column index
    const double* ur = U + li * DP + sh;
    const double* nr = NU + li * DP + sh;
    const double* uc = U + sh + li;
    const double* nc = NU + sh + li;
    constexpr int NHO = (P / 2 + 8) / 8;
    double Vb[2][NHO][2], Vm[2][NHO][2];   // [0]: row batch, [1]: column batch
    if constexpr (DIFF) {
      opd_batch_eo_two<P>(ur, nr, uc, nc, DP, FR, Vb, Vm);
    } else {
      opd_batch_pe<P, false>(ur, 1, frag, Vb[0], Vm[0]);
      opd_batch_pe<P, false>(uc, DP, frag, Vb[1], Vm[1]);
    }
    // x-parts of the own nodes; the node-P value of the row line goes to the ring
#pragma unroll
    for (int j = 0; j < NHO; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int b = 8 * j + 2 * t + e;
        if (b <= P / 2) {
          AX[li * OXP + b] = Vb[0][j][e];
          if (b == 0) {
            R[li] = Vm[0][j][e];
            if (DOT) dacc = fma(ur[P], (A.cx * WS[li]) * Vm[0][j][e], dacc);
          } else if (b < P / 2) {
            AX[li * OXP + (P - b)] = Vm[0][j][e];
          }
        }
      }
    __syncthreads();   // also: every thread is done with this element's window
    // combine with the y-parts (column li); the node-P value of the column line goes to the ring
    {
      const double wyb = A.cy * WS[li];
      auto put = [&](int a, double v) {
        if (a < P) {
          AX[a * OXP + li] = fma(A.cx * WS[a], AX[a * OXP + li], wyb * v);
        } else {
          R[P + li] = v;
          if (DOT) dacc = fma(uc[P * DP], wyb * v, dacc);
        }
      };
#pragma unroll
      for (int j = 0; j < NHO; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int a = 8 * j + 2 * t + e;
          if (a <= P / 2) {
            put(a, Vb[1][j][e]);
            if (a < P / 2) put(P - a, Vm[1][j][e]);
          }
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int idx = tid + k * NT;
      if (idx < OX * OY) {
        const int y = idx / OX, x = idx - y * OX;
        const double val = AX[y * OXP + x];
        A.out[(size_t)(Y0 + y) * N_x + (X0 + x)] = A.f != nullptr ? fv[k] - val : val;
        if (DOT) dacc = fma(U[y * DP + sh + x], val, dacc);
      }
    }
    __syncthreads();   // AX is rewritten by the next element
  }
  if constexpr (DOT) {
    // CTA total in a fixed order: lanes by xor tree, warps in index order (AX is free)
#pragma unroll
    for (int o = 16; o; o >>= 1) dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
    if (lane == 0) AX[warp] = dacc;
    __syncthreads();
    if (tid == 0) {
      double tsum = 0.0;
      for (int w = 0; w < NT / 32; ++w) tsum += AX[w];
      A.partials[blockIdx.x] = tsum;
    }
  }
}

// Halo-free diffusion kernel for orders whose 2P lines fill whole 8-line batches but whose
// rows alone do not (p = 12: rows 0-7 | rows 8-11 + columns 0-3 | columns 4-11): one batch
// per warp, a lane group's line is a row (stride 1) or a column (stride DP); the x-parts and
// y-parts meet in the final loop.  Same ring layout and fixup as opdh_kernel.
template <int P>
struct OpdqGeom {
  static constexpr int NP = P + 1;
  static constexpr int DP = (NP + 2) & ~1;
  static constexpr int WARPS = 2 * P / 8;
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int WIN = ((DP * NP + 15) & ~15);
  static constexpr int OXP = P + 2;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)4 * WIN + (size_t)2 * P * OXP + (size_t)P + NP) + 32;
  static_assert((2 * P) % 8 == 0, "lines must fill whole batches");
};

template <int P>
__global__ void __launch_bounds__(OpdqGeom<P>::THREADS, P <= 12 ? 8 : 5)
opdq_kernel(const __grid_constant__ OpArgs<P> A, const double* __restrict__ frag, double* __restrict__ ring,
            int n_el) {
  SMG_PDL_TRIGGER();
  using G = OpdqGeom<P>;
  constexpr int NP = G::NP, DP = G::DP, OX = P, OY = P, NT = G::THREADS, WIN = G::WIN, OXP = G::OXP;
  extern __shared__ __align__(128) double smd[];
  double* WB = smd;                    // [2][2] windows: NP x DP of u and nu, column shift sh
  double* AX = WB + 4 * WIN;           // OY x OXP x-parts
  double* AY = AX + OY * OXP;          // OY x OXP y-parts
  double* WS = AY + OY * OXP;          // P assembled weights
  double* WT = WS + P;                 // NP GLL weights
  uint64_t* bar = reinterpret_cast<uint64_t*>(WT + NP);   // [2]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int N_x = A.N_x, N_y = A.N_y;
  for (int i = tid; i < P; i += NT) WS[i] = A.wasm[i];
  for (int i = tid; i < NP; i += NT) WT[i] = A.w[i];
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  SMG_PDL_WAIT();
  __syncthreads();
  auto issue = [&](int e, int b) {
    const int tx = e % A.tiles_x, ty = e / A.tiles_x;
    const int X0 = tx * OX, Y0 = ty * OY;
    if (tid == 0) mbar_arrive_expect_tx(bar + b, 2u * pwin_bytes(NP, NP, pwin_shift(X0, N_x)));
    __syncwarp();
    pwin_issue_warp(A.u, N_x, N_y, X0, Y0, NP, NP, WB + (2 * b) * WIN, DP, bar + b);
    pwin_issue_warp(A.nu, N_x, N_y, X0, Y0, NP, NP, WB + (2 * b + 1) * WIN, DP, bar + b);
  };
  if (warp == 0 && (int)blockIdx.x < n_el) issue(blockIdx.x, 0);
  const int line = 8 * warp + g;            // [0,P): row lines, [P,2P): column lines
  const bool isrow = line < P;
  const int li = isrow ? line : line - P;
  int it = 0;
  for (int el = blockIdx.x; el < n_el; el += gridDim.x, ++it) {
    const int bsel = it & 1;
    const int tx = el % A.tiles_x, ty = el / A.tiles_x;
    const int X0 = tx * OX, Y0 = ty * OY;
    const int sh = pwin_shift(X0, N_x);
    double* R = ring + (size_t)el * (2 * P);
    if (warp == 0 && el + (int)gridDim.x < n_el) issue(el + gridDim.x, bsel ^ 1);
    constexpr int KO = (OX * OY + NT - 1) / NT;
    double fv[KO];
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int idx = tid + k * NT;
      fv[k] = (A.f != nullptr && idx < OX * OY) ? __ldg(A.f + (size_t)(Y0 + idx / OX) * N_x + (X0 + idx % OX)) : 0.0;
    }
    const double* U = WB + (2 * bsel) * WIN;
    const double* NU = U + WIN;
    mbar_wait(bar + bsel, (unsigned)(it >> 1) & 1u);
    constexpr int NHO = (P / 2 + 8) / 8;
    double Vb[NHO][2], Vm[NHO][2];
    const int off = isrow ? li * DP + sh : sh + li;
    opd_batch_eo<P, false>(U + off, NU + off, isrow ? 1 : DP, WT, frag, Vb, Vm);
#pragma unroll
    for (int j = 0; j < NHO; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int b = 8 * j + 2 * t + e;
        if (b <= P / 2) {
          double* dst = isrow ? AX + li * OXP : AY + li;
          const int sb = isrow ? 1 : OXP;
          dst[b * sb] = Vb[j][e];
          if (b == 0) R[line] = Vm[j][e];
          else if (b < P / 2) dst[(P - b) * sb] = Vm[j][e];
        }
      }
    __syncthreads();   // parts complete; every thread is done with this element's window
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int idx = tid + k * NT;
      if (idx < OX * OY) {
        const int y = idx / OX, x = idx - y * OX;
        const double val = fma(A.cx * WS[y], AX[y * OXP + x], (A.cy * WS[x]) * AY[y * OXP + x]);
        A.out[(size_t)(Y0 + y) * N_x + (X0 + x)] = A.f != nullptr ? fv[k] - val : val;
      }
    }
    __syncthreads();   // the parts are rewritten by the next element
  }
}

// The same scheme with one WARP per element (p = 12): opdq_kernel's three warps met at two
// CTA barriers per 144-node element and 45 % of its stall samples sat there (ncu,
// profiles/r2c_opdq12_ncu.txt).  Here a warp owns its element: its own two window buffers
// and mbarriers, its own part buffers, the three batches one after the other, __syncwarp
// instead of CTA barriers; a CTA is just W such warps sharing the weights.
template <int P>
struct OpdwGeom {
  static constexpr int NP = P + 1;
  static constexpr int DP = (NP + 2) & ~1;
  static constexpr int WARPS = 4;
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int NB = 2 * P / 8;                       // batches per element
  static constexpr int WIN = ((DP * NP + 15) & ~15);
  static constexpr int OXP = P + 2;
  static constexpr int PERW = 4 * WIN + 2 * P * OXP;          // doubles per warp (16-byte multiple)
  static constexpr size_t SMEM = sizeof(double) * ((size_t)WARPS * PERW + (size_t)P + NP) + 16 * WARPS + 32;
  static_assert((2 * P) % 8 == 0 && (2 * P * OXP) % 2 == 0, "lines must fill whole batches");
};

template <int P>
__global__ void __launch_bounds__(OpdwGeom<P>::THREADS, 6)
opdw_kernel(const __grid_constant__ OpArgs<P> A, const double* __restrict__ frag, double* __restrict__ ring,
            int n_el) {
  SMG_PDL_TRIGGER();
  using G = OpdwGeom<P>;
  constexpr int NP = G::NP, DP = G::DP, OX = P, OY = P, NT = G::THREADS, WIN = G::WIN, OXP = G::OXP;
  extern __shared__ __align__(128) double smd[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  double* WB = smd + warp * G::PERW;   // [2][2] windows of this warp: NP x DP of u and nu
  double* AX = WB + 4 * WIN;           // OY x OXP x-parts
  double* AY = AX + OY * OXP;          // OY x OXP y-parts
  double* WS = smd + G::WARPS * G::PERW;   // P assembled weights (shared by the warps)
  double* WT = WS + P;                 // NP GLL weights
  uint64_t* bar = reinterpret_cast<uint64_t*>(WT + NP) + 2 * warp;   // [2] per warp
  const int N_x = A.N_x, N_y = A.N_y;
  for (int i = tid; i < P; i += NT) WS[i] = A.wasm[i];
  for (int i = tid; i < NP; i += NT) WT[i] = A.w[i];
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  SMG_PDL_WAIT();
  __syncthreads();
  auto issue = [&](int e, int b) {
    const int tx = e % A.tiles_x, ty = e / A.tiles_x;
    const int X0 = tx * OX, Y0 = ty * OY;
    if (lane == 0) mbar_arrive_expect_tx(bar + b, 2u * pwin_bytes(NP, NP, pwin_shift(X0, N_x)));
    __syncwarp();
    pwin_issue_warp(A.u, N_x, N_y, X0, Y0, NP, NP, WB + (2 * b) * WIN, DP, bar + b);
    pwin_issue_warp(A.nu, N_x, N_y, X0, Y0, NP, NP, WB + (2 * b + 1) * WIN, DP, bar + b);
  };
  const int gw = blockIdx.x * G::WARPS + warp, nw = gridDim.x * G::WARPS;
  if (gw < n_el) issue(gw, 0);
  int it = 0;
  for (int el = gw; el < n_el; el += nw, ++it) {
    const int bsel = it & 1;
    const int tx = el % A.tiles_x, ty = el / A.tiles_x;
    const int X0 = tx * OX, Y0 = ty * OY;
    const int sh = pwin_shift(X0, N_x);
    double* R = ring + (size_t)el * (2 * P);
    // the other buffer's readers (this warp, one element ago) are past a __syncwarp
    if (el + nw < n_el) issue(el + nw, bsel ^ 1);
    const double* U = WB + (2 * bsel) * WIN;
    const double* NU = U + WIN;
    // f at this lane's output nodes, requested before the products (loaded at the store they
    // were 60 % of the kernel's stall samples: five dependent global loads per element)
    constexpr int KO = (OX * OY + 31) / 32;
    double fv[KO];
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int idx = lane + 32 * k;
      fv[k] = (A.f != nullptr && idx < OX * OY) ? __ldg(A.f + (size_t)(Y0 + idx / OX) * N_x + (X0 + idx % OX)) : 0.0;
    }
    mbar_wait(bar + bsel, (unsigned)(it >> 1) & 1u);
#pragma unroll
    for (int bt = 0; bt < G::NB; ++bt) {
      const int line = 8 * bt + g;            // [0,P): row lines, [P,2P): column lines
      const bool isrow = line < P;
      const int li = isrow ? line : line - P;
      constexpr int NHO = (P / 2 + 8) / 8;
      double Vb[NHO][2], Vm[NHO][2];
      const int off = isrow ? li * DP + sh : sh + li;
      opd_batch_eo<P, false>(U + off, NU + off, isrow ? 1 : DP, WT, frag, Vb, Vm);
#pragma unroll
      for (int j = 0; j < NHO; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int b = 8 * j + 2 * t + e;
          if (b <= P / 2) {
            double* dst = isrow ? AX + li * OXP : AY + li;
            const int sb = isrow ? 1 : OXP;
            dst[b * sb] = Vb[j][e];
            if (b == 0) R[line] = Vm[j][e];
            else if (b < P / 2) dst[(P - b) * sb] = Vm[j][e];
          }
        }
    }
    __syncwarp();   // parts complete; the warp is done with this element's window
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int idx = lane + 32 * k;
      if (idx < OX * OY) {
        const int y = idx / OX, x = idx - y * OX;
        const double val = fma(A.cx * WS[y], AX[y * OXP + x], (A.cy * WS[x]) * AY[y * OXP + x]);
        A.out[(size_t)(Y0 + y) * N_x + (X0 + x)] = A.f != nullptr ? fv[k] - val : val;
      }
    }
    __syncwarp();   // the parts are rewritten by the next element
  }
}

// One thread per low-side node of an element: (a, 0) for k = a < P takes the left
// element's row-line value (and, at the corner a = 0, the lower element's column-line
// value after it); (0, b) for k = P + b, b >= 1, the lower element's.
template <int P>
__global__ void __launch_bounds__(256) opdh_fixup(double* __restrict__ out, const double* __restrict__ ring, int n_x,
                                                  int n_y, double cx, double cy, double sign,
                                                  const __grid_constant__ OpArgs<P> A) {
  SMG_PDL_ENTRY();
  const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long)n_x * n_y * 2 * P) return;
  const int e = (int)(gid / (2 * P)), k = (int)(gid - (long)e * (2 * P));
  if (k == P) return;   // the corner is handled by k = 0
  const int ey = e / n_x, ex = e - ey * n_x;
  const int el = ey * n_x + wrapi(ex - 1, n_x), ed = wrapi(ey - 1, n_y) * n_x + ex;
  const int a = k < P ? k : 0, b = k < P ? 0 : k - P;
  double* o = out + (size_t)(ey * P + a) * ((size_t)n_x * P) + ex * P + b;
  double v = *o;
  if (k < P) v = fma(sign * cx * A.wasm[a], ring[(size_t)el * (2 * P) + a], v);
  if (k != 0 && k > P) v = fma(sign * cy * A.wasm[b], ring[(size_t)ed * (2 * P) + P + b], v);
  if (k == 0) v = fma(sign * cy * A.wasm[0], ring[(size_t)ed * (2 * P) + P], v);
  *o = v;
}

template <int P, bool DIFF, bool DOT = false>
static int opdh_launch_t(const OpLaunch& L, const double* frag, double* ring, cudaStream_t st, double* dotp = nullptr,
                         int* n_ctas = nullptr) {
  using G = OpdhGeom<P, DIFF>;
  OpArgs<P> A;
  A.u = L.u; A.f = L.f; A.out = L.out; A.nu = L.nu; A.partials = dotp;
  op_fill_consts<P>(A, L, DIFF);
  A.tiles_x = L.n_x;
  A.bulk = 1;
  static DeviceFlag attr;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(opdh_kernel<P, DIFF, DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    if (e != cudaSuccess) return cuda_fail(e, "opdh_kernel smem attribute");
    attr = true;
  }
  static DeviceInt grid_cap;
  if (grid_cap == 0) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, opdh_kernel<P, DIFF, DOT>, G::THREADS, G::SMEM);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int n_el = L.n_x * L.n_y;
  if (n_ctas) *n_ctas = n_el < grid_cap ? n_el : (int)grid_cap;
  const bool pdl = n_el < kPdlMaxElements;
  launch_pdl(pdl, opdh_kernel<P, DIFF, DOT>, dim3(n_el < grid_cap ? n_el : grid_cap), dim3(G::THREADS), G::SMEM, st, A,
             frag, ring, n_el);
  int rc = check_launch("opdh_kernel");
  if (rc) return rc;
  const long nb = (long)L.n_x * L.n_y * 2 * P;
  launch_pdl(pdl, opdh_fixup<P>, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, st, L.out, (const double*)ring, L.n_x,
             L.n_y, L.cx, L.cy, L.f != nullptr ? -1.0 : 1.0, A);
  return check_launch("opdh_fixup");
}

template <int P>
static int opdw_launch_t(const OpLaunch& L, const double* frag, double* ring, cudaStream_t st) {
  using G = OpdwGeom<P>;
  OpArgs<P> A;
  A.u = L.u; A.f = L.f; A.out = L.out; A.nu = L.nu; A.partials = nullptr;
  op_fill_consts<P>(A, L, true);
  A.tiles_x = L.n_x;
  A.bulk = 1;
  static DeviceInt grid_cap;
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(opdw_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    if (e != cudaSuccess) return cuda_fail(e, "opdw_kernel smem attribute");
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, opdw_kernel<P>, G::THREADS, G::SMEM);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int n_el = L.n_x * L.n_y;
  const int want = (n_el + G::WARPS - 1) / G::WARPS;
  const bool pdl = n_el < kPdlMaxElements;
  launch_pdl(pdl, opdw_kernel<P>, dim3(want < grid_cap ? want : (int)grid_cap), dim3(G::THREADS), G::SMEM, st, A, frag,
             ring, n_el);
  int rc = check_launch("opdw_kernel");
  if (rc) return rc;
  const long nb = (long)n_el * 2 * P;
  launch_pdl(pdl, opdh_fixup<P>, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, st, L.out, (const double*)ring, L.n_x,
             L.n_y, L.cx, L.cy, L.f != nullptr ? -1.0 : 1.0, A);
  return check_launch("opdh_fixup");
}

template <int P>
static int opdq_launch_t(const OpLaunch& L, const double* frag, double* ring, cudaStream_t st) {
  using G = OpdqGeom<P>;
  OpArgs<P> A;
  A.u = L.u; A.f = L.f; A.out = L.out; A.nu = L.nu; A.partials = nullptr;
  op_fill_consts<P>(A, L, true);
  A.tiles_x = L.n_x;
  A.bulk = 1;
  static DeviceInt grid_cap;
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(opdq_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    if (e != cudaSuccess) return cuda_fail(e, "opdq_kernel smem attribute");
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, opdq_kernel<P>, G::THREADS, G::SMEM);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int n_el = L.n_x * L.n_y;
  const bool pdl = n_el < kPdlMaxElements;
  launch_pdl(pdl, opdq_kernel<P>, dim3(n_el < grid_cap ? n_el : grid_cap), dim3(G::THREADS), G::SMEM, st, A, frag, ring,
             n_el);
  int rc = check_launch("opdq_kernel");
  if (rc) return rc;
  const long nb = (long)n_el * 2 * P;
  launch_pdl(pdl, opdh_fixup<P>, dim3((unsigned)((nb + 255) / 256)), dim3(256), 0, st, L.out, (const double*)ring, L.n_x,
             L.n_y, L.cx, L.cy, L.f != nullptr ? -1.0 : 1.0, A);
  return check_launch("opdh_fixup");
}

// Lane-ordered B fragments of D^T and D for opd_kernel (host): value for
// (k-tile q, n-tile j, lane (g, t)) = B[4q + t][8j + g].
void opd_fragments(int p, bool diffusion, const double* D, const double* w, std::vector<double>& out) {
  const int NP = p + 1, KT = (NP + 3) / 4, NTL = (NP + 7) / 8;
  if (diffusion) {
    // even/odd halves (opd_batch_eo): B[k][n] for k, n <= H
    //   E [k][n] = (D[n][k] + D[n][P-k]) / 2 (k < H), E [H][n] = D[n][H]
    //   O [k][n] = (D[n][k] - D[n][P-k]) / 2 (k < H)
    //   E2[k][n] = (D[k][n] + D[P-k][n]) / 2 (k < H), E2[H][n] = D[H][n]
    //   O2[k][n] = (D[k][n] - D[P-k][n]) / 2 (k < H)
    const int H = p / 2, KH = (H + 1 + 3) / 4, NH = (H + 1 + 7) / 8;
    auto d = [&](int i, int j) { return D[i * NP + j]; };
    // first product: k-step q holds k = 4q + t; second product: k-step q holds the node
    // k = 8 (q / 2) + 2t + q % 2 that lane t's accumulator of the first product carries
    const int K2 = 2 * NH;
    out.assign((size_t)2 * (KH + K2) * NH * 32, 0.0);
    for (int m = 0; m < 4; ++m)
      for (int q = 0; q < (m < 2 ? KH : K2); ++q)
        for (int j = 0; j < NH; ++j)
          for (int lane = 0; lane < 32; ++lane) {
            const int k = m < 2 ? 4 * q + (lane & 3) : 8 * (q >> 1) + 2 * (lane & 3) + (q & 1);
            const int n = 8 * j + (lane >> 2);
            double v = 0.0;
            if (k <= H && n <= H) {
              if (m == 0) v = k < H ? 0.5 * (d(n, k) + d(n, p - k)) : d(n, H);
              else if (m == 1) v = k < H ? 0.5 * (d(n, k) - d(n, p - k)) : 0.0;
              // G[n] and G[P-n] are scaled by nu w at their nodes: the (mirror-symmetric) weight goes here
              if (m < 2) v *= 0.5 * (w[n] + w[p - n]);
              else if (m == 2) v = k < H ? 0.5 * (d(k, n) + d(p - k, n)) : d(H, n);
              else v = k < H ? 0.5 * (d(k, n) - d(p - k, n)) : 0.0;
            }
            const size_t base = m < 2 ? (size_t)m * KH : (size_t)2 * KH + (size_t)(m - 2) * K2;
            out[((base + q) * NH + j) * 32 + lane] = v;
          }
    if (H % 4 == 0 && NH == 2) {
      // compact tables of opd_batch_eo_two: H / 4 k-steps over k < H; first-product columns in
      // slot order (n-tile 0: node g; n-tile 1: node 8 + g/2 in the even columns, the centre
      // output in column 1 of the odd half), second-product k rows in the same slot order;
      // then the rank-1 centre vectors CE1 (slot-indexed, weight folded) and CE2
      const int KQ = H / 4;
      const size_t off = out.size();
      if ((int)off != opd_two_offset(p)) std::abort();
      out.resize(off + (size_t)opd_two_doubles(p), 0.0);
      auto node1 = [&](int j, int c) { return j == 0 ? c : (c % 2 == 0 ? 8 + c / 2 : (c == 1 ? H : -1)); };
      auto wsym = [&](int n) { return 0.5 * (w[n] + w[p - n]); };
      for (int m = 0; m < 4; ++m)
        for (int q = 0; q < KQ; ++q)
          for (int j = 0; j < NH; ++j)
            for (int lane = 0; lane < 32; ++lane) {
              const int t = lane & 3, g = lane >> 2;
              double v = 0.0;
              if (m < 2) {
                const int k = 4 * q + t, n = node1(j, g);
                if (n >= 0 && n <= H && !(m == 0 && n == H))
                  v = 0.5 * (m == 0 ? d(n, k) + d(n, p - k) : d(n, k) - d(n, p - k)) * wsym(n);
              } else {
                const int k = q == 0 ? 2 * t : (q == 1 ? 2 * t + 1 : 8 + t), n = 8 * j + g;
                if (n <= H && !(m == 2 && n == H))
                  v = 0.5 * (m == 2 ? d(k, n) + d(p - k, n) : d(k, n) - d(p - k, n));
              }
              out[off + ((size_t)(m * KQ + q) * NH + j) * 32 + lane] = v;
            }
      double* ce1 = out.data() + off + (size_t)4 * KQ * NH * 32;
      double* ce2 = ce1 + 16;
      for (int j = 0; j < 2; ++j)
        for (int e = 0; e < 2; ++e)
          for (int t = 0; t < 4; ++t) {
            const int n1 = (j == 0) ? 2 * t + e : (e == 0 ? 8 + t : -1);
            ce1[(2 * j + e) * 4 + t] = (n1 >= 0 && n1 < H) ? d(n1, H) * wsym(n1) : 0.0;
            const int n2 = 8 * j + 2 * t + e;
            ce2[(2 * j + e) * 4 + t] = n2 < H ? d(H, n2) : 0.0;
          }
    }
    return;
  }
  {
    // Poisson even/odd halves (opd_batch_pe): Ee[k][n] = (L[k][n] + L[P-k][n]) / 2
    // (k < H), Ee[H][n] = L[H][n]; Oo[k][n] = (L[k][n] - L[P-k][n]) / 2
    const int H = p / 2, KH = (H + 1 + 3) / 4, NH = (H + 1 + 7) / 8;
    auto l = [&](int i, int j) { return D[i * NP + j]; };
    out.assign((size_t)2 * KH * NH * 32, 0.0);
    for (int m = 0; m < 2; ++m)
      for (int q = 0; q < KH; ++q)
        for (int j = 0; j < NH; ++j)
          for (int lane = 0; lane < 32; ++lane) {
            const int k = 4 * q + (lane & 3), n = 8 * j + (lane >> 2);
            double v = 0.0;
            if (k <= H && n <= H) {
              if (m == 0) v = k < H ? 0.5 * (l(k, n) + l(p - k, n)) : l(H, n);
              else v = k < H ? 0.5 * (l(k, n) - l(p - k, n)) : 0.0;
            }
            out[((size_t)(m * KH + q) * NH + j) * 32 + lane] = v;
          }
    return;
  }
  out.assign((size_t)(diffusion ? 2 : 1) * KT * NTL * 32, 0.0);
  // diffusion: D^T then D; Poisson: L-hat (B[k][n] = L[k][n], the m = 1 form)
  for (int m = diffusion ? 0 : 1; m < 2; ++m)
    for (int q = 0; q < KT; ++q)
      for (int j = 0; j < NTL; ++j)
        for (int lane = 0; lane < 32; ++lane) {
          const int k = 4 * q + (lane & 3), n = 8 * j + (lane >> 2);
          double v = 0.0;
          if (k < NP && n < NP) v = m == 0 ? D[n * NP + k] : D[k * NP + n];   // D^T[k][n], D[k][n]
          out[((size_t)((diffusion ? m : 0) * KT + q) * NTL + j) * 32 + lane] = v;
        }
}

template <int P, bool DIFF>
static int opd_launch_t(const OpLaunch& L, const double* frag, cudaStream_t st) {
  using G = OpdGeom<P, DIFF>;
  OpArgs<P> A;
  A.u = L.u; A.f = L.f; A.out = L.out; A.nu = L.nu; A.partials = nullptr;
  op_fill_consts<P>(A, L, DIFF);
  A.tiles_x = L.n_x;
  A.bulk = 1;
  static DeviceFlag attr;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(opd_kernel<P, DIFF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    if (e != cudaSuccess) return cuda_fail(e, "opd_kernel smem attribute");
    attr = true;
  }
  launch(opd_kernel<P, DIFF>, dim3(L.n_x * L.n_y), dim3(G::THREADS), G::SMEM, st, A, frag);
  return check_launch("opd_kernel");
}

// (a p = 12 diffusion variant -- 3 warps, full and vertex lines mixed per
// batch -- measured 1016 us vs 839 us for op_kernel<12,2,2> at C5's level 3)
// p = 12 diffusion only has the halo-free kernel (opdq_kernel): it needs the caller's ring
// q = A u and per-CTA partials of u . q in one pass (diffusion p = 24 with the operator ring);
// 1 = not applicable
int opdh_apply_dot(const OpLaunch& L, const double* frag, double* ring, double* partials, int* n_ctas,
                   cudaStream_t st) {
  static const int on = env_int("SMG_OPDH_DOT", 1);
  if (!on || !L.diffusion || L.p != 24 || frag == nullptr || ring == nullptr || L.f != nullptr) return 1;
  return opdh_launch_t<24, true, true>(L, frag, ring, st, partials, n_ctas);
}

bool opd_applies(int p, bool diffusion) { return diffusion ? (p == 24 || p == 12) : p == 32; }

// 1 = not applicable (caller uses op_kernel / opw_kernel)
// SMG_OPD=0 disables the tensor-core operator path (read once).
static bool opd_enabled() {
  static const bool on = env_int("SMG_OPD", 1) != 0;
  return on;
}

int opd_launch(const OpLaunch& L, const double* frag, cudaStream_t st) {
  if (!opd_applies(L.p, L.diffusion != 0) || L.partials != nullptr || frag == nullptr || !opd_enabled())
    return 1;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if ((L.n_x * L.p) % 2 != 0 || !al16(L.u) || (L.diffusion && !al16(L.nu))) return 1;
  // halo-free kernel + fixup when the caller passes a ring workspace (SMG_OPDH=0 keeps the fused kernel)
  static const bool hf = env_int("SMG_OPDH", 1) != 0;
  if (L.p == 12) {
    static const bool q12 = env_int("SMG_OPDQ", 1) != 0;
    static const bool w12 = env_int("SMG_OPDW", 1) != 0;   // warp per element (0: a CTA of three warps)
    if (L.ring != nullptr && hf && q12 && w12) return opdw_launch_t<12>(L, frag, L.ring, st);
    return (L.ring != nullptr && hf && q12) ? opdq_launch_t<12>(L, frag, L.ring, st) : 1;
  }
  // tuning aid: one batch per warp at p = 24 (6 warps, 64 registers, 5 CTAs/SM): measured
  // 2063 us vs 1955 us for the lockstep row+column batches of opdh_kernel at C5
  static const int q24 = env_int("SMG_OPDQ24", 0);
  if (L.ring != nullptr && hf && L.diffusion && q24) return opdq_launch_t<24>(L, frag, L.ring, st);
  if (L.ring != nullptr && hf)
    return L.diffusion ? opdh_launch_t<24, true>(L, frag, L.ring, st) : opdh_launch_t<32, false>(L, frag, L.ring, st);
  return L.diffusion ? opd_launch_t<24, true>(L, frag, st) : opd_launch_t<32, false>(L, frag, st);
}

}  // namespace smg
