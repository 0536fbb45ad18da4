// Fused residual + restriction: f_c = R (f - A u) in ONE launch.
//
// Reference: restrict_residual (multigrid.py:188-193) applied to
// residual (operators.py:101-103) -- the down-leg step of the V-cycle
// (multigrid.py:243-245).  The two-launch path writes r to HBM and reads it
// back; here a CTA owning a T x T block of coarse elements computes r on the
// fine rows/columns its restriction needs -- the (T+1) x (T+1) elements
// [t0-1, t0+T) of the op_kernel tiling (the extra low-side element supplies
// the coarse vertex terms) -- straight into shared memory, then restricts it
// with the register-blocked passes of restrict_kernel.  r on every node is
// computed by the same instruction sequence as op_kernel, so the result is
// bitwise identical to the two-launch path; the price is the recomputed
// low-side element row/column ((T+1)^2 / T^2 of the residual work).
#pragma once
#include "smg_op.cuh"
#include "smg_transfer.cuh"

namespace smg {

template <int PF>
struct RRArgs {
  OpArgs<PF> op;               // u, f, nu, operator constants (op.out, op.partials unused)
  double* __restrict__ fc;     // coarse output (n_y PC, n_x PC)
  int tiles_x;
  double J[kTrMaxP * 17];      // J[a*(pc+1)+ac]
};

template <int PC, int PF, int T, bool DIFF>
struct RRGeom {
  using OG = OpGeom<PF, T + 1, T + 1, DIFF>;
  static constexpr int NC = PC + 1;
  static constexpr int FX = (T + 1) * PF;   // fine rows/cols of the residual tile (= OG::OX)
  static constexpr int OXC = T * PC;        // coarse own block
  static constexpr int NT = OG::THREADS;
  static constexpr size_t SMEM =
      sizeof(double) * ((size_t)OG::DP * OG::HY * (DIFF ? 2 : 1) + (size_t)FX * FX + 2 * (size_t)FX * (T + 2) + PF +
                        (size_t)FX * OXC + (size_t)FX * (T + 1) + (size_t)OXC * OXC + (size_t)(T + 1) * OXC +
                        OG::DTAB + 2) +
      16;
};

template <int PC, int PF, int T, bool DIFF>
__global__ void __launch_bounds__(RRGeom<PC, PF, T, DIFF>::NT) rr_kernel(const __grid_constant__ RRArgs<PF> R) {
  SMG_PDL_TRIGGER();   // tables and barrier set up while the preceding grid drains; wait before u / nu / f
  using G = RRGeom<PC, PF, T, DIFF>;
  using OG = typename G::OG;
  constexpr int P = PF, TX = T + 1, TY = T + 1, NP = P + 1;
  constexpr int OX = OG::OX, OY = OG::OY, HX = OG::HX, HY = OG::HY, DP = OG::DP, NT = G::NT;
  constexpr int NC = G::NC, FX = G::FX, OXC = G::OXC;
  constexpr int KO = (OX * OY + NT - 1) / NT;
  const OpArgs<PF>& A = R.op;
  extern __shared__ __align__(16) double smr[];
  double* U = smr;                                  // HY x DP window of u (column shift sh)
  double* NU = U + DP * HY;                        // diffusion only
  double* AX = NU + (DIFF ? DP * HY : 0);          // OY x OX: x+y parts, then r
  double* VX = AX + OX * OY;                       // OY x (TX+1)
  double* VY = VX + OY * (TX + 1);                 // OX x (TY+1)
  double* WS = VY + OX * (TY + 1);                 // P assembled weights
  double* Tx = WS + P;                             // FX x OXC (x-restricted)
  double* VT = Tx + FX * OXC;                      // FX x (T+1)
  double* S = VT + FX * (T + 1);                   // OXC x OXC
  double* VC = S + OXC * OXC;                      // (T+1) x OXC
  double* DS = diff_tab_ptr(VC + (T + 1) * OXC);   // diffusion: D, D^T tables
  uint64_t* bar = reinterpret_cast<uint64_t*>(DS + OG::DTAB);
  const int tid = threadIdx.x;
  if constexpr (OG::DTAB > 0) diff_tab_fill<P>(A.Mt, DS, tid, NT);
  const int tx = blockIdx.x % R.tiles_x, ty = blockIdx.x / R.tiles_x;
  const int N_x = A.N_x, N_y = A.N_y;
  // residual tile origin: one element below/left of the coarse block
  const int X0 = (tx * T - 1) * P, Y0 = (ty * T - 1) * P;

  const int sh = pwin_shift(X0 - P, N_x);
  for (int i = tid; i < P; i += NT) WS[i] = A.wasm[i];
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
  double fv[KO];
#pragma unroll
  for (int k = 0; k < KO; ++k) {
    const int idx = tid + k * NT;
    fv[k] = idx < OX * OY ? __ldg(A.f + (size_t)wrapi(Y0 + idx / OX, N_y) * N_x + wrapi(X0 + idx % OX, N_x)) : 0.0;
  }
  mbar_wait(bar, 0);
  __syncthreads();

  // ---- residual (op_kernel's passes on the (T+1)^2-element tile) ----------
  for (int it = tid; it < OY * (TX + 1); it += NT) {
    const int y = it / (TX + 1), exl = it - y * (TX + 1);
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
  for (int it = tid; it < OX * (TY + 1); it += NT) {
    const int x = it / (TY + 1), eyl = it - x * (TY + 1);
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
#pragma unroll
  for (int k = 0; k < KO; ++k) {
    const int idx = tid + k * NT;
    if (idx < OX * OY) {
      const int y = idx / OX, x = idx - y * OX;
      const int a = y % P, b = x % P;
      double val = AX[idx];
      if (a == 0) val = fma(A.cy * WS[b], VY[x * (TY + 1) + y / P], val);
      AX[idx] = fv[k] - val;   // r
    }
  }
  __syncthreads();

  // ---- restriction of r (restrict_kernel's register-blocked passes) -------
  for (int it = tid; it < FX * (T + 1); it += NT) {
    const int yf = it / (T + 1), e = it - yf * (T + 1);
    const double* f = AX + yf * FX + e * PF;
    double s[NC];
    {
      const double f0 = f[0];
#pragma unroll
      for (int ac = 0; ac < NC; ++ac) s[ac] = R.J[ac] * f0;
    }
#pragma unroll
    for (int bb = 1; bb < PF; ++bb) {
      const double fb = f[bb];
#pragma unroll
      for (int ac = 0; ac < NC; ++ac) s[ac] = fma(R.J[bb * NC + ac], fb, s[ac]);
    }
    VT[yf * (T + 1) + e] = s[PC];
    if (e > 0) {
#pragma unroll
      for (int ac = 0; ac < PC; ++ac) Tx[yf * OXC + (e - 1) * PC + ac] = s[ac];
    }
  }
  __syncthreads();
  for (int it = tid; it < (T + 1) * OXC; it += NT) {
    const int e = it / OXC, xc = it - e * OXC;
    const int exl = xc / PC;
    const bool v0 = xc - exl * PC == 0;
    auto tv = [&](int yf) {
      const double v = Tx[yf * OXC + xc];
      return v0 ? v + VT[yf * (T + 1) + exl] : v;
    };
    double s[NC];
    {
      const double t0 = tv(e * PF);
#pragma unroll
      for (int ac = 0; ac < NC; ++ac) s[ac] = R.J[ac] * t0;
    }
#pragma unroll
    for (int a = 1; a < PF; ++a) {
      const double ta = tv(e * PF + a);
#pragma unroll
      for (int ac = 0; ac < NC; ++ac) s[ac] = fma(R.J[a * NC + ac], ta, s[ac]);
    }
    VC[e * OXC + xc] = s[PC];
    if (e > 0) {
#pragma unroll
      for (int ac = 0; ac < PC; ++ac) S[((e - 1) * PC + ac) * OXC + xc] = s[ac];
    }
  }
  __syncthreads();
  const int Nxc = (N_x / PF) * PC;
  for (int idx = tid; idx < OXC * OXC; idx += NT) {
    const int yc = idx / OXC, xc = idx - yc * OXC;
    const int eyl = yc / PC;
    const double v = S[idx];
    R.fc[(size_t)(ty * OXC + yc) * Nxc + (tx * OXC + xc)] = (yc - eyl * PC == 0) ? v + VC[eyl * OXC + xc] : v;
  }
}

struct RRLaunch {
  OpLaunch op;          // u, f, nu, constants (out/partials ignored)
  double* fc;
  const double* J;      // host (pf+1) x (pc+1)
};

template <int PC, int PF, int T, bool DIFF>
int rr_launch_t(const RRLaunch& L, cudaStream_t st) {
  using G = RRGeom<PC, PF, T, DIFF>;
  static_assert(G::SMEM <= 227 * 1024, "fused residual-restriction tile does not fit");
  RRArgs<PF> R;
  R.op.u = L.op.u; R.op.f = L.op.f; R.op.out = nullptr; R.op.nu = L.op.nu; R.op.partials = nullptr;
  op_fill_consts<PF>(R.op, L.op, DIFF);
  R.op.tiles_x = 0;
  R.op.bulk = 1;
  R.fc = L.fc;
  R.tiles_x = L.op.n_x / T;
  for (int i = 0; i < (PF + 1) * (PC + 1); ++i) R.J[i] = L.J[i];
  static DeviceFlag attr;
  if (!attr) {
    {  // always: static shared memory adds to the dynamic size
      cudaError_t e = cudaFuncSetAttribute(rr_kernel<PC, PF, T, DIFF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)G::SMEM);
      if (e != cudaSuccess) return cuda_fail(e, "rr_kernel smem attribute");
    }
    attr = true;
  }
  launch(rr_kernel<PC, PF, T, DIFF>, dim3((L.op.n_x / T) * (L.op.n_y / T)), dim3(G::NT), G::SMEM, st, R);
  return check_launch("rr_kernel");
}

using RRFn = int (*)(const RRLaunch&, cudaStream_t);
// Fused launcher for (p_c, p_f, kind) on an n_x x n_y mesh, or nullptr.
RRFn rr_dispatch(int pc, int pf, bool diffusion, int n_x, int n_y);

}  // namespace smg
