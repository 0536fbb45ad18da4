// p-multigrid transfers (subsystem 3).
//
// Reference: prolongate / restrict_residual (multigrid.py:180-193) multiply
// by dense global 1D matrices P_y, P_x (multigrid.py:112-124) whose rows
// are ASSIGNED per element (a fine vertex node appears once).  Here both are
// element-local, separable (x pass then y pass) with the (p_f+1) x (p_c+1)
// interpolation matrix J, in gather form -- one thread per output entry:
//   prolongation : fine node (a,b) owned by element e (0 <= a,b < p_f)
//                  u_f += sum_{ac,bc} J[a][ac] U_c,e[ac][bc] J[b][bc]
//   restriction  : owner-computes over fine rows/cols b < p_f of every
//                  element (so shared fine nodes count once, exactly as in
//                  P^T); coarse vertex ac = 0 also collects element e-1's
//                  ac = p_c term, added in a fixed order.
// Deterministic, no atomics.  Tiles are compile-time; data is staged with
// cp.async and J lives in shared memory.
#include "smg_transfer.cuh"
#include "smg_tma.cuh"

namespace smg {

__device__ __forceinline__ void tr_cp_async8(double* smem, const double* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}

template <int PC, int PF, int T>
struct TrGeom {
  static constexpr int NC = PC + 1, NF = PF + 1;
  // prolongation: coarse region incl. high vertex, fine own tile
  static constexpr int CX = T * PC + 1, OXF = T * PF;
  static constexpr int DC = (CX + 2) & ~1, DF = (OXF + 2) & ~1;   // staged row pitches
  // restriction: fine staged incl. the low halo element, coarse own tile
  static constexpr int FX = (T + 1) * PF, OXC = T * PC;
  static constexpr int DX = (FX + 2) & ~1;
  static constexpr int NT = 256;
  static constexpr size_t SMEM_P = sizeof(double) * ((size_t)DC * CX + (size_t)CX * OXF + (size_t)DF * OXF) + 16;
  static constexpr size_t SMEM_R = sizeof(double) * ((size_t)DX * FX + (size_t)FX * OXC + (size_t)FX * (T + 1) +
                                                     (size_t)OXC * OXC + (size_t)(T + 1) * OXC) + 16;
};

template <int PC, int PF, int T>
__global__ void __launch_bounds__(256) prolong_kernel(const __grid_constant__ TrArgs A) {
  SMG_PDL_ENTRY();
  using G = TrGeom<PC, PF, T>;
  constexpr int NC = G::NC, NF = G::NF, CX = G::CX, OX = G::OXF, NT = G::NT;
  extern __shared__ __align__(16) double sm[];
  constexpr int DC = G::DC, DF = G::DF;
  double* C = sm;             // CX x DC coarse values (column shift shc)
  double* Tt = C + DC * CX;   // CX x OX  (x-interpolated)
  double* UF = Tt + CX * OX;  // OX x DF  old fine values (accumulate; column shift shf)
  uint64_t* bar = reinterpret_cast<uint64_t*>(UF + DF * OX);
  const int tid = threadIdx.x;
  const int tx = blockIdx.x % A.tiles_x, ty = blockIdx.x / A.tiles_x;
  const int Nxc = A.n_x * PC, Nyc = A.n_y * PC, Nxf = A.n_x * PF, Nyf = A.n_y * PF;
  const int Xc0 = tx * T * PC, Yc0 = ty * T * PC, Xf0 = tx * OX, Yf0 = ty * OX;
  int shc = 0, shf = 0;
  if (A.bulk) {
    shc = pwin_shift(Xc0, Nxc);
    shf = pwin_shift(Xf0, Nxf);
    if (tid == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(bar, pwin_bytes(CX, CX, shc) + (A.accumulate ? pwin_bytes(OX, OX, shf) : 0u));
    }
    __syncthreads();
    if (tid < 32) {
      pwin_issue_warp(A.src, Nxc, Nyc, Xc0, Yc0, CX, CX, C, DC, bar);
      if (A.accumulate) pwin_issue_warp(A.dst, Nxf, Nyf, Xf0, Yf0, OX, OX, UF, DF, bar);
    }
  } else {
    for (int idx = tid; idx < CX * CX; idx += NT) {
      const int y = idx / CX, x = idx - y * CX;
      tr_cp_async8(C + y * DC + x, A.src + (size_t)wrapi(Yc0 + y, Nyc) * Nxc + wrapi(Xc0 + x, Nxc));
    }
    if (A.accumulate) {
      for (int idx = tid; idx < OX * OX; idx += NT) {
        const int y = idx / OX, x = idx - y * OX;
        tr_cp_async8(UF + y * DF + x, A.dst + (size_t)(Yf0 + y) * Nxf + (Xf0 + x));
      }
    }
  }
  if (A.bulk) mbar_wait(bar, 0);
  else asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  // Register-blocked passes: a thread owns one (line, element) and produces
  // all of its outputs, so every J entry is a uniform parameter-bank operand
  // and each staged value is read from shared memory once.
  // x: Tt[rc][exl*PF + b] = sum_bc J[b][bc] C[rc][exl*PC + bc]
  for (int it = tid; it < CX * T; it += NT) {
    const int rc = it / T, exl = it - rc * T;
    const double* c = C + rc * DC + shc + exl * PC;
    double cv[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) cv[k] = c[k];
    double* out = Tt + rc * OX + exl * PF;
#pragma unroll
    for (int bb = 0; bb < PF; ++bb) {
      double s = A.J[bb * NC] * cv[0];
#pragma unroll
      for (int k = 1; k < NC; ++k) s = fma(A.J[bb * NC + k], cv[k], s);
      out[bb] = s;
    }
  }
  __syncthreads();
  // y: out[eyl*PF + a][xf] = sum_ac J[a][ac] Tt[eyl*PC + ac][xf]
  for (int it = tid; it < T * OX; it += NT) {
    const int eyl = it / OX, xf = it - eyl * OX;
    const double* t = Tt + (eyl * PC) * OX + xf;
    double tv[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) tv[k] = t[k * OX];
#pragma unroll
    for (int a = 0; a < PF; ++a) {
      double s = A.J[a * NC] * tv[0];
#pragma unroll
      for (int k = 1; k < NC; ++k) s = fma(A.J[a * NC + k], tv[k], s);
      const int yf = eyl * PF + a;
      A.dst[(size_t)(Yf0 + yf) * Nxf + (Xf0 + xf)] = A.accumulate ? UF[yf * DF + shf + xf] + s : s;
    }
  }
}

template <int PC, int PF, int T>
__global__ void __launch_bounds__(256) restrict_kernel(const __grid_constant__ TrArgs A) {
  SMG_PDL_ENTRY();
  using G = TrGeom<PC, PF, T>;
  constexpr int NC = G::NC, NF = G::NF, FX = G::FX, OX = G::OXC, NT = G::NT;
  extern __shared__ __align__(16) double sm[];
  constexpr int DX = G::DX;
  double* F = sm;              // FX x DX fine own rows/cols of elements [t0-1, t0+T) (column shift shx)
  double* Tx = F + DX * FX;    // FX x OX  (x-restricted)
  double* VT = Tx + FX * OX;   // FX x (T+1) vertex terms of the x pass
  double* S = VT + FX * (T + 1);  // OX x OX  (y-restricted, before the vertex terms)
  double* VY = S + OX * OX;    // (T+1) x OX vertex terms of the y pass
  uint64_t* bar = reinterpret_cast<uint64_t*>(VY + (T + 1) * OX);
  const int tid = threadIdx.x;
  const int tx = blockIdx.x % A.tiles_x, ty = blockIdx.x / A.tiles_x;
  const int Nxf = A.n_x * PF, Nyf = A.n_y * PF, Nxc = A.n_x * PC;
  const int Xf0 = (tx * T - 1) * PF, Yf0 = (ty * T - 1) * PF;
  int shx = 0;
  if (A.bulk) {
    shx = pwin_shift(Xf0, Nxf);
    if (tid == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(bar, pwin_bytes(FX, FX, shx));
    }
    __syncthreads();
    if (tid < 32) pwin_issue_warp(A.src, Nxf, Nyf, Xf0, Yf0, FX, FX, F, DX, bar);
  } else {
    for (int idx = tid; idx < FX * FX; idx += NT) {
      const int y = idx / FX, x = idx - y * FX;
      tr_cp_async8(F + y * DX + x, A.src + (size_t)wrapi(Yf0 + y, Nyf) * Nxf + wrapi(Xf0 + x, Nxf));
    }
  }
  if (A.bulk) mbar_wait(bar, 0);
  else asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  // Register-blocked passes (see prolong_kernel).  Element e in [0, T] of
  // the staged fine rows is tile element e-1 (e = 0: the left/lower halo
  // element, which only contributes its ac = PC vertex term).
  // x: s[ac] = sum_{b<PF} J[b][ac] F[yf][e PF + b]; the coarse vertex ac = 0
  //    of element e-1 later adds element e-2's ac = PC term (VT)
  for (int it = tid; it < FX * (T + 1); it += NT) {
    const int yf = it / (T + 1), e = it - yf * (T + 1);
    const double* f = F + yf * DX + shx + e * PF;
    double s[NC];
    {
      const double f0 = f[0];
#pragma unroll
      for (int ac = 0; ac < NC; ++ac) s[ac] = A.J[ac] * f0;
    }
#pragma unroll
    for (int bb = 1; bb < PF; ++bb) {
      const double fb = f[bb];
#pragma unroll
      for (int ac = 0; ac < NC; ++ac) s[ac] = fma(A.J[bb * NC + ac], fb, s[ac]);
    }
    VT[yf * (T + 1) + e] = s[PC];
    if (e > 0) {
#pragma unroll
      for (int ac = 0; ac < PC; ++ac) Tx[yf * OX + (e - 1) * PC + ac] = s[ac];
    }
  }
  __syncthreads();
  // y: same along columns on the vertex-combined rows Tx[yf][xc] (+ VT at ac = 0)
  for (int it = tid; it < (T + 1) * OX; it += NT) {
    const int e = it / OX, xc = it - e * OX;
    const int exl = xc / PC;
    const bool v0 = xc - exl * PC == 0;
    auto tv = [&](int yf) {
      const double v = Tx[yf * OX + xc];
      return v0 ? v + VT[yf * (T + 1) + exl] : v;
    };
    double s[NC];
    {
      const double t0 = tv(e * PF);
#pragma unroll
      for (int ac = 0; ac < NC; ++ac) s[ac] = A.J[ac] * t0;
    }
#pragma unroll
    for (int a = 1; a < PF; ++a) {
      const double ta = tv(e * PF + a);
#pragma unroll
      for (int ac = 0; ac < NC; ++ac) s[ac] = fma(A.J[a * NC + ac], ta, s[ac]);
    }
    VY[e * OX + xc] = s[PC];
    if (e > 0) {
#pragma unroll
      for (int ac = 0; ac < PC; ++ac) S[((e - 1) * PC + ac) * OX + xc] = s[ac];
    }
  }
  __syncthreads();
  for (int idx = tid; idx < OX * OX; idx += NT) {
    const int yc = idx / OX, xc = idx - yc * OX;
    const int eyl = yc / PC;
    const double v = S[idx];
    A.dst[(size_t)(ty * OX + yc) * Nxc + (tx * OX + xc)] = (yc - eyl * PC == 0) ? v + VY[eyl * OX + xc] : v;
  }
}

template <int PC, int PF, int T>
int tr_launch_t(const TrArgs& A0, bool prolong, cudaStream_t st) {
  using G = TrGeom<PC, PF, T>;
  TrArgs A = A0;
  A.tiles_x = A.n_x / T;
  {
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    const int nxc = A.n_x * PC, nxf = A.n_x * PF;
    A.bulk = (nxc % 2 == 0) && (nxf % 2 == 0) && al16(A.src) && al16(A.dst) ? 1 : 0;
  }
  const int grid = (A.n_x / T) * (A.n_y / T);
  if (prolong) {
    static DeviceFlag attr;
    if (!attr && G::SMEM_P > 48 * 1024)
      cudaFuncSetAttribute(prolong_kernel<PC, PF, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM_P);
    attr = true;
    launch(prolong_kernel<PC, PF, T>, dim3(grid), dim3(G::NT), G::SMEM_P, st, A);
  } else {
    static DeviceFlag attr;
    if (!attr && G::SMEM_R > 48 * 1024)
      cudaFuncSetAttribute(restrict_kernel<PC, PF, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM_R);
    attr = true;
    launch(restrict_kernel<PC, PF, T>, dim3(grid), dim3(G::NT), G::SMEM_R, st, A);
  }
  return check_launch(prolong ? "prolong_kernel" : "restrict_kernel");
}

// ---- warp-per-element transfers (power-of-two p_f <= 16) ---------------------
// One warp owns one element and works without block-level barriers, so the
// warps of an SM overlap their load / compute / store phases (the tiled
// kernels above serialise them behind __syncthreads with few busy threads).
constexpr int kTrWarps = 8;

// prolongation, fine element e: u_f[e][a][b] (+)= sum J[a][ay] C[ay][ax] J[b][ax]
template <int PC, int PF>
__global__ void __launch_bounds__(32 * kTrWarps) prolong_warp_kernel(const __grid_constant__ TrArgs A) {
  SMG_PDL_TRIGGER();
  constexpr int NC = PC + 1;
  static_assert(32 % PF == 0 || PF % 32 == 0, "p_f must divide the warp");
  constexpr int LPR = PF < 32 ? 32 / PF : 1;     // output rows per warp instruction
  __shared__ double Js[(PF + 1) * NC];
  __shared__ double Cw[kTrWarps][NC * NC];
  __shared__ double Tw[kTrWarps][NC * PF];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (PF + 1) * NC; i += 32 * kTrWarps) Js[i] = A.J[i];
  const int e = blockIdx.x * kTrWarps + warp;
  const int n_el = A.n_x * A.n_y;
  const int ey = e / A.n_x, ex = e - ey * A.n_x;
  const int Nxc = A.n_x * PC, Nyc = A.n_y * PC, Nxf = A.n_x * PF;
  const bool act = e < n_el;
  SMG_PDL_WAIT();   // J (a parameter) is staged above while the preceding grid drains
  // coarse element values (with the high-side shared nodes)
  if (act) {
    for (int i = lane; i < NC * NC; i += 32) {
      const int ay = i / NC, ax = i - ay * NC;
      Cw[warp][i] = A.src[(size_t)wrapi(ey * PC + ay, Nyc) * Nxc + wrapi(ex * PC + ax, Nxc)];
    }
  }
  // old fine values (accumulate)
  constexpr int NO = (PF * PF + 31) / 32;
  double old[NO];
  const int b = lane % PF;
#pragma unroll
  for (int k = 0; k < NO; ++k) {
    const int a = lane / PF + LPR * k;
    old[k] = (act && A.accumulate && a < PF) ? A.dst[(size_t)(ey * PF + a) * Nxf + ex * PF + b] : 0.0;
  }
  __syncthreads();   // Js (once per block)
  if (!act) return;
  // x pass: Tt[ay][b] = sum_ax J[b][ax] C[ay][ax]; lane's b is fixed
  {
    double jb[NC];
#pragma unroll
    for (int ax = 0; ax < NC; ++ax) jb[ax] = Js[b * NC + ax];
    for (int o = lane; o < NC * PF; o += 32) {
      const int ay = o / PF;
      const double* c = &Cw[warp][ay * NC];
      double s = 0.0;
#pragma unroll
      for (int ax = 0; ax < NC; ++ax) s = fma(jb[ax], c[ax], s);
      Tw[warp][ay * PF + b] = s;
    }
  }
  __syncwarp();
  // y pass: out[a][b] = sum_ay J[a][ay] Tt[ay][b]
  double tb[NC];
#pragma unroll
  for (int ay = 0; ay < NC; ++ay) tb[ay] = Tw[warp][ay * PF + b];
#pragma unroll
  for (int k = 0; k < NO; ++k) {
    const int a = lane / PF + LPR * k;
    if (a < PF) {
      double s = 0.0;
#pragma unroll
      for (int ay = 0; ay < NC; ++ay) s = fma(Js[a * NC + ay], tb[ay], s);
      A.dst[(size_t)(ey * PF + a) * Nxf + ex * PF + b] = A.accumulate ? old[k] + s : s;
    }
  }
}

// prolongation for p_f that does not divide the warp (p_f = 3, 6, 12, 24):
// lane b < p_f owns fine column b of the element (x pass over the coarse
// rows with its J row in registers, then all p_f rows of its column; the
// rows are written coalesced across the lanes).  Same sums as the tiled
// kernel's gather form.
template <int PC, int PF>
__global__ void __launch_bounds__(32 * kTrWarps, 2) prolong_warp_g_kernel(const __grid_constant__ TrArgs A) {
  SMG_PDL_ENTRY();
  constexpr int NC = PC + 1;
  static_assert(PF <= 32, "one lane per fine column");
  __shared__ double Js[(PF + 1) * NC];
  __shared__ double Cw[kTrWarps][NC * NC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (PF + 1) * NC; i += 32 * kTrWarps) Js[i] = A.J[i];
  const int e = blockIdx.x * kTrWarps + warp;
  const int n_el = A.n_x * A.n_y;
  const int ey = e / A.n_x, ex = e - ey * A.n_x;
  const int Nxc = A.n_x * PC, Nyc = A.n_y * PC, Nxf = A.n_x * PF;
  const bool act = e < n_el;
  SMG_PDL_WAIT();   // J (a parameter) is staged above while the preceding grid drains
  if (act) {
    for (int i = lane; i < NC * NC; i += 32) {
      const int ay = i / NC, ax = i - ay * NC;
      Cw[warp][i] = A.src[(size_t)wrapi(ey * PC + ay, Nyc) * Nxc + wrapi(ex * PC + ax, Nxc)];
    }
  }
  const int b = lane;
  const bool lb = act && b < PF;
  double old[PF];
  double* out = A.dst + (size_t)(ey * PF) * Nxf + ex * PF + b;
#pragma unroll
  for (int a = 0; a < PF; ++a) old[a] = (lb && A.accumulate) ? out[(size_t)a * Nxf] : 0.0;
  __syncthreads();   // Js (once per block), Cw of this warp
  if (!lb) return;
  // x pass: t[ay] = sum_ax J[b][ax] C[ay][ax]
  double jb[NC], tb[NC];
#pragma unroll
  for (int ax = 0; ax < NC; ++ax) jb[ax] = Js[b * NC + ax];
#pragma unroll
  for (int ay = 0; ay < NC; ++ay) {
    const double* c = &Cw[warp][ay * NC];
    double s = 0.0;
#pragma unroll
    for (int ax = 0; ax < NC; ++ax) s = fma(jb[ax], c[ax], s);
    tb[ay] = s;
  }
  // y pass: out[a][b] = sum_ay J[a][ay] t[ay]
#pragma unroll
  for (int a = 0; a < PF; ++a) {
    double s = 0.0;
#pragma unroll
    for (int ay = 0; ay < NC; ++ay) s = fma(Js[a * NC + ay], tb[ay], s);
    out[(size_t)a * Nxf] = A.accumulate ? old[a] + s : s;
  }
}

// restriction, coarse element e: owned coarse nodes (ay, ax < p_c) from the
// fine blocks of elements e, e-x, e-y, e-xy (row-assigned P^T, as the tiled
// kernel): x pass over the 2p_f fine rows, then y pass.
template <int PF>
constexpr int tr_rwarps() { return PF >= 16 ? 4 : kTrWarps; }

template <int PC, int PF>
__global__ void __launch_bounds__(32 * tr_rwarps<PF>()) restrict_warp_kernel(const __grid_constant__ TrArgs A) {
  SMG_PDL_ENTRY();
  constexpr int NC = PC + 1, R2 = 2 * PF, LD = R2 + 1, RW = tr_rwarps<PF>();
  static_assert(R2 <= 32, "fine region rows per warp");
  __shared__ double Js[(PF + 1) * NC];
  __shared__ double Fw[RW][R2 * LD];
  __shared__ double Hw[RW][R2 * PC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (PF + 1) * NC; i += 32 * RW) Js[i] = A.J[i];
  const int e = blockIdx.x * RW + warp;
  const int n_el = A.n_x * A.n_y;
  const int ey = e / A.n_x, ex = e - ey * A.n_x;
  const int Nxf = A.n_x * PF, Nyf = A.n_y * PF, Nxc = A.n_x * PC;
  const bool act = e < n_el;
  if (act) {
    // fine rows/cols [e*PF - PF, e*PF + PF): R2 x R2 values, lanes along rows
    constexpr int NL = (R2 * R2 + 31) / 32;
    double v[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const int i = lane + 32 * k, ry = i / R2, rx = i - ry * R2;
      v[k] = i < R2 * R2 ? A.src[(size_t)wrapi(ey * PF - PF + ry, Nyf) * Nxf + wrapi(ex * PF - PF + rx, Nxf)] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const int i = lane + 32 * k, ry = i / R2, rx = i - ry * R2;
      if (i < R2 * R2) Fw[warp][ry * LD + rx] = v[k];
    }
  }
  __syncthreads();   // Js (once per block); Fw of this warp
  if (!act) return;
  // x pass: H[ry][ax] = sum_bx J[bx][ax] F[ry][PF+bx] (+ for ax = 0 the left
  // element's vertex term sum_bx J[bx][PC] F[ry][bx]); lane = fine row
  for (int ry = lane; ry < R2; ry += 32) {
    const double* f = &Fw[warp][ry * LD];
    double s[PC];
#pragma unroll
    for (int ax = 0; ax < PC; ++ax) s[ax] = 0.0;
    double vt = 0.0;
#pragma unroll
    for (int bx = 0; bx < PF; ++bx) {
      const double fo = f[PF + bx], fl = f[bx];
#pragma unroll
      for (int ax = 0; ax < PC; ++ax) s[ax] = fma(A.J[bx * NC + ax], fo, s[ax]);
      vt = fma(A.J[bx * NC + PC], fl, vt);
    }
    s[0] += vt;
#pragma unroll
    for (int ax = 0; ax < PC; ++ax) Hw[warp][ry * PC + ax] = s[ax];
  }
  __syncwarp();
  // y pass: f_c[ay][ax] = sum_by J[by][ay] H[PF+by][ax] (+ for ay = 0 the
  // lower element's vertex term sum_by J[by][PC] H[by][ax])
  for (int o = lane; o < PC * PC; o += 32) {
    const int ay = o / PC, ax = o - ay * PC;
    double s = 0.0, vt = 0.0;
#pragma unroll
    for (int by = 0; by < PF; ++by) {
      s = fma(Js[by * NC + ay], Hw[warp][(PF + by) * PC + ax], s);
      vt = fma(Js[by * NC + PC], Hw[warp][by * PC + ax], vt);
    }
    if (ay == 0) s += vt;
    A.dst[(size_t)(ey * PC + ay) * Nxc + ex * PC + ax] = s;
  }
}

// restriction with a 2 x 2 block of coarse elements per CTA (one warp each):
// the 3 x 3 fine elements they read are staged once in shared memory
// (2.25x instead of 4x re-reads of the fine field); the per-warp passes are
// restrict_warp_kernel's.
template <int PC, int PF>
__global__ void __launch_bounds__(128) restrict_blk_kernel(const __grid_constant__ TrArgs A) {
  SMG_PDL_TRIGGER();
  constexpr int NC = PC + 1, R3 = 3 * PF, LD = R3 + 1, R2 = 2 * PF;
  static_assert(R2 <= 32, "fine rows per warp");
  __shared__ double Js[(PF + 1) * NC];
  __shared__ double Fr[R3 * LD];
  __shared__ double Hw[4][R2 * PC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (PF + 1) * NC; i += 128) Js[i] = A.J[i];
  const int bx = blockIdx.x % A.tiles_x, by = blockIdx.x / A.tiles_x;
  const int Nxf = A.n_x * PF, Nyf = A.n_y * PF, Nxc = A.n_x * PC;
  const int Y0 = (2 * by - 1) * PF, X0 = (2 * bx - 1) * PF;   // region origin (fine)
  SMG_PDL_WAIT();
  {
    constexpr int NL = (R3 * R3 + 127) / 128;
    double v[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const int i = threadIdx.x + 128 * k, ry = i / R3, rx = i - ry * R3;
      v[k] = i < R3 * R3 ? A.src[(size_t)wrapi(Y0 + ry, Nyf) * Nxf + wrapi(X0 + rx, Nxf)] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const int i = threadIdx.x + 128 * k, ry = i / R3, rx = i - ry * R3;
      if (i < R3 * R3) Fr[ry * LD + rx] = v[k];
    }
  }
  __syncthreads();
  const int wy = warp >> 1, wx = warp & 1;
  const int ey = 2 * by + wy, ex = 2 * bx + wx;
  const double* F = Fr + (wy * PF) * LD + wx * PF;   // this warp's 2PF x 2PF sub-region
  for (int ry = lane; ry < R2; ry += 32) {
    const double* f = F + ry * LD;
    double s[PC];
#pragma unroll
    for (int ax = 0; ax < PC; ++ax) s[ax] = 0.0;
    double vt = 0.0;
#pragma unroll
    for (int bb = 0; bb < PF; ++bb) {
      const double fo = f[PF + bb], fl = f[bb];
#pragma unroll
      for (int ax = 0; ax < PC; ++ax) s[ax] = fma(A.J[bb * NC + ax], fo, s[ax]);
      vt = fma(A.J[bb * NC + PC], fl, vt);
    }
    s[0] += vt;
#pragma unroll
    for (int ax = 0; ax < PC; ++ax) Hw[warp][ry * PC + ax] = s[ax];
  }
  __syncwarp();
  for (int o = lane; o < PC * PC; o += 32) {
    const int ay = o / PC, ax = o - ay * PC;
    double sacc = 0.0, vt = 0.0;
#pragma unroll
    for (int bb = 0; bb < PF; ++bb) {
      sacc = fma(Js[bb * NC + ay], Hw[warp][(PF + bb) * PC + ax], sacc);
      vt = fma(Js[bb * NC + PC], Hw[warp][bb * PC + ax], vt);
    }
    if (ay == 0) sacc += vt;
    A.dst[(size_t)(ey * PC + ay) * Nxc + ex * PC + ax] = sacc;
  }
}

template <int PC, int PF>
int tr_launch_warp(const TrArgs& A, bool prolong, cudaStream_t st) {
  if (prolong) {
    launch(prolong_warp_kernel<PC, PF>, dim3((A.n_x * A.n_y + kTrWarps - 1) / kTrWarps), dim3(32 * kTrWarps), 0, st, A);
  } else {
    static const int blk = env_int("SMG_TR_BLK", 1);
    if (blk && A.n_x % 2 == 0 && A.n_y % 2 == 0 && 3 * PF * (3 * PF + 1) * 8 <= 40 * 1024) {
      TrArgs B = A;
      B.tiles_x = A.n_x / 2;
      launch(restrict_blk_kernel<PC, PF>, dim3((A.n_x / 2) * (A.n_y / 2)), dim3(128), 0, st, B);
      return check_launch("restrict_blk_kernel");
    }
    constexpr int RW = tr_rwarps<PF>();
    launch(restrict_warp_kernel<PC, PF>, dim3((A.n_x * A.n_y + RW - 1) / RW), dim3(32 * RW), 0, st, A);
  }
  return check_launch(prolong ? "prolong_warp_kernel" : "restrict_warp_kernel");
}

// tile T (elements per side) chosen at run time from the compiled set
template <int PC, int PF>
int tr_launch(const TrArgs& A, int n_x, int n_y, bool prolong, cudaStream_t st) {
  if constexpr (PF == 3) {
    // warp-per-element prolongation where it measured faster than the tiled
    // kernel on B200 (C5 p_f = 3: 79 -> 40 us; slower at p_f = 12: 195 ->
    // 326, 6: 111 -> 157, and at 24 / 32 than the two-element tiles below:
    // 1118 vs 584 us, 136 vs 89 us); restriction stays tiled
    static const int warp = env_int("SMG_TR_WARP", 1);
    if (prolong && warp) {
      TrArgs B = A;
      B.n_x = n_x;
      B.n_y = n_y;
      launch(prolong_warp_g_kernel<PC, PF>, dim3((n_x * n_y + kTrWarps - 1) / kTrWarps), dim3(32 * kTrWarps), 0, st, B);
      return check_launch("prolong_warp_g_kernel");
    }
  }
  if constexpr (PF <= 16 && (PF & (PF - 1)) == 0) {
    static const int warp = env_int("SMG_TR_WARP", 1);
    if (warp) {
      TrArgs B = A;
      B.n_x = n_x;
      B.n_y = n_y;
      return tr_launch_warp<PC, PF>(B, prolong, st);
    }
  }
  // p_f > 16: two coarse elements per side (2.25x the window of one, a
  // quarter of the CTAs; one-element CTAs were latency-bound) -- except the
  // p_f = 32 restriction, measured slower that way (C3: 172 -> 201 us;
  // prolongation 136 -> 89 us, p_f = 24: restrict 1437 -> 834, prolong
  // 1118 -> 584 us)
  constexpr int T0 = PF > 16 ? 2 : 32 / PF;
  const int t0 = (PF >= 32 && !prolong) ? 1 : T0;
  // largest power-of-two T <= t0 dividing the mesh that keeps >= 296 CTAs,
  // else the one with the most CTAs
  int best = 1;
  for (int t = t0; t >= 1; t /= 2) {
    if (n_x % t || n_y % t) continue;
    best = t;
    static const int min_ctas = env_int("SMG_TR_MIN_CTAS", 296);
    if ((long)(n_x / t) * (n_y / t) >= min_ctas) break;
  }
  switch (best) {
    case 16: if constexpr (T0 >= 16) return tr_launch_t<PC, PF, (T0 >= 16 ? 16 : 1)>(A, prolong, st); break;
    case 8: if constexpr (T0 >= 8) return tr_launch_t<PC, PF, (T0 >= 8 ? 8 : 1)>(A, prolong, st); break;
    case 4: if constexpr (T0 >= 4) return tr_launch_t<PC, PF, (T0 >= 4 ? 4 : 1)>(A, prolong, st); break;
    case 2: if constexpr (T0 >= 2) return tr_launch_t<PC, PF, (T0 >= 2 ? 2 : 1)>(A, prolong, st); break;
    default: break;
  }
  return tr_launch_t<PC, PF, 1>(A, prolong, st);
}

TrFn transfer_dispatch(int pc, int pf) {
#define SMG_TR(a, b) if (pc == a && pf == b) return &tr_launch<a, b>;
  SMG_TR(1, 2) SMG_TR(2, 4) SMG_TR(4, 8) SMG_TR(8, 16) SMG_TR(16, 32)
  SMG_TR(1, 3) SMG_TR(3, 6) SMG_TR(6, 12) SMG_TR(12, 24)
#undef SMG_TR
  return nullptr;
}

}  // namespace smg
