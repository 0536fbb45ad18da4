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
  // restriction: fine staged incl. the low halo element, coarse own tile
  static constexpr int FX = (T + 1) * PF, OXC = T * PC;
  static constexpr int NT = 256;
  static constexpr size_t SMEM_P = sizeof(double) * ((size_t)CX * CX + (size_t)CX * OXF + (size_t)OXF * OXF + NF * NC);
  static constexpr size_t SMEM_R = sizeof(double) * ((size_t)FX * FX + (size_t)FX * OXC + NF * NC);
};

template <int PC, int PF, int T>
__global__ void __launch_bounds__(256) prolong_kernel(const __grid_constant__ TrArgs A) {
  SMG_PDL_ENTRY();
  using G = TrGeom<PC, PF, T>;
  constexpr int NC = G::NC, NF = G::NF, CX = G::CX, OX = G::OXF, NT = G::NT;
  extern __shared__ double sm[];
  double* C = sm;             // CX x CX coarse values
  double* Tt = C + CX * CX;   // CX x OX  (x-interpolated)
  double* UF = Tt + CX * OX;  // OX x OX  old fine values (accumulate)
  double* Js = UF + OX * OX;  // NF x NC
  const int tid = threadIdx.x;
  const int tx = blockIdx.x % A.tiles_x, ty = blockIdx.x / A.tiles_x;
  const int Nxc = A.n_x * PC, Nyc = A.n_y * PC, Nxf = A.n_x * PF;
  const int Xc0 = tx * T * PC, Yc0 = ty * T * PC, Xf0 = tx * OX, Yf0 = ty * OX;
  for (int idx = tid; idx < CX * CX; idx += NT) {
    const int y = idx / CX, x = idx - y * CX;
    tr_cp_async8(C + idx, A.src + (size_t)wrapi(Yc0 + y, Nyc) * Nxc + wrapi(Xc0 + x, Nxc));
  }
  if (A.accumulate) {
    for (int idx = tid; idx < OX * OX; idx += NT) {
      const int y = idx / OX, x = idx - y * OX;
      tr_cp_async8(UF + idx, A.dst + (size_t)(Yf0 + y) * Nxf + (Xf0 + x));
    }
  }
  for (int idx = tid; idx < NF * NC; idx += NT) Js[idx] = A.J[idx];
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  // x: Tt[rc][xf] = sum_bc J[b][bc] C[rc][exl*PC + bc]
  for (int idx = tid; idx < CX * OX; idx += NT) {
    const int rc = idx / OX, xf = idx - rc * OX;
    const int exl = xf / PF, b = xf - exl * PF;
    const double* c = C + rc * CX + exl * PC;
    const double* j = Js + b * NC;
    double s = j[0] * c[0];
#pragma unroll
    for (int k = 1; k < NC; ++k) s = fma(j[k], c[k], s);
    Tt[idx] = s;
  }
  __syncthreads();
  // y: out[yf][xf] = sum_ac J[a][ac] Tt[eyl*PC + ac][xf]
  for (int idx = tid; idx < OX * OX; idx += NT) {
    const int yf = idx / OX, xf = idx - yf * OX;
    const int eyl = yf / PF, a = yf - eyl * PF;
    const double* t = Tt + (eyl * PC) * OX + xf;
    const double* j = Js + a * NC;
    double s = j[0] * t[0];
#pragma unroll
    for (int k = 1; k < NC; ++k) s = fma(j[k], t[k * OX], s);
    A.dst[(size_t)(Yf0 + yf) * Nxf + (Xf0 + xf)] = A.accumulate ? UF[idx] + s : s;
  }
}

template <int PC, int PF, int T>
__global__ void __launch_bounds__(256) restrict_kernel(const __grid_constant__ TrArgs A) {
  SMG_PDL_ENTRY();
  using G = TrGeom<PC, PF, T>;
  constexpr int NC = G::NC, NF = G::NF, FX = G::FX, OX = G::OXC, NT = G::NT;
  extern __shared__ double sm[];
  double* F = sm;              // FX x FX fine own rows/cols of elements [t0-1, t0+T)
  double* Tx = F + FX * FX;    // FX x OX  (x-restricted)
  double* Js = Tx + FX * OX;   // NF x NC
  const int tid = threadIdx.x;
  const int tx = blockIdx.x % A.tiles_x, ty = blockIdx.x / A.tiles_x;
  const int Nxf = A.n_x * PF, Nyf = A.n_y * PF, Nxc = A.n_x * PC;
  const int Xf0 = (tx * T - 1) * PF, Yf0 = (ty * T - 1) * PF;
  for (int idx = tid; idx < FX * FX; idx += NT) {
    const int y = idx / FX, x = idx - y * FX;
    tr_cp_async8(F + idx, A.src + (size_t)wrapi(Yf0 + y, Nyf) * Nxf + wrapi(Xf0 + x, Nxf));
  }
  for (int idx = tid; idx < NF * NC; idx += NT) Js[idx] = A.J[idx];
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  // x: Tx[yf][xc] = sum_{b<PF} J[b][ac] F[yf][(exl+1) PF + b]  (+ left element's ac = PC term)
  for (int idx = tid; idx < FX * OX; idx += NT) {
    const int yf = idx / OX, xc = idx - yf * OX;
    const int exl = xc / PC, ac = xc - exl * PC;
    const double* f = F + yf * FX + (exl + 1) * PF;
    double s = Js[ac] * f[0];
#pragma unroll
    for (int b = 1; b < PF; ++b) s = fma(Js[b * NC + ac], f[b], s);
    if (ac == 0) {
      const double* fl = f - PF;
      double s2 = Js[PC] * fl[0];
#pragma unroll
      for (int b = 1; b < PF; ++b) s2 = fma(Js[b * NC + PC], fl[b], s2);
      s += s2;
    }
    Tx[idx] = s;
  }
  __syncthreads();
  // y: out[yc][xc] = sum_{a<PF} J[a][acy] Tx[(eyl+1) PF + a][xc]  (+ lower element's PC term)
  for (int idx = tid; idx < OX * OX; idx += NT) {
    const int yc = idx / OX, xc = idx - yc * OX;
    const int eyl = yc / PC, ac = yc - eyl * PC;
    const double* t = Tx + ((eyl + 1) * PF) * OX + xc;
    double s = Js[ac] * t[0];
#pragma unroll
    for (int a = 1; a < PF; ++a) s = fma(Js[a * NC + ac], t[a * OX], s);
    if (ac == 0) {
      const double* tl = t - PF * OX;
      double s2 = Js[PC] * tl[0];
#pragma unroll
      for (int a = 1; a < PF; ++a) s2 = fma(Js[a * NC + PC], tl[a * OX], s2);
      s += s2;
    }
    A.dst[(size_t)(ty * OX + yc) * Nxc + (tx * OX + xc)] = s;
  }
}

template <int PC, int PF, int T>
int tr_launch_t(const TrArgs& A0, bool prolong, cudaStream_t st) {
  using G = TrGeom<PC, PF, T>;
  TrArgs A = A0;
  A.tiles_x = A.n_x / T;
  const int grid = (A.n_x / T) * (A.n_y / T);
  if (prolong) {
    static bool attr = false;
    if (!attr && G::SMEM_P > 48 * 1024)
      cudaFuncSetAttribute(prolong_kernel<PC, PF, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM_P);
    attr = true;
    launch(prolong_kernel<PC, PF, T>, dim3(grid), dim3(G::NT), G::SMEM_P, st, A);
  } else {
    static bool attr = false;
    if (!attr && G::SMEM_R > 48 * 1024)
      cudaFuncSetAttribute(restrict_kernel<PC, PF, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM_R);
    attr = true;
    launch(restrict_kernel<PC, PF, T>, dim3(grid), dim3(G::NT), G::SMEM_R, st, A);
  }
  return check_launch(prolong ? "prolong_kernel" : "restrict_kernel");
}

// tile T (elements per side) chosen at run time from the compiled set
template <int PC, int PF>
int tr_launch(const TrArgs& A, int n_x, int n_y, bool prolong, cudaStream_t st) {
  constexpr int T0 = PF >= 32 ? 1 : 32 / PF;
  // largest power-of-two T <= T0 dividing the mesh that keeps >= 296 CTAs,
  // else the one with the most CTAs
  int best = 1;
  for (int t = T0; t >= 1; t /= 2) {
    if (n_x % t || n_y % t) continue;
    best = t;
    if ((long)(n_x / t) * (n_y / t) >= 296) break;
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
