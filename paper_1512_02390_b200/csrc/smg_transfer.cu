// p-multigrid transfers (subsystem 3).
//
// Reference: prolongate / restrict_residual (multigrid.py:180-193) multiply
// by dense global 1D matrices P_y, P_x (multigrid.py:112-124) whose rows
// are ASSIGNED per element (a fine vertex node appears once).  Here both
// are element-local and sum-factorized with the (p_f+1) x (p_c+1) matrix J:
//   prolongation : fine node (a,b) owned by element e (0 <= a,b < p_f)
//                  u_f += sum_{ac,bc} J[a][ac] U_c,e[ac][bc] J[b][bc]
//   restriction  : owner-computes over fine rows/cols b < p_f of every
//                  element (so shared fine nodes are counted once, as in
//                  P^T), gathered onto coarse nodes; the coarse vertex
//                  (ac = 0) also collects element e-1's ac = p_c term.
// Both are gather-form per output node: deterministic, no atomics.
#include "smg_transfer.cuh"

namespace smg {

template <int PC, int PF>
__global__ void __launch_bounds__(kTrThreads) prolong_kernel(const __grid_constant__ TrArgs A) {
  constexpr int NC = PC + 1;
  extern __shared__ double sm[];
  const int TX = A.TX, TY = A.TY;
  const int CX = TX * PC + 1, CY = TY * PC + 1;   // coarse tile incl. high vertex
  const int OX = TX * PF;                          // fine own cols
  double* C = sm;                                  // CY x CX
  double* T = C + CX * CY;                         // CY x OX
  const int tid = threadIdx.x, nt = blockDim.x;
  const int tx = blockIdx.x % A.tiles_x, ty = blockIdx.x / A.tiles_x;
  const int Nxc = A.n_x * PC, Nyc = A.n_y * PC, Nxf = A.n_x * PF;
  const int Xc0 = tx * TX * PC, Yc0 = ty * TY * PC;
  for (int idx = tid; idx < CX * CY; idx += nt) {
    const int y = idx / CX, x = idx - y * CX;
    C[idx] = __ldg(A.src + (size_t)wrapi(Yc0 + y, Nyc) * Nxc + wrapi(Xc0 + x, Nxc));
  }
  __syncthreads();
  // x: T[rc][exl*PF + b] = sum_bc C[rc][exl*PC + bc] J[b][bc]
  for (int it = tid; it < CY * TX; it += nt) {
    const int rc = it / TX, exl = it - rc * TX;
    double c[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) c[k] = C[rc * CX + exl * PC + k];
#pragma unroll
    for (int b = 0; b < PF; ++b) {
      double s = A.J[b * NC] * c[0];
#pragma unroll
      for (int k = 1; k < NC; ++k) s = fma(A.J[b * NC + k], c[k], s);
      T[rc * OX + exl * PF + b] = s;
    }
  }
  __syncthreads();
  // y: out[eyl*PF + a][xf] = sum_ac J[a][ac] T[eyl*PC + ac][xf]
  for (int it = tid; it < TY * OX; it += nt) {
    const int eyl = it / OX, xf = it - eyl * OX;
    double t[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) t[k] = T[(eyl * PC + k) * OX + xf];
    const int gyf = (ty * TY + eyl) * PF, gxf = tx * OX + xf;
#pragma unroll
    for (int a = 0; a < PF; ++a) {
      double s = A.J[a * NC] * t[0];
#pragma unroll
      for (int k = 1; k < NC; ++k) s = fma(A.J[a * NC + k], t[k], s);
      double* d = A.dst + (size_t)(gyf + a) * Nxf + gxf;
      *d = A.accumulate ? *d + s : s;
    }
  }
}

template <int PC, int PF>
__global__ void __launch_bounds__(kTrThreads) restrict_kernel(const __grid_constant__ TrArgs A) {
  constexpr int NC = PC + 1;
  extern __shared__ double sm[];
  const int TX = A.TX, TY = A.TY;
  const int FX = (TX + 1) * PF, FY = (TY + 1) * PF;  // fine own rows/cols incl. low halo element
  const int OX = TX * PC, OY = TY * PC;              // coarse own nodes
  double* F = sm;                                    // FY x FX
  double* TXc = F + FX * FY;                         // FY x OX  (x-restricted, own coarse cols)
  double* VX = TXc + FY * OX;                        // FY x (TX+1)
  double* RY = VX + FY * (TX + 1);                   // OY x OX
  double* VY = RY + OY * OX;                         // OX x (TY+1)
  const int tid = threadIdx.x, nt = blockDim.x;
  const int tx = blockIdx.x % A.tiles_x, ty = blockIdx.x / A.tiles_x;
  const int Nxf = A.n_x * PF, Nyf = A.n_y * PF, Nxc = A.n_x * PC;
  const int Xf0 = (tx * TX - 1) * PF, Yf0 = (ty * TY - 1) * PF;
  for (int idx = tid; idx < FX * FY; idx += nt) {
    const int y = idx / FX, x = idx - y * FX;
    F[idx] = __ldg(A.src + (size_t)wrapi(Yf0 + y, Nyf) * Nxf + wrapi(Xf0 + x, Nxf));
  }
  __syncthreads();
  // x pass over every staged fine row: element exl-1 (exl = 0 is the halo element)
  for (int it = tid; it < FY * (TX + 1); it += nt) {
    const int yf = it / (TX + 1), exl = it - yf * (TX + 1);
    const double* fr = F + yf * FX + exl * PF;
    double t[NC];
#pragma unroll
    for (int ac = 0; ac < NC; ++ac) t[ac] = A.J[ac] * fr[0];
#pragma unroll
    for (int b = 1; b < PF; ++b) {
      const double v = fr[b];
#pragma unroll
      for (int ac = 0; ac < NC; ++ac) t[ac] = fma(A.J[b * NC + ac], v, t[ac]);
    }
    if (exl > 0) {
#pragma unroll
      for (int ac = 0; ac < PC; ++ac) TXc[yf * OX + (exl - 1) * PC + ac] = t[ac];
    }
    VX[yf * (TX + 1) + exl] = t[PC];
  }
  __syncthreads();
  // y pass over own coarse columns: element eyl-1 over its own fine rows
  for (int it = tid; it < OX * (TY + 1); it += nt) {
    const int xc = it / (TY + 1), eyl = it - xc * (TY + 1);
    const bool vert = (xc % PC) == 0;
    double t[NC];
    for (int ac = 0; ac < NC; ++ac) t[ac] = 0.0;
#pragma unroll
    for (int a = 0; a < PF; ++a) {
      const int yf = eyl * PF + a;
      double v = TXc[yf * OX + xc];
      if (vert) v += VX[yf * (TX + 1) + xc / PC];
#pragma unroll
      for (int ac = 0; ac < NC; ++ac) t[ac] = fma(A.J[a * NC + ac], v, t[ac]);
    }
    if (eyl > 0) {
#pragma unroll
      for (int ac = 0; ac < PC; ++ac) RY[((eyl - 1) * PC + ac) * OX + xc] = t[ac];
    }
    VY[xc * (TY + 1) + eyl] = t[PC];
  }
  __syncthreads();
  for (int idx = tid; idx < OX * OY; idx += nt) {
    const int y = idx / OX, x = idx - y * OX;
    double v = RY[idx];
    if (y % PC == 0) v += VY[x * (TY + 1) + y / PC];
    A.dst[(size_t)(ty * OY + y) * Nxc + (tx * OX + x)] = v;
  }
}

size_t prolong_smem(int pc, int pf, int TX, int TY) {
  const size_t CX = (size_t)TX * pc + 1, CY = (size_t)TY * pc + 1;
  return sizeof(double) * (CX * CY + CY * (size_t)TX * pf);
}
size_t restrict_smem(int pc, int pf, int TX, int TY) {
  const size_t FX = (size_t)(TX + 1) * pf, FY = (size_t)(TY + 1) * pf;
  const size_t OX = (size_t)TX * pc, OY = (size_t)TY * pc;
  return sizeof(double) * (FX * FY + FY * OX + FY * (TX + 1) + OY * OX + OX * (TY + 1));
}

template <int PC, int PF>
int transfer_launch(const TrArgs& A, int grid, bool prolong, cudaStream_t st) {
  if (prolong) {
    const size_t smem = prolong_smem(PC, PF, A.TX, A.TY);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(prolong_kernel<PC, PF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    prolong_kernel<PC, PF><<<grid, kTrThreads, smem, st>>>(A);
  } else {
    const size_t smem = restrict_smem(PC, PF, A.TX, A.TY);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(restrict_kernel<PC, PF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    restrict_kernel<PC, PF><<<grid, kTrThreads, smem, st>>>(A);
  }
  return check_launch(prolong ? "prolong_kernel" : "restrict_kernel");
}

using TrFn = int (*)(const TrArgs&, int, bool, cudaStream_t);
TrFn transfer_dispatch(int pc, int pf) {
#define SMG_TR(a, b) if (pc == a && pf == b) return &transfer_launch<a, b>;
  SMG_TR(1, 2) SMG_TR(2, 4) SMG_TR(4, 8) SMG_TR(8, 16) SMG_TR(16, 32)
  SMG_TR(1, 3) SMG_TR(3, 6) SMG_TR(6, 12) SMG_TR(12, 24)
#undef SMG_TR
  return nullptr;
}

}  // namespace smg
