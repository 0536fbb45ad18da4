// Contraction-loop microbenchmark, round 2: the Schwarz kernel's line
// contraction t[l][i] = sum_k S[k][i] x_l[k] (H x H factor, L lines per
// thread, k streamed so that only L*H accumulators live in registers), with
// the input fold x_k +- x_{M-1-k} of the real kernel (FOLD) and the output
// written back to shared memory, four stages with distinct factors and a
// block barrier between stages.  Factor operands from
//   SRC 0: the kernel-parameter constant bank (LDCU + uniform operand)
//   SRC 1: shared memory, warp-uniform double2 broadcast loads
// Reports useful TFLOP/s (2 * H^2 per line and stage) against the measured
// DFMA peak (34.2 TF) for several CTAs per SM.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int NSTG = 4;
constexpr int HMAX = 18;
struct Fac { double s[NSTG][HMAX * HMAX]; };

template <int H, int L, int SRC, bool FOLD>
__global__ void __launch_bounds__(128) contract(double* out, int iters, const __grid_constant__ Fac F) {
  constexpr int M = 2 * H - 1;           // window length whose fold gives H
  constexpr int NT = 128;
  constexpr int LINES = NT;   // the L lines of a thread alias other threads' lines (timing only)
  extern __shared__ __align__(16) double sh[];
  double* xa = sh;                        // [M][LINES]
  double* xb = sh + M * LINES;            // [M][LINES]
  double* fs = xb + M * LINES;            // [NSTG][H][H]
  for (int i = threadIdx.x; i < NSTG * H * H; i += NT) fs[i] = F.s[i / (H * H)][i % (H * H)];
  for (int i = threadIdx.x; i < M * LINES; i += NT) { xa[i] = 1e-3 * (i % 97); xb[i] = 0.0; }
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int st = 0; st < NSTG; ++st) {
      const double* in = (st & 1) ? xb : xa;
      double* o = (st & 1) ? xa : xb;
      double t[L][H];
#pragma unroll
      for (int l = 0; l < L; ++l)
#pragma unroll
        for (int i = 0; i < H; ++i) t[l][i] = 0.0;
#pragma unroll
      for (int k = 0; k < H; ++k) {
        double x[L];
#pragma unroll
        for (int l = 0; l < L; ++l) {
          const int ln = (threadIdx.x + l * 32) & (NT - 1);
          const double a = in[k * LINES + ln];
          x[l] = FOLD ? a + in[(M - 1 - k) * LINES + ln] : a;
        }
        double f[H];
        if (SRC == 1) {
          const double2* f2 = reinterpret_cast<const double2*>(fs + st * H * H + k * H);
#pragma unroll
          for (int i = 0; i < H / 2; ++i) { const double2 v = f2[i]; f[2 * i] = v.x; f[2 * i + 1] = v.y; }
          if (H & 1) f[H - 1] = fs[st * H * H + k * H + H - 1];
        } else {
#pragma unroll
          for (int i = 0; i < H; ++i) f[i] = F.s[st][k * H + i];
        }
#pragma unroll
        for (int i = 0; i < H; ++i)
#pragma unroll
          for (int l = 0; l < L; ++l) t[l][i] = fma(f[i], x[l], t[l][i]);
      }
#pragma unroll
      for (int l = 0; l < L; ++l)
#pragma unroll
        for (int i = 0; i < H; ++i) o[i * LINES + ((threadIdx.x + l * 32) & (NT - 1))] = t[l][i];
      __syncthreads();
    }
  }
  if (xa[threadIdx.x] == 1.2345) out[threadIdx.x] = xa[threadIdx.x];
}

template <int H, int L, int SRC, bool FOLD>
int run(double* d, const Fac& F) {
  constexpr int M = 2 * H - 1, NT = 128;
  const size_t smem = sizeof(double) * (2 * (size_t)M * NT + NSTG * H * H);
  CK(cudaFuncSetAttribute(contract<H, L, SRC, FOLD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, contract<H, L, SRC, FOLD>));
  int maxb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, contract<H, L, SRC, FOLD>, NT, smem));
  for (int bps : {1, 2, 3, 4, 6, 8}) {
    if (bps > maxb) break;
    const int blocks = 148 * bps, iters = 100;
    contract<H, L, SRC, FOLD><<<blocks, NT, smem>>>(d, 2, F);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    contract<H, L, SRC, FOLD><<<blocks, NT, smem>>>(d, iters, F);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * H * H * NSTG * (double)L * NT * blocks * iters;
    printf("H %2d L %d %s fold %d regs %3d maxb %d warps/SM %2d: %6.2f TFLOP/s\n", H, L, SRC ? "smem " : "const",
           (int)FOLD, fa.numRegs, maxb, bps * 4, flops / ms / 1e9);
  }
  return 0;
}

int main() {
  double* d; CK(cudaMalloc(&d, 1 << 20));
  Fac F;
  for (int s = 0; s < NSTG; ++s)
    for (int i = 0; i < HMAX * HMAX; ++i) F.s[s][i] = 1e-3 * ((i * 7 + s) % 31);
  run<10, 1, 0, true>(d, F); run<10, 2, 0, true>(d, F); run<10, 3, 0, true>(d, F); run<10, 4, 0, true>(d, F);
  run<10, 2, 1, true>(d, F); run<10, 4, 1, true>(d, F); run<10, 4, 0, false>(d, F);
  run<14, 1, 0, true>(d, F); run<14, 2, 0, true>(d, F); run<14, 3, 0, true>(d, F); run<14, 4, 0, true>(d, F);
  run<18, 1, 0, true>(d, F); run<18, 2, 0, true>(d, F); run<18, 3, 0, true>(d, F);
  return 0;
}
