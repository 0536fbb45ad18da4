// Microbenchmark: FP64 rate of the FD contraction building block (half
// analysis, M = 19: even 10x10, odd 9x9) on shared-memory data.  Variants:
//   A  one line per thread, factors from the constant bank (LDCU)
//   B  two lines per thread (EPT=2) sharing each constant
//   C  one line per thread, factors from shared memory (broadcast LDS.128)
//   D  EPT=2, factors from shared memory
#include <cstdio>
#include <cuda_runtime.h>

constexpr int M = 19, HE = 10, HO = 9, E = 8;
struct CArgs { double Se[HE * HE], So[HO * HO + 1]; };

template <int H, bool ODD, int EPT, bool SMEMS>
__device__ __forceinline__ void lines(const double* __restrict__ S, const double* Bp0, int stride_e, int c, double (&t)[EPT][H]) {
  double xk[EPT][H];
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const double* Bp = Bp0 + q * stride_e;
#pragma unroll
    for (int k = 0; k < H; ++k) {
      if (k < HO) {
        const double a = Bp[k * M + c], b = Bp[(M - 1 - k) * M + c];
        xk[q][k] = ODD ? a - b : a + b;
      } else {
        xk[q][k] = Bp[k * M + c];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < EPT; ++q)
#pragma unroll
    for (int i = 0; i < H; ++i) t[q][i] = S[i] * xk[q][0];
#pragma unroll
  for (int k = 1; k < H; ++k)
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const double s = S[k * H + i];
#pragma unroll
      for (int q = 0; q < EPT; ++q) t[q][i] = fma(s, xk[q][k], t[q][i]);
    }
}

template <int EPT, bool SMEMS>
__global__ void __launch_bounds__(2 * ((E / EPT) * M + 31) / 32 * 32, 2) core(double* out, int reps, const __grid_constant__ CArgs C) {
  __shared__ double B[E * M * M];
  __shared__ double Ss[HE * HE + HO * HO + 1];
  constexpr int NH = ((E / EPT) * M + 31) / 32 * 32;
  const int tid = threadIdx.x;
  const bool odd = tid >= NH;
  const int line = odd ? tid - NH : tid;
  const int e = line / M, c = line - e * M;
  const bool act = e < E / EPT;
  for (int i = tid; i < E * M * M; i += blockDim.x) B[i] = 1e-3 * (i % 97);
  for (int i = tid; i < HE * HE; i += blockDim.x) Ss[i] = C.Se[i];
  for (int i = tid; i < HO * HO; i += blockDim.x) Ss[HE * HE + i] = C.So[i];
  __syncthreads();
  double* Bp = B + e * M * M;
  const int se = (E / EPT) * M * M;
  for (int r = 0; r < reps; ++r) {
    double t[EPT][HE];
    if (act) {
      if (!odd) lines<HE, false, EPT, SMEMS>(SMEMS ? Ss : C.Se, Bp, se, c, t);
      else lines<HO, true, EPT, SMEMS>(SMEMS ? Ss + HE * HE : C.So, Bp, se, c, reinterpret_cast<double(&)[EPT][HO]>(t));
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        if (!odd) {
#pragma unroll
          for (int i = 0; i < HE; ++i) Bp[q * se + i * M + c] = t[q][i] * 0.5;
        } else {
#pragma unroll
          for (int i = 0; i < HO; ++i) Bp[q * se + (HE + i) * M + c] = t[q][i] * 0.5;
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) out[blockIdx.x] = B[5];
}

// E: register-only contraction chain (upper bound of the building block)
template <int EPT>
__global__ void __launch_bounds__(320, 2) coreE(double* out, int reps, const __grid_constant__ CArgs C) {
  double x[EPT][HE];
#pragma unroll
  for (int q = 0; q < EPT; ++q)
#pragma unroll
    for (int k = 0; k < HE; ++k) x[q][k] = 1e-3 * (threadIdx.x + k + q);
  for (int r = 0; r < reps; ++r) {
    double t[EPT][HE];
#pragma unroll
    for (int q = 0; q < EPT; ++q)
#pragma unroll
      for (int i = 0; i < HE; ++i) t[q][i] = C.Se[i] * x[q][0];
#pragma unroll
    for (int k = 1; k < HE; ++k)
#pragma unroll
      for (int i = 0; i < HE; ++i) {
        const double sv = C.Se[k * HE + i];
#pragma unroll
        for (int q = 0; q < EPT; ++q) t[q][i] = fma(sv, x[q][k], t[q][i]);
      }
#pragma unroll
    for (int q = 0; q < EPT; ++q)
#pragma unroll
      for (int i = 0; i < HE; ++i) x[q][i] = t[q][i];
  }
  double sacc = 0;
#pragma unroll
  for (int q = 0; q < EPT; ++q)
#pragma unroll
    for (int i = 0; i < HE; ++i) sacc += x[q][i];
  if (sacc == 1.2345) out[threadIdx.x] = sacc;
}

template <int EPT>
void runE(double* d, const CArgs& C) {
  const int reps = 2000, grid = 148 * 2;
  coreE<EPT><<<grid, 320>>>(d, 10, C);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  coreE<EPT><<<grid, 320>>>(d, reps, C);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("E  EPT%d regs : %.2f TFLOP/s (%.3f ms)\n", EPT, 2.0 * grid * 320 * reps * HE * HE * EPT / ms / 1e9, ms);
}

template <int EPT, bool SMEMS>
void run(const char* name, double* d, const CArgs& C) {
  constexpr int NH = ((E / EPT) * M + 31) / 32 * 32;
  const int reps = 200, grid = 148 * 4;
  core<EPT, SMEMS><<<grid, 2 * NH>>>(d, 10, C);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  core<EPT, SMEMS><<<grid, 2 * NH>>>(d, reps, C);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double fma = (double)grid * reps * E * M * (HE * HE + HO * HO) / 2;  // per rep: E*M lines, half each parity
  printf("%s: %.2f TFLOP/s (%.3f ms) %s\n", name, 2 * 2 * fma / ms / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  CArgs C;
  for (int i = 0; i < HE * HE; ++i) C.Se[i] = 0.1 * (i % 7);
  for (int i = 0; i < HO * HO + 1; ++i) C.So[i] = 0.1 * (i % 3);
  double* d;
  cudaMalloc(&d, 1 << 20);
  run<1, false>("A  EPT1 const", d, C);
  run<2, false>("B  EPT2 const", d, C);
  run<1, true>("C  EPT1 smem ", d, C);
  run<2, true>("D  EPT2 smem ", d, C);
  runE<1>(d, C);
  runE<2>(d, C);
  runE<4>(d, C);
  return 0;
}
