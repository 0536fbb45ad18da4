// Contraction-loop microbenchmark for the Schwarz kernel's DFMA stages:
// t[i] = sum_k S[k][i] x[k] over H x H factors (H = 14, p = 24's even half),
// four stages per "tile" with distinct factors, factor operands from
//   const1 / const2 : the kernel-parameter constant bank, 1 or 2 lines per thread
//   smem1  / smem2  : shared memory (warp-uniform broadcast loads), 1 or 2 lines
// Reports achieved TFLOP/s (useful FMAs x 2) for 8 / 16 / 24 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int H = 14;
constexpr int NSTG = 4;
struct Fac { double s[NSTG][H * H]; };

template <int L, bool SMEM>
__global__ void contract(double* out, int iters, const __grid_constant__ Fac F) {
  extern __shared__ double sh[];
  double* xs = sh;                       // per-thread lines (L*H per thread)
  double* fs = sh + blockDim.x * L * H;  // factors
  if (SMEM)
    for (int i = threadIdx.x; i < NSTG * H * H; i += blockDim.x) fs[i] = F.s[0][i];
  for (int i = threadIdx.x; i < blockDim.x * L * H; i += blockDim.x) xs[i] = 1e-3 * (i % 97);
  __syncthreads();
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int st = 0; st < NSTG; ++st) {
      double x[L][H], t[L][H];
#pragma unroll
      for (int l = 0; l < L; ++l)
#pragma unroll
        for (int k = 0; k < H; ++k) x[l][k] = xs[(l * blockDim.x + threadIdx.x) + k * blockDim.x * L];
      const double* S = SMEM ? fs + st * H * H : F.s[st];
#pragma unroll
      for (int l = 0; l < L; ++l)
#pragma unroll
        for (int i = 0; i < H; ++i) t[l][i] = S[i] * x[l][0];
#pragma unroll
      for (int k = 1; k < H; ++k)
#pragma unroll
        for (int i = 0; i < H; ++i)
#pragma unroll
          for (int l = 0; l < L; ++l) t[l][i] = fma(S[k * H + i], x[l][k], t[l][i]);
#pragma unroll
      for (int l = 0; l < L; ++l)
#pragma unroll
        for (int i = 0; i < H; ++i) acc += t[l][i];
    }
  }
  if (acc == 1.2345) out[threadIdx.x] = acc;
}

template <int L, bool SMEM>
int run(const char* name, double* d, const Fac& F) {
  const int sms = 148;
  for (int warps : {8, 16, 24}) {
    const int threads = 256 / L;  // 8 warps of work per block at L = 1
    const int bps = warps * 32 / threads;
    const size_t smem = sizeof(double) * (threads * L * H + (SMEM ? NSTG * H * H : 0));
    CK(cudaFuncSetAttribute(contract<L, SMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int blocks = sms * bps;
    const int iters = 200;
    contract<L, SMEM><<<blocks, threads, smem>>>(d, 2, F);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    contract<L, SMEM><<<blocks, threads, smem>>>(d, iters, F);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * H * H * NSTG * L * (double)threads * blocks * iters;
    printf("%-7s warps/SM %2d (blocks %d x %d thr): %6.2f TFLOP/s\n", name, warps,
           bps, threads, flops / ms / 1e9);
  }
  return 0;
}

int main() {
  double* d; CK(cudaMalloc(&d, 1 << 20));
  Fac F;
  for (int s = 0; s < NSTG; ++s)
    for (int i = 0; i < H * H; ++i) F.s[s][i] = 1e-3 * ((i * 7 + s) % 31);
  run<1, false>("const1", d, F);
  run<2, false>("const2", d, F);
  run<1, true>("smem1", d, F);
  run<2, true>("smem2", d, F);
  return 0;
}
