// Do the FP64 DFMA pipe and the DMMA tensor sub-pipe run concurrently on
// B200?  One kernel, warps split by role: the first `nd` warps of each CTA
// issue DMMA m8n8k4, the rest DFMA (register operands).  Reports each role's
// TFLOP/s alone and together.  Also a per-warp interleaved variant (every
// warp issues both, MIX DFMAs per DMMA).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int NACC = 8, NMMA = 4;

// role split: warp < nd -> DMMA (itd iterations), else DFMA (itf iterations)
__global__ void mixed(double* out, int nd, int itd, int itf, double a, double b) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp < nd) {
    double x = threadIdx.x * 1e-3, y = threadIdx.x * 2e-3;
    double c[NMMA][2];
#pragma unroll
    for (int i = 0; i < NMMA; ++i) { c[i][0] = i; c[i][1] = -i; }
    for (int it = 0; it < itd; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int i = 0; i < NMMA; ++i)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(x), "d"(y));
    }
#pragma unroll
    for (int i = 0; i < NMMA; ++i) s += c[i][0] + c[i][1];
  } else {
    double acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < itf; ++it) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
    }
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += acc[i];
  }
  if (s == 1.2345) out[threadIdx.x] = s;
}

// every warp issues both: per iteration 8*NMMA DMMAs and MIX*8*NMMA DFMAs
template <int MIX>
__global__ void interleaved(double* out, int iters, double a, double b) {
  double x = threadIdx.x * 1e-3, y = threadIdx.x * 2e-3;
  double c[NMMA][2];
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NMMA; ++i) { c[i][0] = i; c[i][1] = -i; }
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < NMMA; ++i) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(x), "d"(y));
#pragma unroll
        for (int m = 0; m < MIX; ++m) {
          const int j = (i * MIX + m) % NACC;
          acc[j] = fma(acc[j], a, b);
        }
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NMMA; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <int MIX>
int run_inter(double* d, int sms, int threads, int bps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * bps, iters = 4000;
  interleaved<MIX><<<blocks, threads>>>(d, 10, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  interleaved<MIX><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)blocks * threads / 32;
  const double fd = 2.0 * 256 * warps * iters * 8 * NMMA, ff = 2.0 * 32 * warps * iters * 8 * NMMA * MIX;
  printf("interleaved MIX %d threads %4d blocks/SM %d: DMMA %.2f + DFMA %.2f = %.2f TFLOP/s (%.3f ms)\n", MIX, threads,
         bps, fd / ms / 1e9, ff / ms / 1e9, (fd + ff) / ms / 1e9, ms);
  return 0;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  printf("device %s sms %d\n", prop.name, sms);
  double* d; CK(cudaMalloc(&d, 4096 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 512, nw = threads / 32;
  for (int bps : {1, 2}) {
    const int blocks = sms * bps;
    for (int nd : {0, nw, nw / 2, nw / 4, 3 * nw / 4}) {
      // iteration counts chosen so both roles would take about the same time at their own peaks
      const int itd = 4000, itf = 4000 * 2;  // per warp: DMMA 8*4*512 flop/it; DFMA 16*8*64 flop/it
      mixed<<<blocks, threads>>>(d, nd, 10, 10, 1.0000001, 1e-9);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      mixed<<<blocks, threads>>>(d, nd, itd, itf, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double fd = 2.0 * 256 * blocks * nd * (double)itd * 8 * NMMA;
      const double ff = 2.0 * 32 * blocks * (nw - nd) * (double)itf * 16 * NACC;
      printf("split threads %d blocks/SM %d dmma warps %2d / %2d: DMMA %.2f + DFMA %.2f = %.2f TFLOP/s (%.3f ms)\n",
             threads, bps, nd, nw, fd / ms / 1e9, ff / ms / 1e9, (fd + ff) / ms / 1e9, ms);
    }
    if (run_inter<1>(d, sms, threads, bps)) return 1;
    if (run_inter<2>(d, sms, threads, bps)) return 1;
    if (run_inter<4>(d, sms, threads, bps)) return 1;
    if (run_inter<8>(d, sms, threads, bps)) return 1;
    if (run_inter<16>(d, sms, threads, bps)) return 1;
  }
  return 0;
}
