// FP64 pipe microbenchmarks for B200 (sm_100a): DFMA (register operands),
// DFMA with constant-bank (kernel-parameter) operands, and DMMA m8n8k4.
// Prints achieved TFLOP/s for each; used to set the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int NACC = 8;
__global__ void dfma_reg(double* out, int iters, double a, double b) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

struct CParams { double c[256]; };
__global__ void dfma_const(double* out, int iters, const __grid_constant__ CParams P) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  double x = threadIdx.x * 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 256; r += NACC)
#pragma unroll
      for (int i = 0; i < NACC; ++i) acc[i] = fma(x, P.c[r + i], acc[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

constexpr int NMMA = 4;
__global__ void dmma_bench(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[NMMA][2];
#pragma unroll
  for (int i = 0; i < NMMA; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < NMMA; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NMMA; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("device %s sms %d clock %d kHz\n", prop.name, sms, prop.clockRate);
  double* d; CK(cudaMalloc(&d, 4096 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  CParams P; for (int i = 0; i < 256; ++i) P.c[i] = 1e-9 * i;
  for (int threads : {256, 512, 1024}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps;
      if (threads * bps > 2048) continue;
      int iters = 20000;
      dfma_reg<<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_reg<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * blocks * threads * (double)iters * 16 * NACC;
      printf("dfma_reg   threads %4d blocks/SM %d : %.2f TFLOP/s (%.3f ms)\n", threads, bps, flops / ms / 1e9, ms);
      int citers = 2000;
      dfma_const<<<blocks, threads>>>(d, 10, P);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_const<<<blocks, threads>>>(d, citers, P);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * blocks * threads * (double)citers * 256;
      printf("dfma_const threads %4d blocks/SM %d : %.2f TFLOP/s (%.3f ms)\n", threads, bps, flops / ms / 1e9, ms);
      int miters = 4000;
      dmma_bench<<<blocks, threads>>>(d, 10);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_bench<<<blocks, threads>>>(d, miters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 256 * (blocks * threads / 32) * (double)miters * 8 * NMMA;
      printf("dmma       threads %4d blocks/SM %d : %.2f TFLOP/s (%.3f ms)\n", threads, bps, flops / ms / 1e9, ms);
    }
  }
  // long sustained run for the clock record
  cudaEventRecord(e0);
  for (int rep = 0; rep < 20; ++rep) dfma_reg<<<sms * 2, 1024>>>(d, 20000, 1.0000001, 1e-9);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("dfma_reg sustained: %.2f TFLOP/s over %.1f ms\n", 20 * 2.0 * sms * 2 * 1024 * 20000.0 * 16 * NACC / ms / 1e9, ms);
  cudaEventRecord(e0);
  for (int rep = 0; rep < 20; ++rep) dmma_bench<<<sms * 2, 1024>>>(d, 4000);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  printf("dmma sustained: %.2f TFLOP/s over %.1f ms\n", 20 * 2.0 * 256 * (sms * 2 * 1024 / 32) * 4000.0 * 8 * NMMA / ms / 1e9, ms);
  return 0;
}
