// Grid-barrier cost on B200: cooperative_groups grid.sync() vs a hand-rolled
// arrive/spin barrier (one atomic per CTA, generation counter).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_own(unsigned* ctr, int iters) {
  unsigned target = 0;
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      while (ld_acquire(ctr) < target) {}
    }
    __syncthreads();
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* ctr;
  cudaMalloc(&ctr, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int threads : {256, 512, 1024}) {
    for (int per : {1, 2}) {
      if (threads * per > 2048) continue;
      int grid = sms * per, iters = 1000;
      void* args[] = {&iters};
      cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("cg grid.sync   grid=%4d threads=%4d: %.3f us/barrier\n", grid, threads, 1e3 * ms / iters);
      cudaMemset(ctr, 0, 4);
      void* args2[] = {&ctr, &iters};
      cudaLaunchCooperativeKernel((void*)k_own, grid, threads, args2, 0, 0);
      cudaMemset(ctr, 0, 4);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_own, grid, threads, args2, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("own barrier    grid=%4d threads=%4d: %.3f us/barrier  (%s)\n", grid, threads, 1e3 * ms / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
