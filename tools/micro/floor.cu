// Latency floor of a dependent kernel chain on B200 (graph replay, with and
// without programmatic dependent launch): empty kernels, and kernels that
// stream the C2 top-level traffic (read 8 MB + write 8 MB / 2 MB).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, int n, int shrink) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int stride = gridDim.x * blockDim.x;
  for (int k = i; k < n / 2; k += stride) {
    const double2 v = reinterpret_cast<const double2*>(a)[k];
    if (!shrink) reinterpret_cast<double2*>(b)[k] = make_double2(v.x + 1.0, v.y + 1.0);
    else if ((k & 3) == 0) b[k >> 1] = v.x + v.y;
  }
}

template <typename F>
float graph_time(F body, int reps) {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  body(s);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

template <typename... KArgs, typename... Args>
void launch(bool pdl, void (*k)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
}

int main() {
  const int n = 1 << 20;  // 8 MB of doubles
  double *a, *b;
  cudaMalloc(&a, 8 * n);
  cudaMalloc(&b, 8 * n);
  cudaMemset(a, 0, 8 * n);
  const int L = 20;
  for (int pdl = 0; pdl < 2; ++pdl) {
    float t = graph_time([&](cudaStream_t s) { for (int i = 0; i < L; ++i) launch(pdl, k_empty, 1024, 256, s, 0); }, 50);
    printf("pdl=%d  empty kernel x%d: %.2f us per kernel\n", pdl, L, 1e3 * t / L);
    t = graph_time([&](cudaStream_t s) { for (int i = 0; i < L; ++i) launch(pdl, k_copy, 1024, 256, s, (const double*)a, b, n, 0); }, 50);
    printf("pdl=%d  8MB read + 8MB write (L2-resident) x%d: %.2f us per kernel\n", pdl, L, 1e3 * t / L);
    t = graph_time([&](cudaStream_t s) { for (int i = 0; i < L; ++i) launch(pdl, k_copy, 1024, 256, s, (const double*)a, b, n, 1); }, 50);
    printf("pdl=%d  8MB read + 2MB write (L2-resident) x%d: %.2f us per kernel\n", pdl, L, 1e3 * t / L);
    t = graph_time([&](cudaStream_t s) { for (int i = 0; i < L; ++i) launch(pdl, k_copy, 148 * 8, 512, s, (const double*)a, b, n, 0); }, 50);
    printf("pdl=%d  8MB+8MB, 1184x512 threads x%d: %.2f us per kernel\n", pdl, L, 1e3 * t / L);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
