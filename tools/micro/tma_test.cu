// Standalone check of the smg_tma.cuh helpers: TMA box load -> smem -> TMA
// store, with a small and a > 4 KB __grid_constant__ parameter block.
#include <cstdio>
#include <vector>

#include "../../paper_1512_02390_b200/csrc/smg_tma.cuh"

namespace smg {
void set_error(const char*, ...) {}
int cuda_fail(cudaError_t, const char*) { return -3; }
void count_launch() {}
bool pdl_enabled() { return false; }
}  // namespace smg
using namespace smg;

template <int PAD>
struct Args {
  CUtensorMap in, out;
  int x, y, bw, bh;
  double pad[PAD];
};

template <int PAD>
__global__ void k(const __grid_constant__ Args<PAD> A) {
  extern __shared__ unsigned char raw[];
  double* sm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 4096 * 4);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, A.bw * A.bh * 8);
    tma_load_2d(sm, &A.in, A.x, A.y, bar);
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < A.bw * A.bh; i += blockDim.x) sm[i] *= 2.0;
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_2d(&A.out, sm, A.x, A.y);
    bulk_commit();
    bulk_wait0();
  }
}

template <int PAD>
int run(const char* name, int W = 256, int H = 128, int BW = 68, int BH = 35, int X = 10, int Y = 7) {
  std::vector<double> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = i;
  double *din, *dout;
  cudaMalloc(&din, 8 * W * H);
  cudaMalloc(&dout, 8 * W * H);
  cudaMemcpy(din, h.data(), 8 * W * H, cudaMemcpyHostToDevice);
  cudaMemset(dout, 0, 8 * W * H);
  Args<PAD> A;
  if (!tmap_2d(&A.in, din, W, H, BW, BH) || !tmap_2d(&A.out, dout, W, H, BW, BH)) { printf("encode failed\n"); return 1; }
  A.x = X; A.y = Y; A.bw = BW; A.bh = BH;
  const int smem = 4096 * 4 * 8 + 256;
  cudaFuncSetAttribute(k<PAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<PAD><<<1, 128, smem>>>(A);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<double> o(W * H);
  cudaMemcpy(o.data(), dout, 8 * W * H, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const bool in = x >= X && x < X + BW && y >= Y && y < Y + BH;
      const double want = in ? 2.0 * (y * W + x) : 0.0;
      if (o[y * W + x] != want) ++bad;
    }
  printf("%s W=%d box=%dx%d at (%d,%d): sizeof(Args)=%zu err=%s bad=%d\n", name, W, BW, BH, X, Y, sizeof(Args<PAD>), cudaGetErrorString(e), bad);
  return 0;
}

int main() {
  run<4>("small");
  run<700>("large");
  run<700>("prod", 1024, 1024, 68, 35, 63, 31);
  run<700>("prod8", 128, 128, 20, 19, 15, 15);
  run<700>("u", 1024, 1024, 64, 32, 64, 32);
  run<700>("odd", 1024, 1024, 68, 35, 63, 31);
  return 0;
}
