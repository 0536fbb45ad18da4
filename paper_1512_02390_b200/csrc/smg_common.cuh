// Shared helpers for libsmg (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>

#include "../../include/smg.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libsmg targets sm_100a only"
#endif

namespace smg {

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* where);

void count_launch();

bool sync_check_enabled();  // SMG_SYNC_CHECK=1: synchronize after every launch (debug aid)

// Return SMG_ECUDA with the pending launch error, if any (and count the launch).
inline int check_launch(const char* where) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && sync_check_enabled()) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, where);
  return SMG_OK;
}

// Per-device one-time state.  Kernel attributes (max dynamic shared memory,
// cluster permissions) and occupancy-derived grid caps belong to a device, so
// a process that drives several GPUs through the ABI keeps one slot per
// device ordinal; the slots are atomics, so host threads may race on them
// (every writer stores the same value).
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}
template <class T>
struct PerDevice {
  std::atomic<T> v[kMaxDevices]{};
  operator T() const { return v[current_device()].load(std::memory_order_acquire); }
  PerDevice& operator=(T x) {
    v[current_device()].store(x, std::memory_order_release);
    return *this;
  }
};
using DeviceFlag = PerDevice<bool>;
using DeviceInt = PerDevice<int>;

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__host__ __device__ __forceinline__ int wrapi(int i, int n) {
  // periodic index for i in [-n, 2n)
  return i < 0 ? i + n : (i >= n ? i - n : i);
}

// Deterministic block reduction of NV doubles (fixed tree order).
template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV], double* sbuf /*32*NV*/) {
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) sbuf[k * 32 + wid] = v[k];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double t = lane < nw ? sbuf[k * 32 + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      v[k] = t;
    }
  }
}

// ---- programmatic dependent launch (PDL) ------------------------------------
// Every libsmg kernel starts with SMG_PDL_ENTRY(): it waits until the
// preceding grid on the stream has completed and flushed (griddepcontrol.wait)
// before touching global memory, then lets the next grid begin launching
// (griddepcontrol.launch_dependents).  Launched with the programmatic
// stream-serialization attribute, a dependent grid's CTAs are scheduled while
// the previous grid drains, hiding the launch/ramp latency that dominates the
// small per-level kernels of a V-cycle.  SMG_PDL=0 disables the attribute.
#define SMG_PDL_ENTRY()                                            \
  do {                                                             \
    asm volatile("griddepcontrol.wait;\n" ::: "memory");           \
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); \
  } while (0)

// Split form for kernels with a prologue that reads nothing the preceding
// grid writes (constant tables, mbarrier setup): SMG_PDL_TRIGGER() first, the
// prologue, then SMG_PDL_WAIT() before the first dependent global access --
// the prologue overlaps the previous kernel's tail.
#define SMG_PDL_TRIGGER() asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory")
#define SMG_PDL_WAIT() asm volatile("griddepcontrol.wait;\n" ::: "memory")

bool pdl_enabled();
// Integer tuning knob from the environment (read once per name by the caller).
int env_int(const char* name, int def);

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (pdl && pdl_enabled()) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args&&... args) {
  return launch_pdl(true, kern, grid, block, smem, st, std::forward<Args>(args)...);
}

// Meshes from this many elements up launch the persistent tensor-core operator kernels (and
// their fixups) as ordinary stream-ordered grids: the early launch pays on the latency-bound
// levels, but at C5 (512^2 elements) it cost 4-25 % of these kernels (B200, PDL on -> off:
// p = 24 residual 1553 -> 1481 us, p = 12 residual + restriction 934 -> 694 us).
constexpr int kPdlMaxElements = 16384;

constexpr int kReduceBlocks = 592;   // 4 x 148 SMs: fixed => deterministic
constexpr int kReduceThreads = 512;

}  // namespace smg
