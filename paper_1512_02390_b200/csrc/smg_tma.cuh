// TMA (cp.async.bulk.tensor) and mbarrier helpers for libsmg (sm_100a).
//
// The fields are row-major (N_y, N_x) float64 arrays; a 2D tensor map over
// one of them moves a (box_h x box_w) rectangle between HBM and shared memory
// with ONE instruction issued by one thread, instead of one cp.async per node.
// Out-of-range box parts are zero-filled by the hardware (periodic wrap is
// NOT available in TMA; callers take a per-node path for seam tiles).
#pragma once
#include <cuda.h>

#include "smg_common.cuh"

namespace smg {

// Encode a 2D float64 tensor map over base[(H, W)] with a (box_h, box_w) box.
// Returns false (and sets the error string) when TMA cannot describe the
// array: W*8 not a multiple of 16, base not 16-byte aligned, box too large.
bool tmap_2d(CUtensorMap* map, const double* base, int W, int H, int box_w, int box_h);

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

// Generic-proxy shared-memory writes -> visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void tma_load_2d(double* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// L2 prefetch of a box (no shared-memory destination, no completion to wait for).
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];\n" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y)
               : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const double* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }

// Wait until all but the N most recent committed bulk stores have finished
// READING shared memory.
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory"); }

// Wait until all but the N most recent committed bulk stores have completed.
template <int N>
__device__ __forceinline__ void bulk_wait_group() { asm volatile("cp.async.bulk.wait_group %0;\n" ::"n"(N) : "memory"); }

// Wait until every committed bulk store has completed (writes performed).
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// 1D bulk copy global -> shared (16-byte aligned addresses, size % 16 == 0),
// completing on bar (complete_tx).
__device__ __forceinline__ void bulk_g2s(double* dst, const double* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Row width (doubles) that pwin_load_warp moves per window row.
__host__ __device__ constexpr int pwin_width(int W, int sh) { return (W + sh + 1) & ~1; }

// Periodic window loader, issued by the 32 lanes of ONE warp: rows
// [y0, y0+H) x columns [x0, x0+W) of the periodic field f (N_y x N_x, N_x
// even, |x0| < N_x) land in dst with row pitch DP (even, >= pwin_width);
// window column j of row r is dst[r*DP + pwin_shift(x0, N_x) + j] (bulk
// copies move 16-byte aligned pieces).  One copy per row, two where the row
// wraps around the seam (the piece past the seam restarts at column 0 of the
// same row).  The caller arms the mbarrier with pwin_bytes() beforehand.
__host__ __device__ __forceinline__ int pwin_shift(int x0, int N_x) { return (x0 < 0 ? x0 + N_x : x0) & 1; }
__host__ __device__ __forceinline__ unsigned pwin_bytes(int W, int H, int sh) {
  return (unsigned)(H * pwin_width(W, sh) * 8);
}
__device__ __forceinline__ void pwin_issue_warp(const double* __restrict__ f, int N_x, int N_y, int x0, int y0, int W,
                                                int H, double* dst, int DP, uint64_t* bar) {
  const int lane = threadIdx.x & 31;
  const int xs = x0 < 0 ? x0 + N_x : (x0 >= N_x ? x0 - N_x : x0);
  const int sh = xs & 1, xa = xs - sh;
  const int width = pwin_width(W, sh);
  const int lenA = min(width, N_x - xa);
  for (int r = lane; r < H; r += 32) {
    int gy = y0 + r;
    gy = gy < 0 ? gy + N_y : (gy >= N_y ? gy - N_y : gy);
    const double* row = f + (size_t)gy * N_x;
    double* d = dst + r * DP;
    bulk_g2s(d, row + xa, (unsigned)(lenA * 8), bar);
    if (lenA < width) bulk_g2s(d + lenA, row, (unsigned)((width - lenA) * 8), bar);
  }
}

}  // namespace smg
