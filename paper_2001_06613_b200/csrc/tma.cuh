// tma.cuh — the small set of sm_90+/sm_100a asynchronous-copy and barrier primitives the
// warp-specialized kernels use: 1-D TMA bulk copies (cp.async.bulk) completing on an
// mbarrier, mbarrier init/arrive/wait, and named CTA barriers for producer/consumer warps.
#pragma once
#include <stdint.h>

namespace sr {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

// make the mbarrier inits visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared (TMA), completion signalled on `bar` as transaction bytes.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Named barriers (ids 1..15; 0 is __syncthreads)
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace sr

#include <cuda.h>

namespace sr {

// 2-D tiled TMA load: box at element coordinates (x = inner, y = row) of a tensor map.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace sr

namespace sr {

// Bulk L2 prefetch (TMA engine, fire-and-forget).  addr 16-byte aligned, bytes multiple of 16.
__device__ __forceinline__ void l2_prefetch_bulk(const void* addr, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(addr), "r"(bytes) : "memory");
}

// Spread an L2 warm-up of the subset frames over the grid: CTA `cta` of `nctas` prefetches its
// contiguous share of the concatenated frames (each piece inside one frame, <= 64 KiB).
template <typename T>
__device__ __forceinline__ void prefetch_frames_l2(const T* frames, const int* frame_index, int K, long long N,
                                                   int cta, int nctas) {
  const long long fbytes = N * (long long)sizeof(T);
  if ((fbytes & 15) || (reinterpret_cast<uintptr_t>(frames) & 15)) return;
  const long long total = fbytes * K;
  long long chunk = (total + nctas - 1) / nctas;
  chunk = (chunk + 15) & ~15LL;
  long long lo = (long long)cta * chunk, hi = lo + chunk < total ? lo + chunk : total;
  while (lo < hi) {
    const int k = (int)(lo / fbytes);
    const long long off = lo - (long long)k * fbytes;
    long long n = fbytes - off;
    if (n > hi - lo) n = hi - lo;
    if (n > 65536) n = 65536;
    const char* base = reinterpret_cast<const char*>(frames + (long long)frame_index[k] * N);
    l2_prefetch_bulk(base + off, (uint32_t)n);
    lo += n;
  }
}

}  // namespace sr
