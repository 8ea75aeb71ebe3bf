// tma.cuh -- mbarrier + TMA (cp.async.bulk.tensor) primitives for sm_100a, inline PTX.
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace mglu {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// expect `bytes` more transaction bytes on the current phase without arriving (a later arrive
// completes the phase once all expected bytes have landed)
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
  return ok != 0;
}
// Blocking wait with a watchdog: a pipeline that stops making progress (a protocol bug) traps
// after ~2^28 polls -- seconds, far beyond any legitimate stage time -- instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t polls = 0;
  while (!mbar_try_wait(b, parity)) {
    if (++polls == (1u << 28)) __trap();
  }
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
}
// 2-D tiled TMA load global -> shared, completion counted on `bar` (bytes)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}
// same with an L2 cache-policy hint (evict-first for read-once weight streams)
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
// 3-D tiled TMA load (coordinates innermost first) with an L2 cache-policy hint
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;"
      ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
// 3-D tiled TMA load without a cache hint (re-read operands such as x)
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)) : "memory");
}
// L2 prefetch of a 3-D tiled box (no shared-memory destination, no completion)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
               ::"l"(map), "r"(x), "r"(y), "r"(z) : "memory");
}
// 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16), counted on `bar`
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// N consecutive u32 mask words starting at byte `lin` of a TMA box whose rows are `rb` bytes,
// loaded with the swizzle code_swizzle_bytes(rb) (32/64/128-byte rows: that swizzle, else none):
// 16-byte chunk c of a 1024-byte-aligned region lands at chunk c ^ ((lin >> 7) & (rb / 16 - 1)).
// The words of one chunk keep their order, so each chunk is one vector load.
__host__ __device__ constexpr int code_swizzle_bytes(int rb) { return rb == 128 ? 128 : rb == 64 ? 64 : rb == 32 ? 32 : 0; }
template <int N>
__device__ __forceinline__ void lds_words_swz(const uint8_t* base, uint32_t lin, uint32_t rb, uint32_t (&w)[N]) {
  const uint32_t sw = (uint32_t)code_swizzle_bytes((int)rb);
  const uint32_t mask = sw ? sw / 16 - 1 : 0;
  auto at = [&](uint32_t l) { return base + (l ^ (((l >> 7) & mask) << 4)); };
  if constexpr (N == 1) w[0] = *reinterpret_cast<const uint32_t*>(at(lin));
  else if constexpr (N == 2) { const uint2 v = *reinterpret_cast<const uint2*>(at(lin)); w[0] = v.x; w[1] = v.y; }
  else {
#pragma unroll
    for (int q = 0; q < N / 4; ++q) {
      const uint4 v = *reinterpret_cast<const uint4*>(at(lin + 16 * q));
      w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
  }
}

// named barrier over a subset of warps
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace mglu
