// mma_mask.cuh -- register masking of bf16 operands + the legacy-HMMA wrapper used by the
// decode regime (a3/a4 of the hot path): M_i (.) W is built in registers from the packed codes.
#pragma once
#include "common.cuh"

namespace mglu {

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

__device__ __forceinline__ void mma_16816(float (&acc)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// 32-bit AND-mask for the bf16 pair (elements 2Q, 2Q+1 of a thread's 16) under mask I (0-based):
// low half = 0xffff iff bit I of code(2Q), high half = 0xffff iff bit I of code(2Q+1).
// Codes of the 16 elements form a 16*NM-bit string cw[] (element e, mask I at bit NM*e + I).
// Shift the bit to the MSB of its byte, then PRMT with sign-replicate selectors (bit 3 of each
// selector nibble) copies that MSB over two bytes.
template <int NM, int Q, int I>
__device__ __forceinline__ uint32_t mask_word(const uint32_t* cw) {
  constexpr int b0 = NM * (2 * Q) + I, b1 = NM * (2 * Q + 1) + I;
  constexpr int w0 = b0 >> 5, w1 = b1 >> 5;
  constexpr int sh0 = 7 - (b0 & 7), sh1 = 7 - (b1 & 7);
  constexpr uint32_t y0 = (b0 & 31) >> 3, y1 = (b1 & 31) >> 3;
  constexpr uint32_t sel = (8u | y0) | ((8u | y0) << 4) | ((12u | y1) << 8) | ((12u | y1) << 12);
  return prmt(cw[w0] << sh0, cw[w1] << sh1, sel);
}

template <int NM>
__device__ __forceinline__ void codes_from_u4(uint4 v, uint32_t (&c)[4]) {
  c[0] = v.x; c[1] = v.y; c[2] = v.z; c[3] = v.w;
}

}  // namespace mglu
