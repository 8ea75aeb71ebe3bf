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

// Sign-flip masking of a bf16 pair (reading R3 layout).  With sigma = +1 where M_i = 1 (gate)
// and -1 where M_i = 0 (value), the tensor core accumulates u_i = x (sigma (.) W) = s_i - v_i, and
// the epilogue recovers s_i = (t + u_i) / 2, v_i = (t - u_i) / 2 (exact rescaling of the same
// products).  The two mask bits of the pair's columns sit 16 bits apart in the layout word, so
// ONE multiply (FMA pipe) by 2^(15 - bit) brings them to bf16 sign positions 15 and 31 and ONE
// LOP3 (ALU pipe) flips the signs of the value-side elements: W ^ (~S & 0x80008000).
__device__ __forceinline__ uint32_t sign_flip(uint32_t w_pair, uint32_t word, uint32_t mult) {
  uint32_t sh;
  // inline PTX keeps this an IMAD on the FMA pipe (a C++ multiply by a known power of two is
  // strength-reduced to SHF on the ALU pipe, which the LOP3s already load)
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(sh) : "r"(word), "r"(mult));
  return w_pair ^ (~sh & 0x80008000u);
}

}  // namespace mglu
