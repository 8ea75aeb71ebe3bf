// pack.cuh -- a1 (offline binarise + pack) on the device.
// Dense code layout (reading R3): element e = j*d + k has its n_m-bit code at stream bits
// [n_m*e, n_m*e + n_m), little-endian within bytes; mask i is bit (i-1) of the code.
// n_m in {1,2,4,8}, so a code never straddles a byte: byte e/(8/n_m), shift (e % (8/n_m))*n_m.
#pragma once
#include "common.cuh"

namespace mglu {

// bits [n_m][h][d] (0/1) or logits [n_m][h][d] (bit = logit > 0) -> packed, one thread per byte
template <typename SRC>
__global__ void pack_kernel(const SRC* __restrict__ src, int n_m, int64_t hd, uint8_t* __restrict__ packed,
                            int64_t nbytes, int* __restrict__ bad) {
  const int per = 8 / n_m;
  for (int64_t byte = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; byte < nbytes;
       byte += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (int q = 0; q < per; ++q) {
      const int64_t e = byte * per + q;
      if (e >= hd) break;
      for (int i = 0; i < n_m; ++i) {
        const SRC s = src[(int64_t)i * hd + e];
        uint32_t bit;
        if constexpr (sizeof(SRC) == 1) {
          bit = (uint32_t)s;
          if (bit > 1u && bad) atomicOr(bad, 1);
        } else {
          bit = (s > 0.0f) ? 1u : 0u;   // strict threshold (Alg. 2 "(soft_mask > 0)", R4)
        }
        v |= (bit & 1u) << (q * n_m + i);
      }
    }
    packed[byte] = (uint8_t)v;
  }
}

// packed -> bits [n_m][h][d], one thread per element
__global__ void unpack_kernel(const uint8_t* __restrict__ packed, int n_m, int64_t hd,
                              uint8_t* __restrict__ bits) {
  const int per = 8 / n_m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < hd; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t byte = packed[e / per];
    const uint32_t code = (byte >> ((e % per) * n_m)) & ((1u << n_m) - 1u);
    for (int i = 0; i < n_m; ++i) bits[(int64_t)i * hd + e] = (uint8_t)((code >> i) & 1u);
  }
}

}  // namespace mglu
