// pack.cuh -- a1 (offline binarise + pack) on the device.
// Packed layout (reading R3): for row j, 32-column group g and mask i (0-based here), one
// little-endian u32 word at word index (j*(d/32) + g)*n_m + i holds M_{i+1}[j, 32g..32g+31];
// column 32g + e sits at bit (e >> 1) + 16*(e & 1) (even columns in the low half-word, odd
// columns in the high half-word).  n_m bits per weight; d % 32 == 0.
#pragma once
#include "common.cuh"

namespace mglu {

__host__ __device__ __forceinline__ int code_bit_of(int e) { return (e >> 1) + 16 * (e & 1); }

// bits [n_m][h][d] (0/1, low bit used) or logits [n_m][h][d] (bit = logit > 0) -> packed words,
// one thread per output word
template <typename SRC>
__global__ void pack_kernel(const SRC* __restrict__ src, int n_m, int64_t h, int64_t d,
                            uint32_t* __restrict__ words) {
  const int64_t groups = d / 32, nwords = h * groups * n_m;
  const int64_t hd = h * d;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(w % n_m);
    const int64_t jg = w / n_m;
    const int64_t j = jg / groups, g = jg % groups;
    const SRC* row = src + (int64_t)i * hd + j * d + g * 32;
    uint32_t v = 0;
    for (int e = 0; e < 32; ++e) {
      uint32_t bit;
      if constexpr (sizeof(SRC) == 1) bit = (uint32_t)row[e] & 1u;
      else bit = (row[e] > 0.0f) ? 1u : 0u;     // strict threshold (Alg. 2 "(soft_mask > 0)", R4)
      v |= bit << code_bit_of(e);
    }
    words[w] = v;
  }
}

// packed words -> bits [n_m][h][d], one thread per element
__global__ void unpack_kernel(const uint32_t* __restrict__ words, int n_m, int64_t h, int64_t d,
                              uint8_t* __restrict__ bits) {
  const int64_t hd = h * d, groups = d / 32;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < hd; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / d, k = e % d;
    const uint32_t* wg = words + (j * groups + k / 32) * n_m;
    const int b = code_bit_of((int)(k % 32));
    for (int i = 0; i < n_m; ++i) bits[(int64_t)i * hd + e] = (uint8_t)((wg[i] >> b) & 1u);
  }
}

// R3 (interleaved: word (j, g, i)) -> plane-major (word (i, j, g)): one thread per word
__global__ void planes_kernel(const uint32_t* __restrict__ src, int n_m, int64_t h, int64_t groups,
                              uint32_t* __restrict__ dst) {
  const int64_t n = h * groups * n_m;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n; w += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(w % n_m);
    const int64_t jg = w / n_m;                              // j * groups + g
    dst[(int64_t)i * h * groups + jg] = src[w];
  }
}

}  // namespace mglu
