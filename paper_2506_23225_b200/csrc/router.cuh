// router.cuh -- Top-K routing of the routed MGLU variant (Appendix B,
// P:711-730): l = x W_r, G = Softmax(TopK(l)).  One CTA per token: the n_m logits are fp32 dot
// products over d (bf16 inputs, 256 threads stride 8-element groups, warp shuffles and a fixed-order
// cross-warp sum), then one thread keeps the K largest (ties -> lowest index, reading R17) and writes their
// softmax weights (over the K kept logits only, R18) and zeros elsewhere.
#pragma once
#include "common.cuh"

namespace mglu {

template <int NM>
__global__ void __launch_bounds__(256)
router_topk_kernel(const __nv_bfloat16* __restrict__ x, int B, int d, const __nv_bfloat16* __restrict__ Wr, int K,
                   float* __restrict__ G) {
  // one CTA per token: 256 threads split d in 8-element groups, then a fixed-order block reduction
  __shared__ float red[8][NM];
  pdl_wait();                                              // x may be the predecessor's output
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.x;
  float l[NM];
#pragma unroll
  for (int i = 0; i < NM; ++i) l[i] = 0.f;
  const __nv_bfloat16* xb = x + (size_t)b * d;
  for (int k = threadIdx.x * 8; k < d; k += 256 * 8) {     // d % 32 == 0 (handle); 8-element groups
    const uint4 xv = *reinterpret_cast<const uint4*>(xb + k);
    const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      const uint4 wv = *reinterpret_cast<const uint4*>(Wr + (size_t)i * d + k);
      const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        l[i] = fmaf(bf16lo(xw[q]), bf16lo(ww[q]), l[i]);
        l[i] = fmaf(bf16hi(xw[q]), bf16hi(ww[q]), l[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NM; ++i) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l[i] += __shfl_xor_sync(0xffffffffu, l[i], off);
    if (lane == 0) red[warp][i] = l[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      l[i] = red[0][i];
      for (int w = 1; w < 8; ++w) l[i] += red[w][i];
    }
    // TopK: K passes of "largest remaining, lowest index on ties"
    uint32_t kept = 0u;
    for (int r = 0; r < K; ++r) {
      int best = -1;
#pragma unroll
      for (int i = 0; i < NM; ++i)
        if (!((kept >> i) & 1u) && (best < 0 || l[i] > l[best])) best = i;
      kept |= 1u << best;
    }
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < NM; ++i)
      if ((kept >> i) & 1u) mx = fmaxf(mx, l[i]);
    float e[NM], sum = 0.f;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      e[i] = ((kept >> i) & 1u) ? expf(l[i] - mx) : 0.f;
      sum += e[i];
    }
#pragma unroll
    for (int i = 0; i < NM; ++i) G[(size_t)b * NM + i] = e[i] / sum;
  }
  pdl_launch_dependents();
}

}  // namespace mglu
