// gemv_simt.cuh -- CUDA-core fused masked GEMV (the SIMT regime).
//
// Alg. 1 re-laid out for sm_100a without split-K (reading R9 / SURVEY a9): one warp
// owns an output row j of Wt and reduces its whole K range on chip, so the epilogue fuses and
// the result is deterministic.  Per element: load Wt[j,k], x[b,k] and the packed
// code c[j,k]; v = Wt[j,k]*x[b,k]; t += v; s_i += v iff bit (i-1) of c[j,k] is set.  Then a
// warp-shuffle reduction and the fused epilogue y = sum_i g(s_i)(t - s_i)
// (Eq. 3), or Alg. 1's z accumulators in partials mode.
//
// This regime serves fp32 (the tiny config, 1e-5), the debug partials entry point and any B;
// the bf16 decode hot path is the register-masked MMA regime (gemv_mma.cuh).
#pragma once
#include "common.cuh"

namespace mglu {

// Eight consecutive elements of one row (weights or x) as fp32.
template <typename T> struct Row8;
template <> struct Row8<__nv_bfloat16> {
  __device__ static void load(const __nv_bfloat16* p, float (&w)[8]) {
    uint4 v = ld_nc_v4(p);
    w[0] = bf16lo(v.x); w[1] = bf16hi(v.x); w[2] = bf16lo(v.y); w[3] = bf16hi(v.y);
    w[4] = bf16lo(v.z); w[5] = bf16hi(v.z); w[6] = bf16lo(v.w); w[7] = bf16hi(v.w);
  }
  __device__ static void load_x(const __nv_bfloat16* p, float (&w)[8]) {
    uint4 v = *reinterpret_cast<const uint4*>(p);
    w[0] = bf16lo(v.x); w[1] = bf16hi(v.x); w[2] = bf16lo(v.y); w[3] = bf16hi(v.y);
    w[4] = bf16lo(v.z); w[5] = bf16hi(v.z); w[6] = bf16lo(v.w); w[7] = bf16hi(v.w);
  }
};
template <> struct Row8<float> {
  __device__ static void load(const float* p, float (&w)[8]) {
    uint4 a = ld_nc_v4(p), b = ld_nc_v4(p + 4);
    w[0] = __uint_as_float(a.x); w[1] = __uint_as_float(a.y); w[2] = __uint_as_float(a.z); w[3] = __uint_as_float(a.w);
    w[4] = __uint_as_float(b.x); w[5] = __uint_as_float(b.y); w[6] = __uint_as_float(b.z); w[7] = __uint_as_float(b.w);
  }
  __device__ static void load_x(const float* p, float (&w)[8]) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
  }
};

// Mask words of the 32-column group holding 8 consecutive elements (reading R3 layout): n_m
// little-endian u32 words, column 32g + e of mask i at bit (e >> 1) + 16*(e & 1) of word i.
template <int NM>
__device__ __forceinline__ void load_group_words(const uint32_t* p, uint32_t (&w)[NM]) {
#pragma unroll
  for (int i = 0; i < NM; ++i) w[i] = ld_nc_u32(p + i);
}

constexpr int kSimtTok = 4;   // tokens accumulated per pass over a row

template <typename T, int NM, int ACT, bool PARTIALS>
__global__ void __launch_bounds__(256)
gemv_simt_kernel(const T* __restrict__ x, int B, int d, const T* __restrict__ Wt,
                 const uint8_t* __restrict__ codes, int h, T* __restrict__ out,
                 float* __restrict__ z, const float* __restrict__ G, int variant, int act) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int warps_total = gridDim.x * (blockDim.x >> 5);
  const int ngroups = d >> 3;   // 8-element groups per row
  for (int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < h; j += warps_total) {
    const T* wrow = Wt + (size_t)j * d;
    const uint32_t* crow = reinterpret_cast<const uint32_t*>(codes) + (size_t)j * (d / 32) * NM;
    for (int b0 = 0; b0 < B; b0 += kSimtTok) {
      const int nb = min(kSimtTok, B - b0);
      float t[kSimtTok], s[kSimtTok][NM];
#pragma unroll
      for (int b = 0; b < kSimtTok; ++b) {
        t[b] = 0.f;
#pragma unroll
        for (int i = 0; i < NM; ++i) s[b][i] = 0.f;
      }
      for (int g = lane; g < ngroups; g += 32) {
        float w[8];
        Row8<T>::load(wrow + g * 8, w);
        uint32_t cw[NM];
        load_group_words<NM>(crow + (size_t)(g >> 2) * NM, cw);
        const int e0 = (g & 3) * 8;                         // first column of the 8 in the group
#pragma unroll
        for (int b = 0; b < kSimtTok; ++b) {
          if (b < nb) {
            float xv[8];
            Row8<T>::load_x(x + (size_t)(b0 + b) * d + g * 8, xv);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float v = w[e] * xv[e];                 // P:218 v = A[row,k] * x[k]
              t[b] += v;                                    // P:219 t = t + v
              const int bit = ((e0 + e) >> 1) + 16 * (e & 1);   // e0 even
#pragma unroll
              for (int i = 0; i < NM; ++i)                  // P:220-222 bit test, s_i += v
                if ((cw[i] >> bit) & 1u) s[b][i] += v;
            }
          }
        }
      }
      // P:225 reduce across the warp
#pragma unroll
      for (int b = 0; b < kSimtTok; ++b) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          t[b] += __shfl_xor_sync(0xffffffffu, t[b], off);
#pragma unroll
          for (int i = 0; i < NM; ++i) s[b][i] += __shfl_xor_sync(0xffffffffu, s[b][i], off);
        }
      }
      if (lane == 0) {
#pragma unroll
        for (int b = 0; b < kSimtTok; ++b) {
          if (b < nb) {
            if constexpr (PARTIALS) {
              float* zb = z + (size_t)(b0 + b) * 2 * NM * h;
#pragma unroll
              for (int i = 0; i < NM; ++i) {
                zb[(size_t)i * h + j] = s[b][i];               // z[i]      = s_i
                zb[(size_t)(NM + i) * h + j] = t[b] - s[b][i]; // z[n_m+i]  = t - s_i
              }
            } else {
              IoT<T>::store(out + (size_t)(b0 + b) * h + j,
                            mglu_epilogue_v<ACT, NM>(t[b], s[b], G ? G + (size_t)(b0 + b) * NM : nullptr, variant, act));
            }
          }
        }
      }
    }
  }
  pdl_launch_dependents();
}

}  // namespace mglu
