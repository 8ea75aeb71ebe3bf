// common.cuh -- device helpers shared by the libmglu kernels (sm_100a only).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libmglu targets sm_100a only (build with -gencode arch=compute_100a,code=sm_100a)"
#endif

namespace mglu {

enum Act : int { kIdentity = 0, kSwish = 1, kGelu = 2, kRelu = 3, kSigmoid = 4 };

// g of Eq. 1/3 in fp32 (reading R5).  expf/erff (not the __ intrinsics): the epilogue is a
// negligible share of the decode call and the f32 path is held to 1e-5 normwise.
// kRuntimeAct: one instantiation serves every g, chosen by a runtime code (the epilogue is a
// negligible share of every regime, so only the default Swish gets its own compile-time copy)
constexpr int kRuntimeAct = 5;

__device__ __forceinline__ float act_rt(int act, float z);

template <int ACT>
__device__ __forceinline__ float act_g(float z, int act = 0) {
  if constexpr (ACT == kRuntimeAct) return act_rt(act, z);
  else if constexpr (ACT == kIdentity) return z;
  else if constexpr (ACT == kSwish) return z / (1.0f + expf(-z));
  else if constexpr (ACT == kGelu) return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f));
  else if constexpr (ACT == kRelu) return fmaxf(z, 0.0f);
  else return 1.0f / (1.0f + expf(-z));
}

__device__ __forceinline__ float act_rt(int act, float z) {
  switch (act) {
    case kIdentity: return act_g<kIdentity>(z);
    case kSwish: return act_g<kSwish>(z);
    case kGelu: return act_g<kGelu>(z);
    case kRelu: return act_g<kRelu>(z);
    default: return act_g<kSigmoid>(z);
  }
}

// g for the bf16 tensor-core epilogues (tile GEMM, tcgen05 GEMV), which evaluate it for every
// (token, row, mask): Swish and sigmoid by ex2.approx + rcp.approx (__expf / __fdividef; relative
// error ~1e-6, far below the 2^-9 of the bf16 output) instead of expf + an IEEE division -- the
// accurate form cost 16 % of the prefill (profiles/r02/prefill_epilogue.txt).  The fp32 SIMT path
// and the HMMA decode kernel (a few outputs per thread) keep act_g.
template <int ACT>
__device__ __forceinline__ float act_fast(float z, int act = 0);
__device__ __forceinline__ float act_rt_fast(int act, float z) {
  switch (act) {
    case kSwish: return act_fast<kSwish>(z);
    case kSigmoid: return act_fast<kSigmoid>(z);
    default: return act_rt(act, z);
  }
}
template <int ACT>
__device__ __forceinline__ float act_fast(float z, int act) {
  if constexpr (ACT == kRuntimeAct) return act_rt_fast(act, z);
  else if constexpr (ACT == kSwish) return __fdividef(z, 1.0f + __expf(-z));
  else if constexpr (ACT == kSigmoid) return __fdividef(1.0f, 1.0f + __expf(-z));
  else return act_g<ACT>(z);
}

// Eq. 3 epilogue for one output: y = sum_i g(s_i) * (t - s_i)  (value = t - s_i)
// (FAST: act_fast, for the bf16 kernels; the fp32 SIMT path keeps act_g)
template <int ACT, int NM, bool FAST = false>
__device__ __forceinline__ float mglu_epilogue(float t, const float (&s)[NM], int act = 0) {
  float y = 0.0f;
#pragma unroll
  for (int i = 0; i < NM; ++i) y = fmaf((FAST ? act_fast<ACT>(s[i], act) : act_g<ACT>(s[i], act)), t - s[i], y);
  return y;
}

// Top-K routed epilogue (Appendix B): y = sum_i G_i g(s_i) (t - s_i); gw == nullptr is
// the plain Eq. 3 (every G_i = 1)
template <int ACT, int NM, bool FAST = false>
__device__ __forceinline__ float mglu_epilogue_w(float t, const float (&s)[NM], const float* gw, int act = 0) {
  if (!gw) return mglu_epilogue<ACT, NM, FAST>(t, s, act);
  float y = 0.0f;
#pragma unroll
  for (int i = 0; i < NM; ++i) y = fmaf(gw[i] * (FAST ? act_fast<ACT>(s[i], act) : act_g<ACT>(s[i], act)), t - s[i], y);
  return y;
}

// Partial-mask ablation variants (reading R20: per mask term): 1 NG gate = t,
// 2 NV value = t, 3 NM both; 0 = Eq. 3.  Optional routed weights gw.
template <int ACT, int NM, bool FAST = false>
__device__ __forceinline__ float mglu_epilogue_v(float t, const float (&s)[NM], const float* gw, int variant,
                                                 int act = 0) {
  if (variant == 0) return mglu_epilogue_w<ACT, NM, FAST>(t, s, gw, act);
  float y = 0.0f;
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    const float gate = (variant & 1) ? t : s[i];
    const float value = (variant & 2) ? t : t - s[i];
    y = fmaf((gw ? gw[i] : 1.0f) * (FAST ? act_fast<ACT>(gate, act) : act_g<ACT>(gate, act)), value, y);
  }
  return y;
}

__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_nc_v2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_nc_u32(const void* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_nc_u16(const void* p) {
  unsigned short r;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_nc_u8(const void* p) {
  unsigned short r;
  asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(r) : "l"(p));
  return r;
}

// Programmatic dependent launch: W and the codes are constant, so a kernel may stream them
// before the previous grid finishes; x (the predecessor's output) and out (which the
// predecessor may still read) are touched only after pdl_wait().
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

template <typename T> struct IoT;
template <> struct IoT<__nv_bfloat16> {
  __device__ static float load(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  __device__ static void store(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
};
template <> struct IoT<float> {
  __device__ static float load(const float* p) { return *p; }
  __device__ static void store(float* p, float v) { *p = v; }
};

}  // namespace mglu
