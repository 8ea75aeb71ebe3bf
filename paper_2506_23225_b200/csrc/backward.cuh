// backward.cuh -- the training path of MGLU: Eq. 3's gradients under Alg. 2's
// straight-through estimator (reading R21 in DESIGN.md).
//
// With the forward streams s_i = x (M_i (.) W), v_i = x (Mbar_i (.) W) (produced by the forward
// kernels' partials mode) and the upstream gradient dy [B][h]:
//   a_i = dy g'(s_i) v_i,  c_i = dy g(s_i)            (dL/ds_i, dL/dv_i)
//   E_0 = sum_i c_i,  E_i = a_i - c_i                  (coef_kernel, [B][n_m + 1][h] fp32)
//   dL/dx[b,k]  = sum_j W[j,k] (E_0[b,j] + sum_i E_i[b,j] M_i[j,k])          (dx_kernel)
//   P_o[j,k]    = sum_b E_o[b,j] x[b,k]                                       (dw_kernel, fused:)
//   dL/dW[j,k]  = P_0[j,k] + sum_i M_i[j,k] P_i[j,k]
//   dL/dM_i[j,k] = W[j,k] P_i[j,k]      (the STE gradient handed to the soft logits unchanged)
// fp32 accumulation of exact products (bf16 or fp32 inputs), fixed summation orders (deterministic,
// no atomics).  CUDA-core kernels with shared-memory tiles: a correct, deterministic first version
// of this row; the tensor-core form is future work.
#pragma once
#include "common.cuh"
#include "pack.cuh"

namespace mglu {

// g'(z): swish' = sigma (1 + z (1 - sigma)); gelu' = Phi(z) + z phi(z); relu' = [z > 0]; sigmoid'
__device__ __forceinline__ float act_grad_rt(int act, float z) {
  switch (act) {
    case kIdentity: return 1.0f;
    case kSwish: { const float s = 1.0f / (1.0f + expf(-z)); return s * (1.0f + z * (1.0f - s)); }
    case kGelu: return 0.5f * (1.0f + erff(z * 0.70710678118654752f)) + z * expf(-0.5f * z * z) * 0.39894228040143268f;
    case kRelu: return z > 0.0f ? 1.0f : 0.0f;
    default: { const float s = 1.0f / (1.0f + expf(-z)); return s * (1.0f - s); }
  }
}

template <typename T> __device__ __forceinline__ float ld_f(const T* p);
template <> __device__ __forceinline__ float ld_f<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// mask bit M_i[j][k] of the packed layout (reading R3)
__device__ __forceinline__ uint32_t mask_bit(const uint32_t* codes, int n_m, int d, int j, int k, int i) {
  return (codes[((size_t)j * (d / 32) + k / 32) * n_m + i] >> code_bit_of(k & 31)) & 1u;
}

// z [B][2 n_m][h] (s_i, v_i) + dy [B][h] -> E [B][n_m + 1][h]
__global__ void coef_kernel(const float* z, const float* dy, int B, int h, int n_m, int act, float* E) {
  const int64_t total = (int64_t)B * h;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(q / h), j = (int)(q - (int64_t)b * h);
    const float g = dy[q];
    float e0 = 0.f;
    for (int i = 0; i < n_m; ++i) {
      const float s = z[((size_t)b * 2 * n_m + i) * h + j];
      const float v = z[((size_t)b * 2 * n_m + n_m + i) * h + j];
      const float a = g * act_grad_rt(act, s) * v;
      const float c = g * act_rt(act, s);
      e0 += c;
      E[((size_t)b * (n_m + 1) + 1 + i) * h + j] = a - c;
    }
    E[((size_t)b * (n_m + 1)) * h + j] = e0;
  }
}

// dW and d_logits: one CTA per (32 rows j) x (64 columns k) tile; 256 threads, thread = (row r in
// 0..31, column octet) owning 8 columns; b is reduced in chunks of 32 tokens staged in smem.
constexpr int kBwJ = 32, kBwK = 64, kBwB = 32;
template <typename T, int NM>
__global__ void __launch_bounds__(256)
dw_kernel(const T* x, const T* Wt, const uint32_t* codes, const float* E, int B, int d, int h, float* dW,
          float* dlogits) {
  constexpr int NOP = NM + 1;
  __shared__ float es[kBwB][NOP][kBwJ];
  __shared__ float xs[kBwB][kBwK];
  const int j0 = blockIdx.y * kBwJ, k0 = blockIdx.x * kBwK;
  const int r = threadIdx.x >> 3, c8 = (threadIdx.x & 7) * 8;
  float acc[NOP][8];
#pragma unroll
  for (int o = 0; o < NOP; ++o)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[o][q] = 0.f;
  for (int b0 = 0; b0 < B; b0 += kBwB) {
    for (int v = threadIdx.x; v < kBwB * NOP * kBwJ; v += 256) {
      const int bb = v / (NOP * kBwJ), o = (v / kBwJ) % NOP, jj = v % kBwJ;
      es[bb][o][jj] = (b0 + bb < B && j0 + jj < h) ? E[((size_t)(b0 + bb) * NOP + o) * h + j0 + jj] : 0.f;
    }
    for (int v = threadIdx.x; v < kBwB * kBwK; v += 256) {
      const int bb = v / kBwK, kk = v % kBwK;
      xs[bb][kk] = (b0 + bb < B && k0 + kk < d) ? ld_f<T>(x + (size_t)(b0 + bb) * d + k0 + kk) : 0.f;
    }
    __syncthreads();
    for (int bb = 0; bb < kBwB; ++bb) {
      float xv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) xv[q] = xs[bb][c8 + q];
#pragma unroll
      for (int o = 0; o < NOP; ++o) {
        const float e = es[bb][o][r];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[o][q] = fmaf(e, xv[q], acc[o][q]);
      }
    }
    __syncthreads();
  }
  const int j = j0 + r;
  if (j >= h) return;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int k = k0 + c8 + q;
    if (k >= d) break;
    const float w = ld_f<T>(Wt + (size_t)j * d + k);
    float g = acc[0][q];
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      if (mask_bit(codes, NM, d, j, k, i)) g += acc[1 + i][q];
      if (dlogits) dlogits[((size_t)i * h + j) * d + k] = w * acc[1 + i][q];
    }
    if (dW) dW[(size_t)j * d + k] = g;
  }
}

// dx: one CTA per (32 tokens b) x (64 columns k) tile; 256 threads, thread = (token r, column
// octet); the reduction over j runs in chunks of 32 rows staged in smem (W, E, mask words).
template <typename T, int NM>
__global__ void __launch_bounds__(256)
dx_kernel(const T* Wt, const uint32_t* codes, const float* E, int B, int d, int h, float* dx) {
  constexpr int NOP = NM + 1;
  __shared__ float ws[kBwJ][kBwK];
  __shared__ float es[kBwB][NOP][kBwJ + 1];
  __shared__ uint32_t ms[kBwJ][2][NM];                     // mask words of the tile's two 32-column groups
  const int b0 = blockIdx.y * kBwB, k0 = blockIdx.x * kBwK;
  const int r = threadIdx.x >> 3, c8 = (threadIdx.x & 7) * 8;
  float acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.f;
  for (int j0 = 0; j0 < h; j0 += kBwJ) {
    for (int v = threadIdx.x; v < kBwJ * kBwK; v += 256) {
      const int jj = v / kBwK, kk = v % kBwK;
      ws[jj][kk] = (j0 + jj < h && k0 + kk < d) ? ld_f<T>(Wt + (size_t)(j0 + jj) * d + k0 + kk) : 0.f;
    }
    for (int v = threadIdx.x; v < kBwB * NOP * kBwJ; v += 256) {
      const int bb = v / (NOP * kBwJ), o = (v / kBwJ) % NOP, jj = v % kBwJ;
      es[bb][o][jj] = (b0 + bb < B && j0 + jj < h) ? E[((size_t)(b0 + bb) * NOP + o) * h + j0 + jj] : 0.f;
    }
    for (int v = threadIdx.x; v < kBwJ * 2 * NM; v += 256) {
      const int jj = v / (2 * NM), gq = (v / NM) % 2, i = v % NM;
      const int gcol = k0 / 32 + gq;
      ms[jj][gq][i] = (j0 + jj < h && gcol < d / 32) ? codes[((size_t)(j0 + jj) * (d / 32) + gcol) * NM + i] : 0u;
    }
    __syncthreads();
    for (int jj = 0; jj < kBwJ; ++jj) {
      float e[NOP];
#pragma unroll
      for (int o = 0; o < NOP; ++o) e[o] = es[r][o][jj];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int kk = c8 + q;
        float coef = e[0];
#pragma unroll
        for (int i = 0; i < NM; ++i)
          if ((ms[jj][kk >> 5][i] >> code_bit_of(kk & 31)) & 1u) coef += e[1 + i];
        acc[q] = fmaf(ws[jj][kk], coef, acc[q]);
      }
    }
    __syncthreads();
  }
  const int b = b0 + r;
  if (b >= B) return;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int k = k0 + c8 + q;
    if (k < d) dx[(size_t)b * d + k] = acc[q];
  }
}

}  // namespace mglu
