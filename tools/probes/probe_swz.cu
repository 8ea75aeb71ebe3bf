// Probe: does a 1-row TMA box with SWIZZLE_128B written at (1024-aligned base + r*128) land
// exactly where the r-th row of an 8-row box written at the base lands?  (i.e. is the swizzle a
// function of the absolute smem address?)
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap m8, const __grid_constant__ CUtensorMap m1, uint16_t* out) {
  __shared__ __align__(1024) uint16_t a[8 * 64];
  __shared__ __align__(1024) uint16_t b[8 * 64];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar)), "r"(2048));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(smem_u32(a)), "l"(&m8), "r"(0), "r"(0), "r"(smem_u32(&bar)) : "memory");
    for (int r = 0; r < 8; ++r)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   :: "r"(smem_u32(b + r * 64)), "l"(&m1), "r"(0), "r"(r), "r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" :: "r"(smem_u32(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += blockDim.x) { out[i] = a[i]; out[512 + i] = b[i]; }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  uint16_t h[8 * 256];
  for (int i = 0; i < 8 * 256; ++i) h[i] = i;   // element (r, c) = r*256 + c
  uint16_t* d; CK(cudaMalloc(&d, sizeof(h))); CK(cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice));
  uint16_t* o; CK(cudaMalloc(&o, 2048));
  void* fn; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)fn;
  CUtensorMap m8, m1;
  cuuint64_t dims[2] = {256, 8}, str[1] = {512};
  cuuint32_t b8[2] = {64, 8}, b1[2] = {64, 1}, es[2] = {1, 1};
  if (enc(&m8, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, b8, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
      enc(&m1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, b1, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) { printf("encode failed\n"); return 1; }
  k<<<1, 128>>>(m8, m1, o);
  CK(cudaDeviceSynchronize());
  uint16_t r[1024]; CK(cudaMemcpy(r, o, 2048, cudaMemcpyDeviceToHost));
  int same = 0, formula = 0;
  for (int i = 0; i < 512; ++i) same += r[i] == r[512 + i];
  // expected SW128: element (row, col) at byte addr row*128 + ((col*2/16) ^ row)*16 + (col*2)%16
  for (int row = 0; row < 8; ++row)
    for (int col = 0; col < 64; ++col) {
      int byte = row * 128 + ((((col * 2) >> 4) ^ row) << 4) + ((col * 2) & 15);
      formula += r[byte / 2] == row * 256 + col;
    }
  printf("8-row box vs 1-row boxes identical: %d/512; matches SW128 formula: %d/512\n", same, formula);
  printf("row1 first 16 elements (8-row box): "); for (int i = 0; i < 16; ++i) printf("%d ", r[64 + i]); printf("\n");
  printf("row1 first 16 elements (1-row box): "); for (int i = 0; i < 16; ++i) printf("%d ", r[512 + 64 + i]); printf("\n");
  return 0;
}
