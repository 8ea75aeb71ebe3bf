// Probe: TMA (cp.async.bulk.tensor.2d) fed smem ring for the decode access pattern: one CTA per
// SM owns a contiguous row range; per stage a 16-row x KS-element W tile (+ its codes) lands in
// shared memory; 16 consumer warps read it (XOR) and release the slot.  Back-to-back launches
// over 4 rotating 147 MB layers.  Measures whether the pattern can stream at HBM speed.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(cnt)); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b))); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile("{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}" :: "r"(smem_u32(b)), "r"(phase));
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               :: "r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}

// KS elements of K per stage; W boxes of 16 rows x 256 elements; code box 16 rows x KS/8 u32 (n_m=4)
template <int STAGES, int KS, int ORDER>
__global__ void __launch_bounds__(17 * 32, 1)
tma_pattern(const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapC, int d, int h, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int WB = 16 * KS * 2, CB = 16 * KS / 2, SB = WB + CB;
  uint64_t* full = (uint64_t*)(smem + STAGES * SB);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int base = h / gridDim.x, rem = h % gridDim.x;
  int r0 = blockIdx.x * base + min((int)blockIdx.x, rem);
  int nrows = base + ((int)blockIdx.x < rem);
  int ntiles = (nrows + 15) / 16;
  const int all_tiles = h / 16;
  if (ORDER == 1) { r0 = blockIdx.x * 16; ntiles = (all_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x; }
  const int kst = d / KS;
  const int n = ntiles * kst;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 16); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 16) {
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (int i = 0; i < n; ++i) {
        int tile = i / kst, ks = i % kst;
        if (ORDER == 2) { tile = i % ntiles; ks = i / ntiles; }
        const int rowbase = ORDER == 1 ? (blockIdx.x + tile * gridDim.x) * 16 : r0 + tile * 16;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], SB);
        uint8_t* st = smem + s * SB;
        for (int b = 0; b < KS / 256; ++b)
          tma2d(st + b * 16 * 256 * 2, &mapW, ks * KS + b * 256, rowbase, &full[s]);
        tma2d(st + WB, &mapC, ks * KS / 8, rowbase, &full[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else {
    uint32_t acc = 0;
    int s = 0; uint32_t ph = 0;
    const int r = lane >> 2, c = lane & 3;
    for (int i = 0; i < n; ++i) {
      mbar_wait(&full[s], ph);
      const uint8_t* st = smem + s * SB;
      // warp w: k slice [64w, 64w+64) of the stage (KS = 1024)
      const int kk = warp * 64 + c * 16;
      const int box = kk / 256, kin = kk % 256;
      const uint4* pa = (const uint4*)(st + box * 8192 + r * 512 + kin * 2);
      const uint4* pb = (const uint4*)(st + box * 8192 + (r + 8) * 512 + kin * 2);
      uint4 a0 = pa[0], a1 = pa[1], b0 = pb[0], b1 = pb[1];
      const uint2* ca = (const uint2*)(st + WB + r * (KS / 2) + kk / 2);
      const uint2* cb = (const uint2*)(st + WB + (r + 8) * (KS / 2) + kk / 2);
      uint2 x0 = *ca, x1 = *cb;
      acc ^= a0.x ^ a0.y ^ a0.z ^ a0.w ^ a1.x ^ a1.y ^ a1.z ^ a1.w ^ b0.x ^ b0.y ^ b0.z ^ b0.w ^ b1.x ^ b1.y ^ b1.z ^ b1.w ^ x0.x ^ x0.y ^ x1.x ^ x1.y;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
    if (acc == 0x1234567u) out[0] = acc;
  }
}


__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// per CTA: contiguous row range; stage = ROWS full rows of W (bulk, CHUNK-byte copies) + their codes
template <int STAGES, int ROWS, int CHUNK>
__global__ void __launch_bounds__(17 * 32, 1)
seq_pattern(const uint16_t* __restrict__ W, const uint8_t* __restrict__ C, int d, int h, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int WB = ROWS * d * 2, CB = ROWS * d / 2, SB = WB + CB;
  uint64_t* full = (uint64_t*)(smem + STAGES * SB);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int base = h / gridDim.x, rem = h % gridDim.x;
  const int r0 = blockIdx.x * base + min((int)blockIdx.x, rem);
  const int nrows = base + ((int)blockIdx.x < rem);
  const int n = (nrows + ROWS - 1) / ROWS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 16); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 16) {
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (int i = 0; i < n; ++i) {
        const int rows = min(ROWS, nrows - i * ROWS);
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], rows * (d * 2 + d / 2));
        uint8_t* st = smem + s * SB;
        const uint8_t* wsrc = (const uint8_t*)(W + (size_t)(r0 + i * ROWS) * d);
        for (int o = 0; o < rows * d * 2; o += CHUNK) bulk_g2s(st + o, wsrc + o, min(CHUNK, rows * d * 2 - o), &full[s]);
        const uint8_t* csrc = C + (size_t)(r0 + i * ROWS) * d / 2;
        for (int o = 0; o < rows * d / 2; o += CHUNK) bulk_g2s(st + WB + o, csrc + o, min(CHUNK, rows * d / 2 - o), &full[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else {
    uint32_t acc = 0;
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < n; ++i) {
      mbar_wait(&full[s], ph);
      const uint4* q = (const uint4*)(smem + s * SB);
      for (int j = threadIdx.x; j < SB / 16; j += 512) { uint4 v = q[j]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
    if (acc == 0x1234567u) out[0] = acc;
  }
}

__global__ void fill(uint4* p, size_t n, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = make_uint4(v, v * 3, v * 5, i);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int d = 4096, h = 14336, L = 4;
  size_t wbytes = (size_t)h * d * 2, cbytes = (size_t)h * d / 2;
  uint16_t* W[L]; uint8_t* C[L];
  for (int l = 0; l < L; ++l) {
    CK(cudaMalloc(&W[l], wbytes)); CK(cudaMalloc(&C[l], cbytes));
    fill<<<1184, 256>>>((uint4*)W[l], wbytes / 16, l); fill<<<1184, 256>>>((uint4*)C[l], cbytes / 16, l + 7);
  }
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)fn;
  CUtensorMap mw[L], mc[L];
  for (int l = 0; l < L; ++l) {
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)h}, strides[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {256, 16}, es[2] = {1, 1};
    CUresult r1 = enc(&mw[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W[l], dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t cd[2] = {(cuuint64_t)d / 8, (cuuint64_t)h}, cs[1] = {(cuuint64_t)d / 2};
    cuuint32_t cbox[2] = {128, 16};
    CUresult r2 = enc(&mc[l], CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, C[l], cd, cs, cbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r1 || r2) { printf("encode failed %d %d\n", r1, r2); return 1; }
  }
  uint32_t* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double bytes = wbytes + cbytes;
  auto run = [&](auto kern, int stages, const char* name) {
    const int SB = 16 * 1024 * 2 + 16 * 1024 / 2;
    int sm = stages * SB + 256;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    for (int rep = 0; rep < 2; ++rep) {
      const int K = 200;
      for (int k = 0; k < 8; ++k) kern<<<148, 544, sm>>>(mw[k % L], mc[k % L], d, h, out);
      cudaEventRecord(e0);
      for (int k = 0; k < K; ++k) kern<<<148, 544, sm>>>(mw[k % L], mc[k % L], d, h, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%-40s %7.2f us/call  %6.0f GB/s\n", name, ms * 1e3 / K, bytes * K / (ms * 1e-3) / 1e9);
    }
    CK(cudaGetLastError());
    return 0;
  };
  auto runseq = [&](auto kern, int stages, int rows, const char* name) {
    int sm = stages * rows * (d * 2 + d / 2) + 256;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    for (int rep = 0; rep < 2; ++rep) {
      const int K = 200;
      for (int k = 0; k < 8; ++k) kern<<<148, 544, sm>>>(W[k % L], C[k % L], d, h, out);
      cudaEventRecord(e0);
      for (int k = 0; k < K; ++k) kern<<<148, 544, sm>>>(W[k % L], C[k % L], d, h, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%-40s %7.2f us/call  %6.0f GB/s\n", name, ms * 1e3 / K, bytes * K / (ms * 1e-3) / 1e9);
    }
    CK(cudaGetLastError());
    return 0;
  };
  runseq(seq_pattern<4, 4, 8192>, 4, 4, "seq 4st x 4 rows, 8K copies");
  runseq(seq_pattern<4, 4, 32768>, 4, 4, "seq 4st x 4 rows, 32K copies");
  runseq(seq_pattern<5, 4, 16384>, 5, 4, "seq 5st x 4 rows, 16K copies");
  runseq(seq_pattern<3, 4, 16384>, 3, 4, "seq 3st x 4 rows, 16K copies");
  runseq(seq_pattern<8, 2, 16384>, 8, 2, "seq 8st x 2 rows, 16K copies");
  run(tma_pattern<4, 1024, 0>, 4, "tma 4st contiguous ranges");
  run(tma_pattern<4, 1024, 1>, 4, "tma 4st tile-interleaved CTAs");
  run(tma_pattern<4, 1024, 2>, 4, "tma 4st k-outer");
  CK(cudaDeviceSynchronize());
  return 0;
}
