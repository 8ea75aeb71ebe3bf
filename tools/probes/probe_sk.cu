// Probe: can the stream-K decode pattern stream W + codes at HBM speed?  One CTA per SM walks a
// contiguous range of (128-row tile, KS-column unit) pairs; per unit one 3-D TMA box of W
// (64 cols x R rows x KS/64 blocks, SW128) + one 2-D box of codes (n_m = 4) land in a ring of S
// stages; one consumer warp waits and releases immediately.  Reports us/call over 4 rotating
// 147 MB layers and the mean issue->arrival latency (cycles) seen by CTA 0.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2506_23225_b200/csrc/tma.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)
using namespace mglu;

template <int R, int KS>
__global__ void __launch_bounds__(64, 1)
probe(const __grid_constant__ CUtensorMap mW, const __grid_constant__ CUtensorMap mC, int d, int h, int S,
      int order, long long* lat) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int WB = R * KS * 2, CB = R * KS / 2;
  constexpr int SB = (WB + CB + 1023) / 1024 * 1024;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * SB);
  uint64_t* empty = full + S;
  long long* tiss = reinterpret_cast<long long*>(empty + S);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int upt = d / KS, tiles = h / R;
  const int units = upt * tiles;
  const int base = units / gridDim.x, rem = units % gridDim.x;
  const int c = blockIdx.x;
  const int u0 = c * base + min(c, rem), u1 = u0 + base + (c < rem);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == 0 && lane == 0) {
    const uint64_t pol = policy_evict_first();
    int s = 0; uint32_t ph = 0;
    for (int u = u0; u < u1; ++u) {
      int tile, ks;
      if (order == 0) { tile = u / upt; ks = u % upt; }          // tile-major (stream-K ranges)
      else { ks = u / tiles; tile = u % tiles; }                 // k-major (all SMs on one k band)
      mbar_wait(&empty[s], ph ^ 1);
      tiss[s] = clock64();
      mbar_arrive_expect_tx(&full[s], (uint32_t)(WB + CB));
      tma_load_3d_hint(smem + (size_t)s * SB, &mW, 0, tile * R, ks * (KS / 64), &full[s], pol);
      tma_load_2d_hint(smem + (size_t)s * SB + WB, &mC, ks * KS / 8, tile * R, &full[s], pol);
      if (++s == S) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    int s = 0; uint32_t ph = 0;
    long long acc = 0; int n = 0;
    for (int u = u0; u < u1; ++u) {
      mbar_wait(&full[s], ph);
      const long long t = clock64();
      acc += t - tiss[s];
      ++n;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == S) { s = 0; ph ^= 1; }
    }
    if (lane == 0 && c == 0) lat[0] = acc / (n ? n : 1);
  }
}

__global__ void fill(uint4* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4((uint32_t)i * 2654435761u + seed, seed, (uint32_t)i, 7u);
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
  long long* lat; CK(cudaMalloc(&lat, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double bytes = wbytes + cbytes;
  auto run = [&](auto kern, int R, int KS, int S, int order) -> int {
    CUtensorMap mw[L], mc[L];
    for (int l = 0; l < L; ++l) {
      cuuint64_t dims[3] = {64, (cuuint64_t)h, (cuuint64_t)d / 64}, strides[2] = {(cuuint64_t)d * 2, 128};
      cuuint32_t box[3] = {64, (cuuint32_t)R, (cuuint32_t)KS / 64}, es[3] = {1, 1, 1};
      CUresult r1 = enc(&mw[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, W[l], dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      cuuint64_t cd[2] = {(cuuint64_t)d / 8, (cuuint64_t)h}, cs[1] = {(cuuint64_t)d / 2};
      cuuint32_t cbox[2] = {(cuuint32_t)KS / 8, (cuuint32_t)R}, ces[2] = {1, 1};
      CUresult r2 = enc(&mc[l], CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, C[l], cd, cs, cbox, ces, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r1 || r2) { printf("encode failed %d %d\n", r1, r2); return 1; }
    }
    const int SB = (R * KS * 2 + R * KS / 2 + 1023) / 1024 * 1024;
    const int sm = S * SB + 1024 + 16 * S + 8 * S;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    const int K = 200;
    for (int k = 0; k < 8; ++k) kern<<<148, 64, sm>>>(mw[k % L], mc[k % L], d, h, S, order, lat);
    cudaEventRecord(e0);
    for (int k = 0; k < K; ++k) kern<<<148, 64, sm>>>(mw[k % L], mc[k % L], d, h, S, order, lat);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    CK(cudaGetLastError());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long l0; CK(cudaMemcpy(&l0, lat, 8, cudaMemcpyDeviceToHost));
    printf("R %3d KS %3d S %2d order %d (stage %3d KB, inflight %3d KB): %7.2f us/call %6.0f GB/s  lat %lld cyc\n", R, KS, S,
           order, SB / 1024, S * SB / 1024, ms * 1e3 / K, bytes * K / (ms * 1e-3) / 1e9, l0);
    return 0;
  };
  run(probe<64, 256>, 64, 256, 4, 0);
  run(probe<32, 512>, 32, 512, 4, 0);
  run(probe<16, 1024>, 16, 1024, 4, 0);
  run(probe<8, 2048>, 8, 2048, 4, 0);
  run(probe<8, 1024>, 8, 1024, 8, 0);
  run(probe<8, 512>, 8, 512, 8, 0);
  run(probe<64, 256>, 64, 256, 5, 0);
  run(probe<8, 2048>, 8, 2048, 5, 0);
  return 0;
}
