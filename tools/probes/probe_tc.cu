// Probe: tcgen05.mma issue/commit costs for the prefill kernel's shapes (M = 128, N = BN, K = 16,
// bf16 -> fp32).  One CTA per SM, 148 CTAs.  Warp 1 issues `steps` k16 steps of `nop` MMAs each
// (nop accumulators of BN columns); variants:
//   mode 0: TS (A in TMEM), one commit at the end
//   mode 1: TS, commit every `ce` steps (no waits)
//   mode 2: TS, commit every `ce` steps and wait for the commit `lag` commits back (round trip)
//   mode 3: SS (A in smem), one commit at the end
//   mode 4: TS + 4 warps continuously tcgen05.st-ing 8 columns each (store interference)
//   mode 5: TS, commit every ce steps; warps 4..7 wait each commit and arrive on a second barrier
//           the MMA warp waits on before the next group (the full masker handshake)
// Prints cycles per k16 step and the effective fraction of the 128*N/256-cycle floor.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2506_23225_b200/csrc/tcgen05.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)
using namespace mglu;

template <int MODE, int BN, int NOP, int CE, int LAG, int ST = -1>
__global__ void __launch_bounds__(256, 1)
probe(int steps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* bt = smem;                  // B tile BN x 64 bf16 (SW128), 4 k16 slices
  uint8_t* at = smem + 256 * 128;      // A tile 128 x 64 bf16 (SW128) for SS
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 256 * 128 + 128 * 128);   // [8] commit ring + [8] ack ring
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 17);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (256 * 128 + 128 * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&bars[i], i < 8 ? 1 : 128);
    mbar_init(&bars[16], 1);
    mbar_fence_init();
  }
  fence_async_smem();
  if (warp == 0) tmem_alloc(slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  constexpr uint32_t idesc = idesc_bf16_f32(128, BN);
  constexpr uint32_t acol = 448;
  constexpr bool COMMITS = MODE == 1 || MODE == 2 || MODE == 5;
  if (warp == 1) {
    const uint64_t bd0 = smem_desc_kmajor(smem_u32(bt), 128);
    const uint64_t ad0 = smem_desc_kmajor(smem_u32(at), 128);
    long long t0 = clock64();
    int ncommit = 0;
    for (int s0 = 0; s0 < steps; s0 += 4) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int s = s0 + kk;
        if (elect_one()) {
#pragma unroll
          for (int op = 0; op < NOP; ++op) {
            if (MODE == 3) tc_mma_ss(tmem + op * BN, ad0 + kk * 2, bd0 + kk * 2, idesc, s > 0);
            else tc_mma_ts(tmem + op * BN, tmem + acol + (uint32_t)(kk * 8), bd0 + kk * 2, idesc, s > 0);
          }
          if (COMMITS && (kk + 1) % CE == 0) tc_commit(&bars[(ncommit + kk / CE) & 7]);
        }
        __syncwarp();
        if (COMMITS && (kk + 1) % CE == 0) {
          const int nc = ncommit + kk / CE + 1;
          if (MODE == 2 && nc > LAG) {
            const int c = nc - 1 - LAG;
            mbar_wait(&bars[c & 7], (uint32_t)(c >> 3) & 1u);
          }
          if (MODE == 5 && nc > LAG) {
            const int c = nc - 1 - LAG;
            mbar_wait(&bars[8 + (c & 7)], (uint32_t)(c >> 3) & 1u);
            tc_fence_after();
          }
        }
      }
      if (COMMITS) ncommit += 4 / CE;
    }
    if (elect_one()) tc_commit(&bars[16]);
    __syncwarp();
    mbar_wait(&bars[16], 0);
    long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  } else if (warp >= 4 && MODE == 4) {
    uint32_t v[8] = {0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u};
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int nst = ST < 0 ? steps * NOP / 4 : steps * ST;
    for (int s = 0; s < nst; ++s) {
      tmem_st8(tmem + lane_off + 480 + (s & 3) * 8, v);
      tmem_st_wait();
    }
  } else if (warp >= 4 && MODE == 5) {
    const int ncom = steps / CE;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t v[8] = {0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u};
    for (int c = 0; c < ncom; ++c) {
      mbar_wait(&bars[c & 7], (uint32_t)(c >> 3) & 1u);
      tc_fence_after();
constexpr int NST = ST < 0 ? NOP : ST;
#pragma unroll
      for (int op = 0; op < NST; ++op) tmem_st8(tmem + lane_off + 480 + (op & 3) * 8, v);
      if (NST) tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars[8 + (c & 7)]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int MODE, int BN, int NOP, int CE, int LAG, int ST = -1>
int run(long long* d_out) {
  const size_t smem = 256 * 128 + 128 * 128 + 1024 + 256;
  auto k = probe<MODE, BN, NOP, CE, LAG, ST>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int steps = 4096;
  k<<<148, 256, smem>>>(64, d_out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 256, smem>>>(steps, d_out);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  CK(cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double floor = 128.0 * BN / 256.0 * NOP;
  const double tflops = 2.0 * 128 * BN * 16 * NOP * (double)steps * 148 / (ms * 1e-3) / 1e12;
  printf("ST %2d mode %d BN %3d nop %d ce %d lag %d: %.1f cyc/step (floor %.0f, eff %.2f)  %.3f ms  %.0f TFLOP/s\n",
         ST, MODE, BN, NOP, CE, LAG, avg / steps, floor, floor / (avg / steps), ms, tflops);
  return 0;
}

int main() {
  long long* d_out;
  CK(cudaMalloc(&d_out, 148 * sizeof(long long)));
  run<0, 16, 5, 1, 0>(d_out);
  // TS MMAs (N = 16, 5 per k16 step) with 4 warps concurrently tcgen05.st-ing ST x8 columns per step
  run<4, 16, 5, 1, 0, 1>(d_out); run<4, 16, 5, 1, 0, 2>(d_out); run<4, 16, 5, 1, 0, 5>(d_out); run<4, 16, 5, 1, 0, 10>(d_out);
  run<4, 64, 5, 1, 0, 5>(d_out);
  return 0;
}
