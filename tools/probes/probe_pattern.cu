// Probe: can the decode kernel's access pattern (16-row tiles, per-thread 32 B of rows r and
// r+8 + codes, K split across 16 warps) stream at HBM speed when the math is removed?
// Variants: load width, prefetch depth, warps/CTA, K-split order.  Back-to-back PDL-less
// launches over 4 rotating 147 MB layers; per-call time.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void ld_v8(const void* p, uint32_t (&w)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]) : "l"(p));
}
__device__ __forceinline__ uint2 ld_v2(const void* p) {
  uint2 r; asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p)); return r;
}

struct St { uint32_t wa[8], wb[8]; uint2 ca, cb; };

// DEPTH-stage register ring; WARPS warps; interleaved or blocked K split
template <int WARPS, int DEPTH, bool INTERLEAVE>
__global__ void __launch_bounds__(WARPS * 32, 1)
pattern(const uint16_t* __restrict__ Wt, const uint8_t* __restrict__ codes, int d, int h, uint32_t* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
  const int base = h / gridDim.x, rem = h % gridDim.x;
  const int r0 = blockIdx.x * base + min((int)blockIdx.x, rem);
  const int nrows = base + ((int)blockIdx.x < rem);
  const int ntiles = (nrows + 15) / 16;
  const int nch = d / 64, nkw = nch / WARPS;
  const int n = ntiles * nkw;
  uint32_t acc = 0;
  St st[DEPTH];
  auto load = [&](St& s, int i) {
    const int tile = i / nkw, kcl = i % nkw;
    const int kc = INTERLEAVE ? warp + WARPS * kcl : warp * nkw + kcl;
    const int ra = tile * 16 + r, rb = ra + 8;
    const int k = kc * 64 + c * 16;
    if (ra < nrows) { size_t e = (size_t)(r0 + ra) * d + k; ld_v8(Wt + e, s.wa); s.ca = ld_v2(codes + e / 2); }
    else { for (int q = 0; q < 8; ++q) s.wa[q] = 0; s.ca = make_uint2(0, 0); }
    if (rb < nrows) { size_t e = (size_t)(r0 + rb) * d + k; ld_v8(Wt + e, s.wb); s.cb = ld_v2(codes + e / 2); }
    else { for (int q = 0; q < 8; ++q) s.wb[q] = 0; s.cb = make_uint2(0, 0); }
  };
  auto use = [&](const St& s) {
#pragma unroll
    for (int q = 0; q < 8; ++q) acc ^= s.wa[q] ^ s.wb[q];
    acc ^= s.ca.x ^ s.ca.y ^ s.cb.x ^ s.cb.y;
  };
#pragma unroll
  for (int p = 0; p < DEPTH - 1; ++p) if (p < n) load(st[p], p);
  for (int i0 = 0; i0 < n; i0 += DEPTH) {
#pragma unroll
    for (int u = 0; u < DEPTH; ++u) {
      const int i = i0 + u;
      if (i < n) {
        if (i + DEPTH - 1 < n) load(st[(u + DEPTH - 1) % DEPTH], i + DEPTH - 1);
        use(st[u]);
      }
    }
  }
  if (acc == 0x1234567u) out[0] = acc;
}

__global__ void fill(uint4* p, size_t n, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = make_uint4(v, v * 3, v * 5, i);
}

int main() {
  const int d = 4096, h = 14336, L = 4;
  size_t wbytes = (size_t)h * d * 2, cbytes = (size_t)h * d / 2;
  uint16_t* W[L]; uint8_t* C[L];
  for (int l = 0; l < L; ++l) {
    CK(cudaMalloc(&W[l], wbytes)); CK(cudaMalloc(&C[l], cbytes));
    fill<<<1184, 256>>>((uint4*)W[l], wbytes / 16, l); fill<<<1184, 256>>>((uint4*)C[l], cbytes / 16, l + 7);
  }
  uint32_t* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double bytes = wbytes + cbytes;
  auto run = [&](auto kern, int grid, int threads, const char* name) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 0));
    for (int rep = 0; rep < 2; ++rep) {
      const int K = 200;
      for (int k = 0; k < 8; ++k) kern<<<grid, threads>>>(W[k % L], C[k % L], d, h, out);
      cudaEventRecord(e0);
      for (int k = 0; k < K; ++k) kern<<<grid, threads>>>(W[k % L], C[k % L], d, h, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%-40s %7.2f us/call  %6.0f GB/s\n", name, ms * 1e3 / K, bytes * K / (ms * 1e-3) / 1e9);
    }
    return 0;
  };
  run(pattern<16, 3, false>, 148, 512, "16w depth3 blocked");
  run(pattern<16, 3, true>, 148, 512, "16w depth3 interleaved");
  run(pattern<16, 4, true>, 148, 512, "16w depth4 interleaved");
  run(pattern<16, 6, true>, 148, 512, "16w depth6 interleaved");
  run(pattern<8, 4, true>, 148, 256, "8w depth4 interleaved");
  run(pattern<8, 4, true>, 296, 256, "8w depth4 interleaved 2cta/SM");
  run(pattern<16, 3, true>, 296, 512, "16w depth3 interleaved 2cta/SM");
  run(pattern<32, 3, true>, 148, 1024, "32w depth3 interleaved");
  run(pattern<4, 4, true>, 592, 128, "4w depth4 interleaved 4cta/SM");
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  return 0;
}
