// Probe: per-call time of a 146.8 MB read-once stream when K calls run back to back over
// rotating distinct buffers (each call cold: 6 x 146.8 MB >> 126 MB L2), plain launches vs a
// CUDA graph vs programmatic dependent launch (PDL).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int U, bool PDL>
__global__ void stream_read(const uint4* __restrict__ p, size_t n, uint32_t* out) {
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  uint32_t acc = 0;
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = tid;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldnc(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n; i += stride) { uint4 v = ldnc(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (PDL) asm volatile("griddepcontrol.launch_dependents;");
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void wscrub(uint4* p, size_t n, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = make_uint4(v, v, v, v);
}

int main() {
  int nsm = 148;
  uint32_t* dout; CK(cudaMalloc(&dout, 64));
  cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int NB = 6;
  size_t bytes = 146800640, n = bytes / 16;
  uint4* bufs[NB];
  for (int b = 0; b < NB; ++b) { CK(cudaMalloc(&bufs[b], bytes)); wscrub<<<nsm * 8, 256, 0, st>>>(bufs[b], n, b); }
  uint4* sb; CK(cudaMalloc(&sb, 512ull << 20));
  const int K = 60;
  for (int rotate : {NB, 1}) {
    // plain launches
    for (int rep = 0; rep < 3; ++rep) {
      wscrub<<<nsm * 8, 256, 0, st>>>(sb, (512ull << 20) / 16, rep);
      cudaEventRecord(e0, st);
      for (int k = 0; k < K; ++k) stream_read<4, false><<<nsm * 4, 256, 0, st>>>(bufs[k % rotate], n, dout);
      cudaEventRecord(e1, st); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("rotate %d plain   : %.2f us/call  %.0f GB/s\n", rotate, ms * 1e3 / K, bytes * K / (ms * 1e-3) / 1e9);
    }
    // PDL launches
    for (int rep = 0; rep < 3; ++rep) {
      wscrub<<<nsm * 8, 256, 0, st>>>(sb, (512ull << 20) / 16, rep);
      cudaEventRecord(e0, st);
      for (int k = 0; k < K; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nsm * 4); cfg.blockDim = dim3(256); cfg.stream = st;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, stream_read<4, true>, (const uint4*)bufs[k % rotate], n, dout));
      }
      cudaEventRecord(e1, st); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("rotate %d PDL     : %.2f us/call  %.0f GB/s\n", rotate, ms * 1e3 / K, bytes * K / (ms * 1e-3) / 1e9);
    }
    // graph
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
    for (int k = 0; k < K; ++k) stream_read<4, false><<<nsm * 4, 256, 0, st>>>(bufs[k % rotate], n, dout);
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int rep = 0; rep < 3; ++rep) {
      wscrub<<<nsm * 8, 256, 0, st>>>(sb, (512ull << 20) / 16, rep);
      cudaEventRecord(e0, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("rotate %d graph   : %.2f us/call  %.0f GB/s\n", rotate, ms * 1e3 / K, bytes * K / (ms * 1e-3) / 1e9);
    }
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}
