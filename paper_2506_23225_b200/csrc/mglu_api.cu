// mglu_api.cu -- the C ABI of libmglu (declared and documented in include/mglu.h).
//
// Host side only: argument validation, regime dispatch, launch configuration (PDL launches so
// back-to-back calls overlap their prologues), the host packers and the e2e host-buffer entry.
// Every arithmetic step of the forward pass runs in the kernels (gemv_simt.cuh, gemv_mma.cuh,
// gemm_tc.cuh); there is no CPU fallback.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/mglu.h"
#include "common.cuh"
#include "gemv_mma.cuh"
#include "gemv_simt.cuh"
#include "gemm_tc.cuh"
#include "pack.cuh"

struct mglu_ctx {
  int64_t d = 0, h = 0;
  int n_m = 0, act = 0, dtype = 0, device = 0;
  int path = MGLU_PATH_AUTO;
  int last_path = 0, last_launches = 0;
  int num_sms = 148;
  int max_smem_optin = 0;
  std::mutex mu;
  std::string err;
  // e2e staging (mglu_forward_host)
  void* x_stage = nullptr;
  size_t x_stage_bytes = 0;
  void* y_stage = nullptr;
  size_t y_stage_bytes = 0;
  mglu::TcState tc;
};

namespace {

const char* kStatusStr[] = {"MGLU_OK", "MGLU_ERR_INVALID_ARG", "MGLU_ERR_UNSUPPORTED",
                            "MGLU_ERR_MISALIGNED", "MGLU_ERR_CUDA", "MGLU_ERR_OOM"};

bool valid_nm(int n_m) { return n_m == 1 || n_m == 2 || n_m == 4 || n_m == 8; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
size_t elem_bytes(int dtype) { return dtype == MGLU_BF16 ? 2 : 4; }

mglu_status cuda_fail(mglu_ctx* hd, cudaError_t e, const char* what) {
  if (hd) {
    std::lock_guard<std::mutex> g(hd->mu);
    hd->err = std::string(what) + ": " + cudaGetErrorString(e);
  }
  return MGLU_ERR_CUDA;
}

mglu_status set_err(mglu_ctx* hd, mglu_status s, const std::string& msg) {
  if (hd) {
    std::lock_guard<std::mutex> g(hd->mu);
    hd->err = msg;
  }
  return s;
}

// launch with programmatic stream serialisation (PDL): the kernels call griddepcontrol.wait
// before touching x / out, so the next call's W/code streaming overlaps this call's tail.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ------------------------------------------------------------------ SIMT dispatch
template <typename T, int NM, int ACT, bool PARTIALS>
cudaError_t run_simt(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* codes,
                     void* out, float* z, cudaStream_t st) {
  const int warps_per_block = 8;
  int64_t blocks = (hd->h + warps_per_block - 1) / warps_per_block;
  const int64_t cap = (int64_t)hd->num_sms * 8;
  if (blocks > cap) blocks = cap;
  return launch_pdl(mglu::gemv_simt_kernel<T, NM, ACT, PARTIALS>, dim3((unsigned)blocks),
                    dim3(warps_per_block * 32), 0, st, (const T*)x, B, (int)hd->d, (const T*)Wt,
                    (const uint8_t*)codes, (int)hd->h, (T*)out, z);
}

template <typename T, bool PARTIALS, int NM>
cudaError_t simt_act(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* codes,
                     void* out, float* z, cudaStream_t st) {
  switch (hd->act) {
    case MGLU_ACT_IDENTITY: return run_simt<T, NM, mglu::kIdentity, PARTIALS>(hd, x, B, Wt, codes, out, z, st);
    case MGLU_ACT_SWISH: return run_simt<T, NM, mglu::kSwish, PARTIALS>(hd, x, B, Wt, codes, out, z, st);
    case MGLU_ACT_GELU: return run_simt<T, NM, mglu::kGelu, PARTIALS>(hd, x, B, Wt, codes, out, z, st);
    case MGLU_ACT_RELU: return run_simt<T, NM, mglu::kRelu, PARTIALS>(hd, x, B, Wt, codes, out, z, st);
    default: return run_simt<T, NM, mglu::kSigmoid, PARTIALS>(hd, x, B, Wt, codes, out, z, st);
  }
}

template <typename T, bool PARTIALS>
cudaError_t simt_nm(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* codes,
                    void* out, float* z, cudaStream_t st) {
  switch (hd->n_m) {
    case 1: return simt_act<T, PARTIALS, 1>(hd, x, B, Wt, codes, out, z, st);
    case 2: return simt_act<T, PARTIALS, 2>(hd, x, B, Wt, codes, out, z, st);
    case 4: return simt_act<T, PARTIALS, 4>(hd, x, B, Wt, codes, out, z, st);
    default: return simt_act<T, PARTIALS, 8>(hd, x, B, Wt, codes, out, z, st);
  }
}

// ------------------------------------------------------------------ MMA dispatch
bool mma_can_serve(const mglu_ctx* hd, int64_t B) {
  return hd->dtype == MGLU_BF16 && hd->d % 64 == 0 && B >= 1 && B <= 8 && hd->d <= 16384;
}

size_t mma_smem_bytes(const mglu_ctx* hd, int Bp) {
  return (size_t)Bp * (hd->d + 8) * 2 + (size_t)mglu::kMmaWarps * (hd->n_m + 1) * 16 * Bp * 4;
}

template <int NM, int ACT>
cudaError_t run_mma(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* codes,
                    void* out, cudaStream_t st) {
  mglu::MmaParams p;
  p.x = (const __nv_bfloat16*)x;
  p.Wt = (const __nv_bfloat16*)Wt;
  p.codes = (const uint8_t*)codes;
  p.out = (__nv_bfloat16*)out;
  p.B = B;
  p.d = (int)hd->d;
  p.h = (int)hd->h;
  p.Bp = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : 8;
  int64_t ncta = (hd->h + 15) / 16;
  if (ncta > hd->num_sms) ncta = hd->num_sms;
  p.rows_base = (int)(hd->h / ncta);
  p.rows_rem = (int)(hd->h % ncta);
  const int nch = (int)(hd->d / 64);
  int wkl = 0;
  while (wkl < 4 && (nch % (1 << (wkl + 1))) == 0) ++wkl;   // WK = largest pow2 <= 16 | nch
  p.wk_log2 = wkl;
  const size_t smem = mma_smem_bytes(hd, p.Bp);
  auto kern = mglu::gemv_mma_kernel<NM, ACT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(kern, dim3((unsigned)ncta), dim3(mglu::kMmaWarps * 32), smem, st, p);
}

template <int NM>
cudaError_t mma_act(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* codes, void* out,
                    cudaStream_t st) {
  switch (hd->act) {
    case MGLU_ACT_IDENTITY: return run_mma<NM, mglu::kIdentity>(hd, x, B, Wt, codes, out, st);
    case MGLU_ACT_SWISH: return run_mma<NM, mglu::kSwish>(hd, x, B, Wt, codes, out, st);
    case MGLU_ACT_GELU: return run_mma<NM, mglu::kGelu>(hd, x, B, Wt, codes, out, st);
    case MGLU_ACT_RELU: return run_mma<NM, mglu::kRelu>(hd, x, B, Wt, codes, out, st);
    default: return run_mma<NM, mglu::kSigmoid>(hd, x, B, Wt, codes, out, st);
  }
}

cudaError_t mma_nm(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* codes, void* out,
                   cudaStream_t st) {
  switch (hd->n_m) {
    case 1: return mma_act<1>(hd, x, B, Wt, codes, out, st);
    case 2: return mma_act<2>(hd, x, B, Wt, codes, out, st);
    case 4: return mma_act<4>(hd, x, B, Wt, codes, out, st);
    default: return mma_act<8>(hd, x, B, Wt, codes, out, st);
  }
}

mglu_status check_ptrs(mglu_ctx* hd, const void* x, int64_t B, const void* Wt, const void* codes,
                       const void* out) {
  if (!hd) return MGLU_ERR_INVALID_ARG;
  if (B < 0) return set_err(hd, MGLU_ERR_INVALID_ARG, "B < 0");
  if (!x || !Wt || !codes || !out) return set_err(hd, MGLU_ERR_INVALID_ARG, "null data pointer");
  if (!aligned16(x) || !aligned16(Wt) || !aligned16(codes) || !aligned16(out))
    return set_err(hd, MGLU_ERR_MISALIGNED, "data pointers must be 16-byte aligned");
  if (B > (int64_t)1 << 30) return set_err(hd, MGLU_ERR_INVALID_ARG, "B too large");
  return MGLU_OK;
}

}  // namespace

extern "C" {

const char* mglu_version(void) { return "0.1.0"; }

const char* mglu_status_string(mglu_status s) {
  if ((int)s < 0 || (int)s > 5) return "MGLU_ERR_UNKNOWN";
  return kStatusStr[(int)s];
}

const char* mglu_last_error(mglu_handle hd) {
  if (!hd) return "null handle";
  std::lock_guard<std::mutex> g(hd->mu);
  return hd->err.c_str();
}

size_t mglu_packed_mask_bytes(int64_t d, int64_t h, int n_m) {
  if (d < 0 || h < 0 || !valid_nm(n_m)) return 0;
  return (size_t)((h * d * n_m + 7) / 8);
}

mglu_status mglu_create(mglu_handle* out, int64_t d, int64_t h, int n_m, int act, int dtype,
                        int device) {
  if (!out) return MGLU_ERR_INVALID_ARG;
  *out = nullptr;
  if (d < 1 || h < 1 || act < 0 || act > 4 || (dtype != MGLU_BF16 && dtype != MGLU_F32) || device < 0)
    return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m) || d % 8 != 0 || h > ((int64_t)1 << 31) - 1 || d > ((int64_t)1 << 24))
    return MGLU_ERR_UNSUPPORTED;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev) return MGLU_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return MGLU_ERR_CUDA;
  if (prop.major != 10) return MGLU_ERR_UNSUPPORTED;   // sm_100a kernels only
  mglu_ctx* hd = new (std::nothrow) mglu_ctx();
  if (!hd) return MGLU_ERR_OOM;
  hd->d = d; hd->h = h; hd->n_m = n_m; hd->act = act; hd->dtype = dtype; hd->device = device;
  hd->num_sms = prop.multiProcessorCount;
  hd->max_smem_optin = (int)prop.sharedMemPerBlockOptin;
  *out = hd;
  return MGLU_OK;
}

mglu_status mglu_destroy(mglu_handle hd) {
  if (!hd) return MGLU_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(hd->device);
  if (hd->x_stage) cudaFree(hd->x_stage);
  if (hd->y_stage) cudaFree(hd->y_stage);
  mglu::tc_release(hd->tc);
  cudaSetDevice(prev);
  delete hd;
  return MGLU_OK;
}

mglu_status mglu_set_path(mglu_handle hd, int path) {
  if (!hd || path < MGLU_PATH_AUTO || path > MGLU_PATH_TCGEN05) return MGLU_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> g(hd->mu);
  hd->path = path;
  return MGLU_OK;
}

int mglu_last_launch_count(mglu_handle hd) { return hd ? hd->last_launches : -1; }
int mglu_last_path(mglu_handle hd) { return hd ? hd->last_path : -1; }

mglu_status mglu_forward(mglu_handle hd, const void* x, int64_t B, const void* Wt,
                         const void* packed, void* out, void* stream) {
  mglu_status s = check_ptrs(hd, x, B, Wt, packed, out);
  if (s != MGLU_OK) return s;
  hd->last_launches = 0;
  if (B == 0) return MGLU_OK;
  int path;
  {
    std::lock_guard<std::mutex> g(hd->mu);
    path = hd->path;
  }
  if (path == MGLU_PATH_AUTO) {
    if (hd->dtype == MGLU_BF16 && mglu::tc_can_serve(hd->d, hd->h, hd->n_m, B) && B > 64)
      path = MGLU_PATH_TCGEN05;
    else if (mma_can_serve(hd, B))
      path = MGLU_PATH_MMA;
    else
      path = MGLU_PATH_SIMT;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != hd->device) cudaSetDevice(hd->device);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  int launches = 0;
  if (path == MGLU_PATH_MMA) {
    if (!mma_can_serve(hd, B)) {
      if (prev != hd->device) cudaSetDevice(prev);
      return set_err(hd, MGLU_ERR_UNSUPPORTED, "MMA path needs bf16, d % 64 == 0, 1 <= B <= 8");
    }
    e = mma_nm(hd, x, (int)B, Wt, packed, out, st);
    launches = 1;
  } else if (path == MGLU_PATH_TCGEN05) {
    if (hd->dtype != MGLU_BF16 || !mglu::tc_can_serve(hd->d, hd->h, hd->n_m, B)) {
      if (prev != hd->device) cudaSetDevice(prev);
      return set_err(hd, MGLU_ERR_UNSUPPORTED, "tcgen05 path needs bf16, d % 64 == 0, h % 128 == 0");
    }
    e = mglu::tc_forward(hd->tc, hd->d, hd->h, hd->n_m, hd->act, x, B, Wt, packed, out, st, &launches);
  } else {
    e = hd->dtype == MGLU_BF16
            ? simt_nm<__nv_bfloat16, false>(hd, x, (int)B, Wt, packed, out, nullptr, st)
            : simt_nm<float, false>(hd, x, (int)B, Wt, packed, out, nullptr, st);
    launches = 1;
  }
  if (prev != hd->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(hd, e, "mglu_forward launch");
  hd->last_path = path;
  hd->last_launches = launches;
  return MGLU_OK;
}

mglu_status mglu_forward_partials(mglu_handle hd, const void* x, int64_t B, const void* Wt,
                                  const void* packed, float* z, void* stream) {
  mglu_status s = check_ptrs(hd, x, B, Wt, packed, z);
  if (s != MGLU_OK) return s;
  hd->last_launches = 0;
  if (B == 0) return MGLU_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != hd->device) cudaSetDevice(hd->device);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = hd->dtype == MGLU_BF16
                      ? simt_nm<__nv_bfloat16, true>(hd, x, (int)B, Wt, packed, nullptr, z, st)
                      : simt_nm<float, true>(hd, x, (int)B, Wt, packed, nullptr, z, st);
  if (prev != hd->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(hd, e, "mglu_forward_partials launch");
  hd->last_path = MGLU_PATH_SIMT;
  hd->last_launches = 1;
  return MGLU_OK;
}

mglu_status mglu_forward_host(mglu_handle hd, const void* x_host, int64_t B, const void* Wt,
                              const void* packed, void* out_host, void* stream) {
  if (!hd) return MGLU_ERR_INVALID_ARG;
  if (B < 0 || !x_host || !out_host || !Wt || !packed)
    return set_err(hd, MGLU_ERR_INVALID_ARG, "null pointer or B < 0");
  if (B == 0) return MGLU_OK;
  const size_t xb = (size_t)B * hd->d * elem_bytes(hd->dtype);
  const size_t yb = (size_t)B * hd->h * elem_bytes(hd->dtype);
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != hd->device) cudaSetDevice(hd->device);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  if (xb > hd->x_stage_bytes) {
    if (hd->x_stage) { cudaStreamSynchronize(st); cudaFree(hd->x_stage); hd->x_stage = nullptr; }
    e = cudaMalloc(&hd->x_stage, xb);
    if (e != cudaSuccess) { hd->x_stage_bytes = 0; if (prev != hd->device) cudaSetDevice(prev); return MGLU_ERR_OOM; }
    hd->x_stage_bytes = xb;
  }
  if (yb > hd->y_stage_bytes) {
    if (hd->y_stage) { cudaStreamSynchronize(st); cudaFree(hd->y_stage); hd->y_stage = nullptr; }
    e = cudaMalloc(&hd->y_stage, yb);
    if (e != cudaSuccess) { hd->y_stage_bytes = 0; if (prev != hd->device) cudaSetDevice(prev); return MGLU_ERR_OOM; }
    hd->y_stage_bytes = yb;
  }
  e = cudaMemcpyAsync(hd->x_stage, x_host, xb, cudaMemcpyHostToDevice, st);
  if (prev != hd->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(hd, e, "H2D x");
  mglu_status s = mglu_forward(hd, hd->x_stage, B, Wt, packed, hd->y_stage, stream);
  if (s != MGLU_OK) return s;
  cudaSetDevice(hd->device);
  e = cudaMemcpyAsync(out_host, hd->y_stage, yb, cudaMemcpyDeviceToHost, st);
  if (prev != hd->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(hd, e, "D2H y");
  return MGLU_OK;
}

// ------------------------------------------------------------------ packing
mglu_status mglu_pack_masks_host(const uint8_t* bits, int n_m, int64_t h, int64_t d, uint8_t* packed) {
  if (!bits || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m)) return MGLU_ERR_UNSUPPORTED;
  const int64_t hd = h * d;
  const int per = 8 / n_m;
  const int64_t nbytes = (hd * n_m + 7) / 8;
  for (int64_t byte = 0; byte < nbytes; ++byte) {
    uint32_t v = 0;
    for (int q = 0; q < per; ++q) {
      const int64_t e = byte * per + q;
      if (e >= hd) break;
      for (int i = 0; i < n_m; ++i) {
        const uint8_t b = bits[(int64_t)i * hd + e];
        if (b > 1) return MGLU_ERR_INVALID_ARG;
        v |= (uint32_t)b << (q * n_m + i);
      }
    }
    packed[byte] = (uint8_t)v;
  }
  return MGLU_OK;
}

mglu_status mglu_pack_logits_host(const float* logits, int n_m, int64_t h, int64_t d, uint8_t* packed) {
  if (!logits || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m)) return MGLU_ERR_UNSUPPORTED;
  const int64_t hd = h * d;
  const int per = 8 / n_m;
  const int64_t nbytes = (hd * n_m + 7) / 8;
  for (int64_t byte = 0; byte < nbytes; ++byte) {
    uint32_t v = 0;
    for (int q = 0; q < per; ++q) {
      const int64_t e = byte * per + q;
      if (e >= hd) break;
      for (int i = 0; i < n_m; ++i)
        v |= (logits[(int64_t)i * hd + e] > 0.0f ? 1u : 0u) << (q * n_m + i);   // strict (R4)
    }
    packed[byte] = (uint8_t)v;
  }
  return MGLU_OK;
}

mglu_status mglu_unpack_masks_host(const uint8_t* packed, int n_m, int64_t h, int64_t d, uint8_t* bits) {
  if (!bits || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m)) return MGLU_ERR_UNSUPPORTED;
  const int64_t hd = h * d;
  const int per = 8 / n_m;
  for (int64_t e = 0; e < hd; ++e) {
    const uint32_t code = (packed[e / per] >> ((e % per) * n_m)) & ((1u << n_m) - 1u);
    for (int i = 0; i < n_m; ++i) bits[(int64_t)i * hd + e] = (uint8_t)((code >> i) & 1u);
  }
  return MGLU_OK;
}

static mglu_status device_launch_check(cudaError_t e) {
  return e == cudaSuccess ? MGLU_OK : MGLU_ERR_CUDA;
}

mglu_status mglu_pack_masks_device(const uint8_t* bits, int n_m, int64_t h, int64_t d, uint8_t* packed,
                                   void* stream) {
  if (!bits || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m)) return MGLU_ERR_UNSUPPORTED;
  const int64_t hd = h * d, nbytes = (hd * n_m + 7) / 8;
  if (nbytes == 0) return MGLU_OK;
  int64_t blocks = (nbytes + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  // 0/1 validation flag: written only on a bad value; the host cannot see it without a sync,
  // so the device packer clamps (bit & 1) and documents the host packer as the validating one.
  mglu::pack_kernel<uint8_t><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(bits, n_m, hd, packed, nbytes, nullptr);
  return device_launch_check(cudaGetLastError());
}

mglu_status mglu_pack_logits_device(const float* logits, int n_m, int64_t h, int64_t d, uint8_t* packed,
                                    void* stream) {
  if (!logits || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m)) return MGLU_ERR_UNSUPPORTED;
  const int64_t hd = h * d, nbytes = (hd * n_m + 7) / 8;
  if (nbytes == 0) return MGLU_OK;
  int64_t blocks = (nbytes + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  mglu::pack_kernel<float><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(logits, n_m, hd, packed, nbytes, nullptr);
  return device_launch_check(cudaGetLastError());
}

mglu_status mglu_unpack_masks_device(const uint8_t* packed, int n_m, int64_t h, int64_t d, uint8_t* bits,
                                     void* stream) {
  if (!bits || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m)) return MGLU_ERR_UNSUPPORTED;
  const int64_t hd = h * d;
  if (hd == 0) return MGLU_OK;
  int64_t blocks = (hd + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  mglu::unpack_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(packed, n_m, hd, bits);
  return device_launch_check(cudaGetLastError());
}

}  // extern "C"
