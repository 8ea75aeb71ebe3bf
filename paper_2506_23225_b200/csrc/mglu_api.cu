// mglu_api.cu -- the C ABI of libmglu (declared and documented in include/mglu.h).
//
// Host side only: argument validation, regime dispatch, launch configuration (PDL launches so
// back-to-back calls overlap their prologues), the host packers and the e2e host-buffer entry.
// Every arithmetic step of the forward pass runs in the kernels (gemv_simt.cuh, gemv_mma.cuh,
// gemm_tc.cuh); there is no CPU fallback.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <string>
#include <type_traits>

#include "../../include/mglu.h"
#include "common.cuh"
#include "gemv_mma.cuh"
#include "gemv_simt.cuh"
#include "gemm_tc.cuh"
#include "gemv_tc.cuh"
#include "pack.cuh"
#include "router.cuh"
#include "backward.cuh"


struct mglu_ctx {
  int64_t d = 0, h = 0;
  int n_m = 0, act = 0, dtype = 0, device = 0;
  int path = MGLU_PATH_AUTO;
  int variant = 0;           // partial-mask ablation variant (mglu_set_variant)
  int debug = 0;             // test hooks (mglu_set_debug)
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
  // TMA descriptor cache of the decode path
  struct DecMaps {
    bool valid = false;
    const void* Wt = nullptr;
    const void* codes = nullptr;
    bool planes = false;           // codes in the plane-major layout (routed, row f2)
    uint64_t stamp = 0;
    mglu::DecMaps maps;
  };
  std::array<DecMaps, 16> dec_cache;
  uint64_t dec_clock = 0;
  // W / code descriptors of the tcgen05 paths, keyed by (kind, Wt, codes, box shape): only x's
  // descriptor is encoded per call
  struct TcMaps {
    bool valid = false;
    int kind = 0, a = 0, b = 0;
    const void* Wt = nullptr;
    const void* codes = nullptr;
    uint64_t stamp = 0;
    CUtensorMap m[4];
  };
  std::array<TcMaps, 16> tc_cache;
  // stream-K decode (tcgen05) workspace: published partials + one ticket per 128-row tile (0
  // between calls: a tile's last arriver re-arms it), allocated / grown on first use
  float* sk_ws = nullptr;
  size_t sk_ws_bytes = 0;
  uint32_t* sk_tickets = nullptr;
  // training path (mglu_backward): forward streams z [B][2 n_m][h] + coefficients E [B][n_m+1][h]
  float* bw_ws = nullptr;
  size_t bw_ws_bytes = 0;
  // fused FFN block (row f1): grid-barrier counter + generation, zeroed once, self-resetting
  unsigned* ffn_bar = nullptr;

};

namespace {

// per-call arguments beyond (x, B, Wt, codes, out) that reach every launcher
struct Call {
  cudaStream_t st;
  const float* G = nullptr;   // routed gate weights [B][n_m] (mglu_forward_routed), nullptr: Eq. 3
  int K = 0;                  // K of the routed call (0: unknown -> every mask evaluated)
  float* z = nullptr;         // mglu_forward_partials: Alg. 1's z [B][2 n_m][h] instead of y
  bool row_split = false;     // tcgen05 GEMV: row split (MGLU_PATH_TCROW) instead of stream-K
  bool planes = false;        // routed call with plane-major codes (mglu_forward_routed_planes)
};

const char* kStatusStr[] = {"MGLU_OK", "MGLU_ERR_INVALID_ARG", "MGLU_ERR_UNSUPPORTED",
                            "MGLU_ERR_MISALIGNED", "MGLU_ERR_CUDA", "MGLU_ERR_OOM"};

// mask counts: the tensor-core and HMMA kernels take n_m in {1, 2, 4, 8}; the SIMT kernel also
// serves the other counts up to 8 and n_m = 16
bool fast_nm(int n_m) { return n_m == 1 || n_m == 2 || n_m == 4 || n_m == 8; }
bool valid_nm(int n_m) { return (n_m >= 1 && n_m <= 8) || n_m == 16; }
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

// the opt-in dynamic shared-memory limit is a per-kernel (per-device) attribute: raise it to the
// device maximum once per kernel instead of on every launch
cudaError_t smem_optin(const void* kern, int device, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_pair(kern, device);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[key] = bytes;
  return e;
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
                     void* out, float* z, const Call& cl) {
  const int warps_per_block = 8;
  int64_t blocks = (hd->h + warps_per_block - 1) / warps_per_block;
  const int64_t cap = (int64_t)hd->num_sms * 8;
  if (blocks > cap) blocks = cap;
  return launch_pdl(mglu::gemv_simt_kernel<T, NM, ACT, PARTIALS>, dim3((unsigned)blocks),
                    dim3(warps_per_block * 32), 0, cl.st, (const T*)x, B, (int)hd->d, (const T*)Wt,
                    (const uint8_t*)codes, (int)hd->h, (T*)out, z, cl.G, hd->variant, hd->act);
}

template <typename T, bool PARTIALS, int NM>
cudaError_t simt_act(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* codes,
                     void* out, float* z, const Call& cl) {
  switch (hd->act) {
    case MGLU_ACT_SWISH: return run_simt<T, NM, mglu::kSwish, PARTIALS>(hd, x, B, Wt, codes, out, z, cl);
    default: return run_simt<T, NM, mglu::kRuntimeAct, PARTIALS>(hd, x, B, Wt, codes, out, z, cl);   // g at runtime
  }
}

template <typename T, bool PARTIALS>
cudaError_t simt_nm(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* codes,
                    void* out, float* z, const Call& cl) {
#ifdef MGLU_DEC_ONLY
  return cudaErrorInvalidValue;
#endif
  switch (hd->n_m) {
    case 1: return simt_act<T, PARTIALS, 1>(hd, x, B, Wt, codes, out, z, cl);
    case 2: return simt_act<T, PARTIALS, 2>(hd, x, B, Wt, codes, out, z, cl);
    case 3: return simt_act<T, PARTIALS, 3>(hd, x, B, Wt, codes, out, z, cl);
    case 4: return simt_act<T, PARTIALS, 4>(hd, x, B, Wt, codes, out, z, cl);
    case 5: return simt_act<T, PARTIALS, 5>(hd, x, B, Wt, codes, out, z, cl);
    case 6: return simt_act<T, PARTIALS, 6>(hd, x, B, Wt, codes, out, z, cl);
    case 7: return simt_act<T, PARTIALS, 7>(hd, x, B, Wt, codes, out, z, cl);
    case 8: return simt_act<T, PARTIALS, 8>(hd, x, B, Wt, codes, out, z, cl);
    case 16: return simt_act<T, PARTIALS, 16>(hd, x, B, Wt, codes, out, z, cl);
    default: return cudaErrorInvalidValue;                  // (n_m = 0 dense handles never get here)
  }
}

// ------------------------------------------------------------------ MMA (TMA-fed decode) dispatch
bool mma_can_serve(const mglu_ctx* hd, int64_t B) {
  // 128-column code blocks of 16 * n_m bytes tile the rows exactly; n_m >= 4 keeps one token group
  // (B <= 4: two groups' accumulators do not fit the 96-register budget without spilling -- and the
  // stream-K tcgen05 GEMV is faster there anyway, profiles/r02_decode.txt)
  return hd->dtype == MGLU_BF16 && (hd->n_m == 0 || fast_nm(hd->n_m)) && hd->d % 128 == 0 && B >= 1 &&
         B <= (hd->n_m >= 4 ? 4 : 8) && hd->d <= 32768;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encoder() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  });
  return fn;
}

CUtensorMapSwizzle swizzle_for(int span) {
  return span == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : span == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
}

// 3-D row-major view [blocks][rows][inner] of a [rows][cols] tensor: inner = `inner` elements of
// `esize` bytes, blocks of `inner` columns (stride inner*esize), rows (stride cols*esize)
bool encode_3d_blocks(CUtensorMap* m, CUtensorMapDataType dt, size_t esize, const void* base, uint64_t cols,
                      uint64_t rows, uint32_t inner, uint32_t brows, uint32_t bblocks, CUtensorMapSwizzle swz) {
  EncodeTiledFn enc = get_encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {inner, rows, cols / inner};
  cuuint64_t strides[2] = {cols * esize, inner * esize};
  cuuint32_t box[3] = {inner, brows, bblocks};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// descriptor cache keyed by (Wt, codes).  W: 64-column blocks (SW128); codes: 128-column blocks of
// 16*n_m bytes (swizzle = span).  Round type ti (T = 8 >> ti tiles): boxes of 8T rows x
// (2 WPT | WPT) blocks, WPT = 2 << ti.
bool dec_maps(mglu_ctx* hd, const void* Wt, const void* codes, mglu::DecMaps* out, bool planes = false) {
  std::lock_guard<std::mutex> g(hd->mu);
  for (auto& e : hd->dec_cache)
    if (e.valid && e.Wt == Wt && e.codes == codes && e.planes == planes) {
      e.stamp = ++hd->dec_clock;
      *out = e.maps;
      return true;
    }
  const int NM = hd->n_m;
  const int span = 16 * NM;
  const auto sw = CU_TENSOR_MAP_SWIZZLE_128B;
  const auto csw = span == 16 ? CU_TENSOR_MAP_SWIZZLE_NONE : swizzle_for(span);
  const uint64_t crow_u32 = (uint64_t)hd->d * NM / 32;
  mglu::DecMaps m;
  for (int ti = 0; ti < 4; ++ti) {
    const uint32_t rows = 64u >> ti, wpt = 2u << ti;
    if (!encode_3d_blocks(&m.w[ti], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wt, hd->d, hd->h, 64, rows, 2 * wpt, sw))
      return false;
    if (NM == 0) m.c[ti] = m.w[ti];                          // dense projection: W boxes only
    else if (planes) {
      // plane-major codes: one [n_m h][d/32] u32 tensor, boxes of 8T rows x KS/32 words
      EncodeTiledFn enc = get_encoder();
      cuuint64_t dims[2] = {(cuuint64_t)hd->d / 32, (cuuint64_t)(NM * hd->h)};
      cuuint64_t strides[1] = {(cuuint64_t)hd->d / 32 * 4};
      cuuint32_t box[2] = {8u << ti, rows};
      cuuint32_t es[2] = {1, 1};
      if (!enc || enc(&m.c[ti], CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(codes), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    } else if (!encode_3d_blocks(&m.c[ti], CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, codes, crow_u32, hd->h, span / 4, rows, wpt, csw))
      return false;
  }
  size_t victim = 0;
  for (size_t i = 0; i < hd->dec_cache.size(); ++i) {
    if (!hd->dec_cache[i].valid) { victim = i; break; }
    if (hd->dec_cache[i].stamp < hd->dec_cache[victim].stamp) victim = i;
  }
  auto& e = hd->dec_cache[victim];
  e.valid = true; e.Wt = Wt; e.codes = codes; e.planes = planes; e.stamp = ++hd->dec_clock;
  e.maps = m;
  *out = m;
  return true;
}

// cached W / code descriptors of a tcgen05 path (see mglu_ctx::tc_cache); `build` encodes m[0..3]
template <typename Build>
bool tc_maps(mglu_ctx* hd, int kind, const void* Wt, const void* codes, int a, int b, CUtensorMap* out, Build build) {
  std::lock_guard<std::mutex> g(hd->mu);
  for (auto& e : hd->tc_cache)
    if (e.valid && e.kind == kind && e.Wt == Wt && e.codes == codes && e.a == a && e.b == b) {
      e.stamp = ++hd->dec_clock;
      std::memcpy(out, e.m, sizeof(e.m));
      return true;
    }
  CUtensorMap m[4];
  if (!build(m)) return false;
  size_t victim = 0;
  for (size_t i = 0; i < hd->tc_cache.size(); ++i) {
    if (!hd->tc_cache[i].valid) { victim = i; break; }
    if (hd->tc_cache[i].stamp < hd->tc_cache[victim].stamp) victim = i;
  }
  auto& e = hd->tc_cache[victim];
  e.valid = true; e.kind = kind; e.Wt = Wt; e.codes = codes; e.a = a; e.b = b; e.stamp = ++hd->dec_clock;
  std::memcpy(e.m, m, sizeof(m));
  std::memcpy(out, m, sizeof(m));
  return true;
}

// shared-memory budget of the HMMA decode kernel in KB (sets the ring depth; MGLU_DEC_SMEM_KB
// overrides, for experiments)
int dec_smem_kb() {
  static const int v = [] {
    const char* e = getenv("MGLU_DEC_SMEM_KB");
    return e ? atoi(e) : 200;
  }();
  return v;
}

// grid of the HMMA decode kernel (experiments: MGLU_DEC_CTAS caps it below the SM count)
int dec_ctas() {
  static const int v = [] {
    const char* e = getenv("MGLU_DEC_CTAS");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// CTAs of the HMMA decode kernel for this layer: every SM but 4 on large layers -- measured on two
// boxes at config 3 B = 1: 24.64 vs 24.99 us (the driver's 20-step line 25.24 vs 25.65), config 2
// within 1 %, config 5 -0.4 % (profiles/r02/dec_grid.txt); MGLU_DEC_CTAS overrides (experiments)
int64_t dec_grid(const mglu_ctx* hd) {
  const int64_t tiles = (hd->h + 7) / 8;
  const int64_t grid = dec_ctas() > 0 ? std::min(dec_ctas(), hd->num_sms)
                     : (tiles >= (int64_t)hd->num_sms * 8 ? hd->num_sms - 4 : hd->num_sms);
  return std::max<int64_t>(1, std::min<int64_t>(tiles, grid));
}

// deeper ring for the CTAs with one tile more (MGLU_DEC_HEAVY=0 disables)
#ifndef MGLU_DEC_HEAVY_DEFAULT
#define MGLU_DEC_HEAVY_DEFAULT 1
#endif
int dec_heavy() {
  static const int v = [] {
    const char* e = getenv("MGLU_DEC_HEAVY");
    return e ? atoi(e) : MGLU_DEC_HEAVY_DEFAULT;
  }();
  return v;
}

// one-shot L2 prefetch depth of the decode kernel (stages past the ring; MGLU_DEC_L2PF overrides)
int dec_l2pf() {
  static const int v = [] {
    const char* e = getenv("MGLU_DEC_L2PF");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// x in smem, split by pair parity and zero-padded to the last column any stage can touch (the
// widest round type a CTA of this grid runs): u32 words per parity array
int dec_xpar(const mglu_ctx* hd, const mglu::DecParams& p) {
  int64_t maxcol = hd->d;
  for (int64_t nt : {(int64_t)p.tiles_base, (int64_t)p.tiles_base + (p.tiles_rem ? 1 : 0)}) {
    for (int ti = 0; ti < 4; ++ti) {
      const bool used = ti == 0 ? nt >= 8 : ((nt & 7) >> (3 - ti)) & 1;
      if (!used) continue;
      const int64_t ks = 256 << ti;
      maxcol = std::max<int64_t>(maxcol, (hd->d + ks - 1) / ks * ks);
    }
  }
  return (int)(maxcol / 2) / 2 + 8;
}

template <int NM, int ACT, int NB, int KSEL, bool PL = false>
cudaError_t run_mma_nb(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* codes,
                       void* out, const Call& cl) {
  mglu::DecParams p;
  p.x = (const __nv_bfloat16*)x;
  p.out = (__nv_bfloat16*)out;
  p.G = cl.G;
  p.z = cl.z;
  p.variant = hd->variant;
  p.act = hd->act;
  p.B = B;
  p.d = (int)hd->d;
  p.h = (int)hd->h;
  // whole 8-row tiles per CTA, one CTA per SM (the last tile of a ragged h is zero-filled by TMA)
  const int64_t tiles = (hd->h + 7) / 8;
  const int64_t ncta = dec_grid(hd);
  p.ncta = (int)ncta;
  p.tiles_base = (int)(tiles / ncta);
  p.tiles_rem = (int)(tiles % ncta);
  p.l2pf = dec_l2pf();
  p.light_drop = 0;
  mglu::DecMaps maps;
  if (!dec_maps(hd, Wt, codes, &maps, PL)) return cudaErrorInvalidValue;
  p.xpar = dec_xpar(hd, p);
  constexpr size_t SB = mglu::dec_stage_bytes_pl<NM, KSEL, PL>();
  const size_t xbytes = (size_t)2 * B * p.xpar * 4;
  const size_t partbytes = (size_t)mglu::kDecConsumers * 32 * NB * ((KSEL > 0 ? KSEL : NM) + 1) * 4;
  const size_t fixed = xbytes + partbytes + 1024;
  // (dense handles with a long reduction stage a large x: let them use the whole opt-in budget)
  const size_t cap = std::min<size_t>((size_t)hd->max_smem_optin, NM == 0 ? (size_t)hd->max_smem_optin : (size_t)dec_smem_kb() * 1024);
  if (cap < fixed) return cudaErrorInvalidConfiguration;
  int S = (int)((cap - fixed) / (SB + 16));
  S = std::min(8, S);
  if (S < 2) return cudaErrorInvalidConfiguration;
  p.stages = S;
  // heavier CTAs (tiles_base + 1 tiles) one stage deeper than the light ones when a stage fits
  // beside the light CTAs' ring (MGLU_DEC_HEAVY=0 disables, for experiments)
  if (p.tiles_rem && dec_heavy() && S >= 3 && S < 8 && (size_t)(S + 1) * (SB + 16) + fixed <= (size_t)hd->max_smem_optin) {
    p.stages = S + 1;
    p.light_drop = 1;
  }
  const size_t smem = (size_t)p.stages * SB + 2 * p.stages * sizeof(uint64_t) + partbytes + xbytes;
  auto kern = mglu::gemv_mma_kernel<NM, ACT, NB, KSEL, PL>;
  cudaError_t e = smem_optin((const void*)kern, hd->device, std::max((int)smem, hd->max_smem_optin));
  if (e != cudaSuccess) return e;
  return launch_pdl(kern, dim3((unsigned)ncta), dim3(mglu::kDecThreads), smem, cl.st, p, maps);
}

template <int NM, int ACT>
cudaError_t run_mma(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* codes,
                    void* out, const Call& cl) {
  // routed (Top-K) swish forward: evaluate only the masks some token selected -- at most K per
  // token, so min(n_m, B*K) slots, rounded up to a power of two (other activations and larger
  // unions run all masks with the weights in the epilogue)
  if (cl.planes) {
    // plane-major codes: routed Swish calls of B <= 4 only (the selected planes are all a stage loads)
    if constexpr (ACT == mglu::kSwish && NM >= 1) {
      if (!cl.G || cl.K <= 0 || hd->variant != 0 || B > 4) return cudaErrorNotSupported;
      const int u = std::min(NM, B * cl.K);
      if (u <= 1) return run_mma_nb<NM, ACT, 1, 1, true>(hd, x, B, Wt, codes, out, cl);
      if constexpr (NM >= 2)
        if (u <= 2) return run_mma_nb<NM, ACT, 1, 2, true>(hd, x, B, Wt, codes, out, cl);
      if constexpr (NM >= 4)
        if (u <= 4) return run_mma_nb<NM, ACT, 1, 4, true>(hd, x, B, Wt, codes, out, cl);
      if constexpr (NM >= 8) return run_mma_nb<NM, ACT, 1, 8, true>(hd, x, B, Wt, codes, out, cl);
    }
    return cudaErrorNotSupported;
  }
  if constexpr (ACT == mglu::kSwish && NM >= 2) {
    // (B > 4: B*K >= 5 tokens' selections cover min(n_m, 5) >= every slot count below -- all masks)
    if (cl.G && cl.K > 0 && hd->variant == 0 && B <= 4) {
      const int u = std::min(NM, B * cl.K);
      if (u <= 1) return run_mma_nb<NM, ACT, 1, 1>(hd, x, B, Wt, codes, out, cl);
      if (u <= 2 && NM > 2) return run_mma_nb<NM, ACT, 1, 2>(hd, x, B, Wt, codes, out, cl);
      if constexpr (NM == 8)
        if (u <= 4) return run_mma_nb<NM, ACT, 1, 4>(hd, x, B, Wt, codes, out, cl);
    }
  }
  if constexpr (NM > 0) {
    if (cl.z) {                                       // partials: a compile-time instantiation (KSEL = -1)
      if constexpr (NM >= 4) return B <= 4 ? run_mma_nb<NM, mglu::kIdentity, 1, -1>(hd, x, B, Wt, codes, out, cl) : cudaErrorInvalidValue;
      else return B <= 4 ? run_mma_nb<NM, mglu::kIdentity, 1, -1>(hd, x, B, Wt, codes, out, cl)
                         : run_mma_nb<NM, mglu::kIdentity, 2, -1>(hd, x, B, Wt, codes, out, cl);
    }
  }
  if constexpr (NM >= 4) return B <= 4 ? run_mma_nb<NM, ACT, 1, 0>(hd, x, B, Wt, codes, out, cl) : cudaErrorInvalidValue;
  else return B <= 4 ? run_mma_nb<NM, ACT, 1, 0>(hd, x, B, Wt, codes, out, cl)
                     : run_mma_nb<NM, ACT, 2, 0>(hd, x, B, Wt, codes, out, cl);
}

template <int NM>
cudaError_t mma_act(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* codes, void* out,
                    const Call& cl) {
  switch (hd->act) {
    case MGLU_ACT_SWISH: return run_mma<NM, mglu::kSwish>(hd, x, B, Wt, codes, out, cl);
    default: return run_mma<NM, mglu::kRuntimeAct>(hd, x, B, Wt, codes, out, cl);   // g at runtime
  }
}

cudaError_t mma_nm(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* codes, void* out,
                   const Call& cl) {
#ifdef MGLU_DEC_ONLY   // experiment build (tools): the n_m in {1, 4} Swish decode kernels only
  if (hd->act != MGLU_ACT_SWISH || B > 4 || cl.G) return cudaErrorInvalidValue;
  if (hd->n_m == 4) return run_mma_nb<4, mglu::kSwish, 1, 0>(hd, x, B, Wt, codes, out, cl);
  if (hd->n_m == 1) return run_mma_nb<1, mglu::kSwish, 1, 0>(hd, x, B, Wt, codes, out, cl);
  return cudaErrorInvalidValue;
#endif
  switch (hd->n_m) {
    case 0: return run_mma<0, mglu::kIdentity>(hd, x, B, Wt, codes, out, cl);   // dense projection
    case 1: return mma_act<1>(hd, x, B, Wt, codes, out, cl);
    case 2: return mma_act<2>(hd, x, B, Wt, codes, out, cl);
    case 4: return mma_act<4>(hd, x, B, Wt, codes, out, cl);
    default: return mma_act<8>(hd, x, B, Wt, codes, out, cl);
  }
}

// ------------------------------------------------------------------ fused FFN block (row f1)
// DecParams of one handle's decode pass over `ncta` CTAs (whole 8-row tiles per CTA)
mglu::DecParams dec_params(const mglu_ctx* hd, const void* x, int B, void* out, int64_t ncta) {
  mglu::DecParams p;
  p.x = (const __nv_bfloat16*)x;
  p.out = (__nv_bfloat16*)out;
  p.G = nullptr;
  p.z = nullptr;
  p.variant = hd->variant;
  p.act = hd->act;
  p.B = B;
  p.d = (int)hd->d;
  p.h = (int)hd->h;
  const int64_t tiles = (hd->h + 7) / 8;
  p.ncta = (int)ncta;
  p.tiles_base = (int)(tiles / ncta);
  p.tiles_rem = (int)(tiles % ncta);
  p.l2pf = 0;
  p.light_drop = 0;
  p.xpar = dec_xpar(hd, p);
  return p;
}

template <int NM, int ACT>
cudaError_t run_ffn(mglu_ctx* up, mglu_ctx* down, const void* x, int B, const void* Wt, const void* codes,
                    const void* Wo, void* ymid, void* out, cudaStream_t st) {
  // each phase keeps the partition its standalone launch uses (so the result is bit-identical to the
  // composition); the grid is the wider of the two, the extra CTAs own no tiles in the other phase
  const int64_t n1 = dec_grid(up), n2 = dec_grid(down), ncta = std::max(n1, n2);
  mglu::DecParams p1 = dec_params(up, x, B, ymid, n1);
  mglu::DecParams p2 = dec_params(down, ymid, B, out, n2);
  mglu::DecMaps m1, m2;
  if (!dec_maps(up, Wt, codes, &m1) || !dec_maps(down, Wo, nullptr, &m2)) return cudaErrorInvalidValue;
  constexpr size_t SB = mglu::dec_stage_bytes<NM>();
  const size_t xbytes = (size_t)2 * B * std::max(p1.xpar, p2.xpar) * 4;
  const size_t partbytes = (size_t)mglu::kDecConsumers * 32 * (NM + 1) * 4;
  const size_t fixed = xbytes + partbytes + 1024;
  const size_t cap = std::min<size_t>((size_t)up->max_smem_optin, (size_t)dec_smem_kb() * 1024 + 32 * 1024);
  if (cap < fixed + 2 * (SB + 16)) return cudaErrorInvalidConfiguration;
  const int S = (int)std::min<size_t>(8, (cap - fixed) / (SB + 16));
  p1.stages = p2.stages = S;
  const size_t smem = (size_t)S * SB + 2 * S * sizeof(uint64_t) + partbytes + xbytes;
  auto kern = mglu::ffn_mma_kernel<NM, ACT>;
  cudaError_t e = smem_optin((const void*)kern, up->device, std::max((int)smem, up->max_smem_optin));
  if (e != cudaSuccess) return e;
  if (!up->ffn_bar) {
    if ((e = cudaMalloc(&up->ffn_bar, 2 * sizeof(unsigned))) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(up->ffn_bar, 0, 2 * sizeof(unsigned), st)) != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ncta);
  cfg.blockDim = dim3(mglu::kDecThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;               // the grid barrier needs every CTA resident
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // W streams before the previous call ends
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  e = cudaLaunchKernelEx(&cfg, kern, p1, m1, p2, m2, up->ffn_bar);
  if (e == cudaErrorNotSupported || e == cudaErrorInvalidValue) {   // runtime without cooperative + PDL
    (void)cudaGetLastError();
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, p1, m1, p2, m2, up->ffn_bar);
  }
  return e;
}

cudaError_t ffn_nm(mglu_ctx* up, mglu_ctx* down, const void* x, int B, const void* Wt, const void* codes,
                   const void* Wo, void* ymid, void* out, cudaStream_t st) {
  const bool sw = up->act == MGLU_ACT_SWISH;
  switch (up->n_m) {
    case 1: return sw ? run_ffn<1, mglu::kSwish>(up, down, x, B, Wt, codes, Wo, ymid, out, st)
                      : run_ffn<1, mglu::kRuntimeAct>(up, down, x, B, Wt, codes, Wo, ymid, out, st);
    case 2: return sw ? run_ffn<2, mglu::kSwish>(up, down, x, B, Wt, codes, Wo, ymid, out, st)
                      : run_ffn<2, mglu::kRuntimeAct>(up, down, x, B, Wt, codes, Wo, ymid, out, st);
    case 4: return sw ? run_ffn<4, mglu::kSwish>(up, down, x, B, Wt, codes, Wo, ymid, out, st)
                      : run_ffn<4, mglu::kRuntimeAct>(up, down, x, B, Wt, codes, Wo, ymid, out, st);
    case 8: return sw ? run_ffn<8, mglu::kSwish>(up, down, x, B, Wt, codes, Wo, ymid, out, st)
                      : cudaErrorNotSupported;     // (the runtime-g n_m = 8 fused kernel would spill)
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------ tcgen05 (prefill) dispatch
bool tc_can_serve(const mglu_ctx* hd, int64_t B) {
  // TMA of the mask words: rows of d/32 * n_m u32 words must be 16-byte multiples
  return hd->dtype == MGLU_BF16 && (fast_nm(hd->n_m) || hd->n_m == 16) && (hd->d / 32 * hd->n_m) % 4 == 0 && B >= 1 &&
         B <= ((int64_t)1 << 31) - 1;
}

// 2-D row-major [rows][cols] bf16 tensor, box [brows][bcols]
bool encode_2d_bf16(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t bcols, uint32_t brows,
                    CUtensorMapSwizzle swz) {
  EncodeTiledFn enc = get_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {bcols, brows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA swizzle of a code box with rb-byte rows (the kernels read it through lds_words_swz)
CUtensorMapSwizzle code_swizzle(int rb) {
  switch (mglu::code_swizzle_bytes(rb)) {
    case 128: return CU_TENSOR_MAP_SWIZZLE_128B;
    case 64: return CU_TENSOR_MAP_SWIZZLE_64B;
    case 32: return CU_TENSOR_MAP_SWIZZLE_32B;
    default: return CU_TENSOR_MAP_SWIZZLE_NONE;
  }
}

// 2-D row-major [rows][cols] u32 tensor, box [brows][bcols]
bool encode_2d_u32(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t bcols, uint32_t brows,
                   CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
  EncodeTiledFn enc = get_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {bcols, brows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int tc_max_stages() {
  static const int v = [] {
    const char* e = getenv("MGLU_TC_STAGES");   // experiments: ring depth cap of the tile GEMM
    return e ? std::max(2, atoi(e)) : 8;
  }();
  return v;
}

template <int NM, int ACT, int BN>
cudaError_t run_tc_bn(mglu_ctx* hd, const void* x, int64_t B, const void* Wt, const void* codes, void* out,
                      const Call& cl) {
  CUtensorMap mX, mW, mC;
  const auto sw = CU_TENSOR_MAP_SWIZZLE_128B;
  CUtensorMap m[4];
  if (!encode_2d_bf16(&mX, x, hd->d, B, mglu::kTcK, BN, sw) ||
      !tc_maps(hd, 3, Wt, codes, mglu::tc_code_words<NM>(), 0, m, [&](CUtensorMap* o) {
        const bool ok = encode_2d_bf16(&o[0], Wt, hd->d, hd->h, mglu::kTcK, 128, sw) &&
                        encode_2d_u32(&o[1], codes, (uint64_t)hd->d / 32 * NM, hd->h, mglu::tc_code_words<NM>(), 128,
                                      code_swizzle(mglu::tc_code_words<NM>() * 4));
        o[2] = o[0];
        o[3] = o[1];
        return ok;
      }))
    return cudaErrorInvalidValue;
  mW = m[0];
  mC = m[1];
  mglu::TcParams p;
  p.out = (__nv_bfloat16*)out;
  p.G = cl.G;
  p.z = cl.z;
  p.variant = hd->variant;
  p.act = hd->act;
  p.B = (int)B;
  p.d = (int)hd->d;
  p.h = (int)hd->h;
  constexpr size_t SB = mglu::tc_stage_bytes<NM, BN>();
  const size_t fixed = 1024 + 256 + mglu::tc_red_bytes<NM, BN>();   // alignment slack + barriers + split buffer
  const size_t cap = (size_t)hd->max_smem_optin;
  if (cap < fixed + 2 * SB) return cudaErrorInvalidConfiguration;
  const int S = (int)std::min<size_t>((size_t)tc_max_stages(), (cap - fixed) / SB);
  p.stages = S;
  const size_t smem = (size_t)S * SB + fixed;
  auto kern = mglu::gemm_tc_kernel<NM, ACT, BN>;
  cudaError_t e = smem_optin((const void*)kern, hd->device, std::max((int)smem, hd->max_smem_optin));
  if (e != cudaSuccess) return e;
  constexpr int NSPLIT = mglu::tc_split<NM>();
  const dim3 grid((unsigned)((B + BN - 1) / BN), (unsigned)((hd->h + 127) / 128), NSPLIT);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(mglu::kTcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = cl.st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;          // mask-split CTAs (n_m = 8: 2, 16: 4) share DSMEM
  at[1].val.clusterDim.x = 1;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = NSPLIT;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, p, mX, mW, mC);
}

// token tile: small batches take the smallest tile that holds them (the MMA work then scales with
// B and the kernel streams W and the mask words at HBM rate); large batches the TMEM-limited tile
template <int NM, int ACT>
cudaError_t run_tc(mglu_ctx* hd, const void* x, int64_t B, const void* Wt, const void* codes, void* out,
                   const Call& cl) {
  if (B <= 16) return run_tc_bn<NM, ACT, 16>(hd, x, B, Wt, codes, out, cl);
  if (B <= 32) return run_tc_bn<NM, ACT, 32>(hd, x, B, Wt, codes, out, cl);
  if constexpr (mglu::TcCfg<NM>::BN <= 32) return run_tc_bn<NM, ACT, 32>(hd, x, B, Wt, codes, out, cl);
  else {
    if (B <= 64 || mglu::TcCfg<NM>::BN == 64) return run_tc_bn<NM, ACT, 64>(hd, x, B, Wt, codes, out, cl);
    return run_tc_bn<NM, ACT, mglu::TcCfg<NM>::BN>(hd, x, B, Wt, codes, out, cl);
  }
}

template <int NM>
cudaError_t tc_act(mglu_ctx* hd, const void* x, int64_t B, const void* Wt, const void* codes, void* out,
                   const Call& cl) {
  switch (hd->act) {
    case MGLU_ACT_SWISH: return run_tc<NM, mglu::kSwish>(hd, x, B, Wt, codes, out, cl);
    default: return run_tc<NM, mglu::kRuntimeAct>(hd, x, B, Wt, codes, out, cl);   // g at runtime
  }
}

cudaError_t tc_nm(mglu_ctx* hd, const void* x, int64_t B, const void* Wt, const void* codes, void* out,
                  const Call& cl) {
#ifdef MGLU_DEC_ONLY
  return cudaErrorInvalidValue;
#endif
  switch (hd->n_m) {
    case 1: return tc_act<1>(hd, x, B, Wt, codes, out, cl);
    case 2: return tc_act<2>(hd, x, B, Wt, codes, out, cl);
    case 4: return tc_act<4>(hd, x, B, Wt, codes, out, cl);
    case 8: return tc_act<8>(hd, x, B, Wt, codes, out, cl);
    case 16: return tc_act<16>(hd, x, B, Wt, codes, out, cl);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------ tcgen05 stream-K decode dispatch
constexpr int kSkMaxB = 64;
constexpr int kAutoMmaMaxB = 4, kAutoSkMaxB = 16, kAutoRowMaxB = 32;

bool sk_can_serve(const mglu_ctx* hd, int64_t B) {
  // 128-column units; mask-word rows of d/32 * n_m u32 words must be 16-byte multiples (TMA)
  return hd->dtype == MGLU_BF16 && fast_nm(hd->n_m) && hd->d % 64 == 0 && (hd->d / 32 * hd->n_m) % 4 == 0 && B >= 1 &&
         B <= kSkMaxB && (hd->n_m < 8 || B <= 32);
}

// stream-K workspace, grown on demand (the first call of a larger batch): 2 published partials per
// CTA (its first and last segments) of (n_m + 1) x B x 128 fp32, and one ticket per 128-row tile
// (zeroed once; the last arriver of a tile re-arms it)
cudaError_t sk_workspace(mglu_ctx* hd, size_t ws_bytes, cudaStream_t st) {
  const size_t tiles = (size_t)((hd->h + 127) / 128);
  if (!hd->sk_tickets) {
    cudaError_t e = cudaMalloc(&hd->sk_tickets, tiles * sizeof(uint32_t));
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(hd->sk_tickets, 0, tiles * sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
  }
  if (hd->sk_ws_bytes < ws_bytes) {
    if (hd->sk_ws) { cudaStreamSynchronize(st); cudaFree(hd->sk_ws); hd->sk_ws = nullptr; hd->sk_ws_bytes = 0; }
    cudaError_t e = cudaMalloc(&hd->sk_ws, ws_bytes);
    if (e != cudaSuccess) return e;
    hd->sk_ws_bytes = ws_bytes;
  }
  return cudaSuccess;
}

// row split (each tile owned by one CTA over the whole d: no cross-CTA reduction, no workspace,
// k-order independent of h) when every SM gets at least kSkRowMin rows; stream-K below that (small
// shards, where 128-row tiles would leave the maskers mostly idle rows)
constexpr int64_t kSkRowMin = 64;
int sk_rows_env() {
  static const int v = [] {
    const char* e = getenv("MGLU_SK_ROWS");   // experiments / tests: 0 forces stream-K, 1 the row split
    return e ? atoi(e) : -1;
  }();
  return v;
}
int sk_max_wstages() {
  static const int v = [] {
    const char* e = getenv("MGLU_SK_WSTAGES");   // experiments: W ring depth cap
    return e ? atoi(e) : 3;   // 3: measured best after the epilogue fix (row split B = 8: 29.7 us vs 30.7 with 5, 31.3 with 6; profiles/r02/tc_gemv_experiments.txt)
  }();
  return v;
}
// AUTO's choice between the two forms of the tcgen05 GEMV (profiles/r02/tcrow_sweep.txt, config 3):
// the row split wins once the stream-K fix-up grows with B (from B = 5, tied there) on layers wide enough to give
// every SM kSkRowMin rows; at n_m = 8 the maskers' cost per 128-row unit dominates and the row
// split's partly idle lanes lose (config 5, B = 1: 159 vs 129 us)
int sk_ctas() {
  static const int v = [] {
    const char* e = getenv("MGLU_SK_CTAS");   // experiments: row-split grid
    return e ? atoi(e) : 0;
  }();
  return v;
}
int sk_xstages() {
  static const int v = [] {
    const char* e = getenv("MGLU_SK_XSTAGES");   // experiments: x ring depth
    return e ? std::max(2, atoi(e)) : 4;
  }();
  return v;
}
bool auto_row_split(const mglu_ctx* hd, int64_t B) {
  const int env = sk_rows_env();
  if (env >= 0) return env == 1;
  // n_m = 8: only while every CTA has a single tile (h <= 128 #SM; config 3 B = 8: 45.9 vs 51.0 us),
  // two 97-row tiles per CTA lose to stream-K (config 5 B = 8: 168.6 vs 149.5 us)
  if (B < 5) return false;
  if (hd->h >= (int64_t)hd->num_sms * kSkRowMin) return hd->n_m <= 4 || hd->h <= (int64_t)hd->num_sms * 128;
  // narrow layers (h-shards): the row split costs ~29 us whatever the rows (every CTA walks all of d),
  // which beats the stream-K fix-up from B = 16 and the tile GEMM up to B = 32 (h = 1792 / 3584 /
  // 7168, B = 16: 29.4 / 29.5 / 29.7 us vs stream-K 45.1 / 30.6 / 29.4; profiles/r02/narrow_paths.txt)
  return hd->n_m <= 4 && B >= 16;
}

template <int NM, int BN, int MG>
cudaError_t run_sk_bn(mglu_ctx* hd, const void* x, int64_t B, const void* Wt, const void* codes, void* out,
                      const Call& cl) {
  using C = mglu::SkCfg<NM, BN, MG>;
  CUtensorMap mW, mX, mC, mWb, mCb;
  const auto sw = CU_TENSOR_MAP_SWIZZLE_128B;
  constexpr int KB = C::KS / 64;
  mglu::SkParams p;
  p.out = (__nv_bfloat16*)out;
  p.G = cl.G;
  p.z = cl.z;
  p.variant = hd->variant;
  p.B = (int)B;
  p.d = (int)hd->d;
  p.h = (int)hd->h;
  p.act = hd->act;
  p.upt = (int)((hd->d + C::KS - 1) / C::KS);   // a final partial unit reads zero-filled boxes
  p.row_mode = cl.row_split ? 1 : 0;
  if (!encode_3d_blocks(&mX, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, hd->d, B, 64, BN, KB, sw))
    return cudaErrorInvalidValue;
  int64_t G;
  if (p.row_mode) {
    // G CTAs x tpc tiles of tr_base or tr_base + 1 (<= 128) rows; the first tr_rem tiles are the big
    // ones.  Boxes of exactly a tile's rows: nothing is read twice or past the tile.
    // every SM but 4, as the HMMA kernel (config 3 B = 8 / 16 / 32: 29.41 / 30.14 / 35.15 us vs
    // 29.78 / 30.55 / 36.10 on all 148; profiles/r02/dec_grid.txt)
    G = std::min<int64_t>(sk_ctas() > 0 ? std::min(sk_ctas(), hd->num_sms) : std::max(1, hd->num_sms - 4), hd->h);
    p.tpc = (int)((hd->h + G * 128 - 1) / (G * 128));
    const int64_t nt = G * p.tpc;
    p.tr_base = (int)(hd->h / nt);
    p.tr_rem = (int)(hd->h % nt);
    const uint32_t rb = (uint32_t)p.tr_base + (p.tr_rem ? 1u : 0u);
    const uint64_t crow = (uint64_t)hd->d / 32 * NM;
    CUtensorMap m[4];
    if (!tc_maps(hd, 1, Wt, codes, (int)rb, p.tr_base * 64 + C::CWORDS, m, [&](CUtensorMap* o) {
          return encode_2d_bf16(&o[0], Wt, hd->d, hd->h, 64, rb, sw) &&
                 encode_2d_u32(&o[1], codes, crow, hd->h, C::CWORDS, rb, code_swizzle(C::CWORDS * 4)) &&
                 encode_2d_bf16(&o[2], Wt, hd->d, hd->h, 64, (uint32_t)p.tr_base, sw) &&
                 encode_2d_u32(&o[3], codes, crow, hd->h, C::CWORDS, (uint32_t)p.tr_base, code_swizzle(C::CWORDS * 4));
        }))
      return cudaErrorInvalidValue;
    mW = m[0]; mC = m[1]; mWb = m[2]; mCb = m[3];
    p.units_base = p.units_rem = 0;
    p.ws = nullptr;
    p.tickets = nullptr;
  } else {
    CUtensorMap m[4];
    if (!tc_maps(hd, 2, Wt, codes, C::CWORDS, 0, m, [&](CUtensorMap* o) {
          const bool ok = encode_3d_blocks(&o[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Wt, hd->d, hd->h, 64, 128, KB, sw) &&
                          encode_2d_u32(&o[1], codes, (uint64_t)hd->d / 32 * NM, hd->h, C::CWORDS, 128, code_swizzle(C::CWORDS * 4));
          o[2] = o[0];
          o[3] = o[1];
          return ok;
        }))
      return cudaErrorInvalidValue;
    mW = m[0]; mC = m[1]; mWb = m[2]; mCb = m[3];
    const int64_t units = (hd->h + 127) / 128 * p.upt;
    G = std::min<int64_t>(sk_ctas() > 0 ? std::min(sk_ctas(), hd->num_sms) : hd->num_sms, units);
    p.units_base = (int)(units / G);
    p.units_rem = (int)(units % G);
    p.tpc = p.tr_base = p.tr_rem = 0;
    cudaError_t e = sk_workspace(hd, (size_t)hd->num_sms * 2 * C::NOP * BN * 128 * sizeof(float), cl.st);
    if (e != cudaSuccess) return e;
    p.ws = hd->sk_ws;
    p.tickets = hd->sk_tickets;
  }
  // one accumulator set (and the TMEM it frees as A slots) when the CTA has a single segment
  const bool one_seg = p.row_mode && p.tpc == 1;
  // stage layout: 64-column W blocks of the tile's rows (rounded to the 8-row swizzle atom) and the
  // code box behind them -- in the row split a stage holds only the tile's rows, so more stages fit
  if (p.row_mode) {
    const int rmax = p.tr_base + (p.tr_rem ? 1 : 0);
    p.wblk = (rmax + 7) / 8 * 1024;
    p.wsb = (C::KS / 64 * p.wblk + rmax * C::CWORDS * 4 + 1023) / 1024 * 1024;
  } else {
    p.wblk = 16384;
    p.wsb = C::WSB;
  }
  const size_t cap = (size_t)hd->max_smem_optin;
  p.xstages = sk_xstages();
  const size_t fixed = 1024 + 512 + (size_t)p.xstages * C::XB;   // alignment slack + barriers + x ring
  if (cap < fixed + 2 * (size_t)p.wsb) return cudaErrorInvalidConfiguration;
  p.wstages = (int)std::min<size_t>(sk_max_wstages(), (cap - fixed) / p.wsb);
  const size_t smem = (size_t)p.wstages * p.wsb + fixed;
  auto kern = one_seg ? mglu::gemv_tc_kernel<NM, BN, MG, true> : mglu::gemv_tc_kernel<NM, BN, MG, false>;
  cudaError_t e = smem_optin((const void*)kern, hd->device, hd->max_smem_optin);
  if (e != cudaSuccess) return e;
  return launch_pdl(kern, dim3((unsigned)G), dim3(C::THREADS), smem, cl.st, p, mW, mX, mC, mWb, mCb);
}

// two masker groups when the TMEM budget allows, else one
template <int NM, int BN>
cudaError_t run_sk_mg(mglu_ctx* hd, const void* x, int64_t B, const void* Wt, const void* codes, void* out,
                      const Call& cl) {
#ifndef MGLU_SK_MG8
#define MGLU_SK_MG8 2
#endif
  if constexpr (NM >= 8 && MGLU_SK_MG8 == 4 && mglu::SkCfg<NM, BN, 4>::ok) return run_sk_bn<NM, BN, 4>(hd, x, B, Wt, codes, out, cl);
  if constexpr (mglu::SkCfg<NM, BN, 2>::ok) return run_sk_bn<NM, BN, 2>(hd, x, B, Wt, codes, out, cl);
  else return run_sk_bn<NM, BN, 1>(hd, x, B, Wt, codes, out, cl);
}

template <int NM>
cudaError_t run_sk(mglu_ctx* hd, const void* x, int64_t B, const void* Wt, const void* codes, void* out,
                   const Call& cl) {
  if (B <= 16) return run_sk_mg<NM, 16>(hd, x, B, Wt, codes, out, cl);
  if (B <= 32) return run_sk_mg<NM, 32>(hd, x, B, Wt, codes, out, cl);
  if constexpr (NM < 8) return run_sk_mg<NM, 64>(hd, x, B, Wt, codes, out, cl);
  return cudaErrorInvalidValue;
}

cudaError_t sk_nm(mglu_ctx* hd, const void* x, int64_t B, const void* Wt, const void* codes, void* out,
                  const Call& cl) {
#ifdef MGLU_DEC_ONLY
  return cudaErrorInvalidValue;
#endif
  switch (hd->n_m) {
    case 1: return run_sk<1>(hd, x, B, Wt, codes, out, cl);
    case 2: return run_sk<2>(hd, x, B, Wt, codes, out, cl);
    case 4: return run_sk<4>(hd, x, B, Wt, codes, out, cl);
    default: return run_sk<8>(hd, x, B, Wt, codes, out, cl);
  }
}

mglu_status check_ptrs(mglu_ctx* hd, const void* x, int64_t B, const void* Wt, const void* codes,
                       const void* out) {
  if (!hd) return MGLU_ERR_INVALID_ARG;
  if (B < 0) return set_err(hd, MGLU_ERR_INVALID_ARG, "B < 0");
  if (!x || !Wt || (!codes && hd->n_m) || !out) return set_err(hd, MGLU_ERR_INVALID_ARG, "null data pointer");
  if (!aligned16(x) || !aligned16(Wt) || (hd->n_m && !aligned16(codes)) || !aligned16(out))
    return set_err(hd, MGLU_ERR_MISALIGNED, "data pointers must be 16-byte aligned");
  if (B > (int64_t)1 << 30) return set_err(hd, MGLU_ERR_INVALID_ARG, "B too large");
  return MGLU_OK;
}

}  // namespace

// ------------------------------------------------------------------ packing helpers
static void put_le32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}
static uint32_t get_le32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

template <typename BitOf>
static void pack_words(int n_m, int64_t h, int64_t d, uint8_t* packed, BitOf bit_of) {
  const int64_t groups = d / 32;
  for (int64_t j = 0; j < h; ++j)
    for (int64_t g = 0; g < groups; ++g)
      for (int i = 0; i < n_m; ++i) {
        uint32_t v = 0;
        for (int e = 0; e < 32; ++e) v |= bit_of(i, j, g * 32 + e) << mglu::code_bit_of(e);
        put_le32(packed + ((j * groups + g) * n_m + i) * 4, v);
      }
}

static mglu_status device_launch_check(cudaError_t e) {
  return e == cudaSuccess ? MGLU_OK : MGLU_ERR_CUDA;
}

static unsigned grid_for(int64_t n) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  return (unsigned)std::max<int64_t>(1, blocks);
}

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
  if (d < 0 || h < 0 || !valid_nm(n_m) || d % 32) return 0;
  return (size_t)(h * d * n_m / 8);
}

mglu_status mglu_create(mglu_handle* out, int64_t d, int64_t h, int n_m, int act, int dtype,
                        int device) {
  if (!out) return MGLU_ERR_INVALID_ARG;
  *out = nullptr;
  if (d < 1 || h < 1 || act < 0 || act > 4 || (dtype != MGLU_BF16 && dtype != MGLU_F32) || device < 0)
    return MGLU_ERR_INVALID_ARG;
  if ((!valid_nm(n_m) && n_m != 0) || d % 32 != 0 || h > ((int64_t)1 << 31) - 1 || d > ((int64_t)1 << 24))
    return MGLU_ERR_UNSUPPORTED;
  if (n_m == 0 && dtype != MGLU_BF16) return MGLU_ERR_UNSUPPORTED;   // dense projection: bf16 MMA path
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

mglu_status mglu_reserve(mglu_handle hd, int64_t max_B, void* stream) {
  if (!hd || max_B < 0) return MGLU_ERR_INVALID_ARG;
  if (hd->dtype != MGLU_BF16 || !fast_nm(hd->n_m) || max_B == 0) return MGLU_OK;   // no stream-K path
  const int64_t b = std::min<int64_t>(max_B, hd->n_m == 8 ? 32 : kSkMaxB);
  const int64_t bn = b <= 16 ? 16 : b <= 32 ? 32 : 64;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != hd->device) cudaSetDevice(hd->device);
  const cudaError_t e = sk_workspace(hd, (size_t)hd->num_sms * 2 * (hd->n_m + 1) * bn * 128 * sizeof(float),
                                     (cudaStream_t)stream);
  if (prev != hd->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? MGLU_ERR_OOM : cuda_fail(hd, e, "mglu_reserve");
  return MGLU_OK;
}

mglu_status mglu_destroy(mglu_handle hd) {
  if (!hd) return MGLU_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(hd->device);
  if (hd->x_stage) cudaFree(hd->x_stage);
  if (hd->y_stage) cudaFree(hd->y_stage);
  if (hd->sk_ws) cudaFree(hd->sk_ws);
  if (hd->sk_tickets) cudaFree(hd->sk_tickets);
  if (hd->bw_ws) cudaFree(hd->bw_ws);
  if (hd->ffn_bar) cudaFree(hd->ffn_bar);
  cudaSetDevice(prev);
  delete hd;
  return MGLU_OK;
}

mglu_status mglu_set_path(mglu_handle hd, int path) {
  if (!hd || path < MGLU_PATH_AUTO || path > MGLU_PATH_TCROW) return MGLU_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> g(hd->mu);
  hd->path = path;
  return MGLU_OK;
}

mglu_status mglu_set_variant(mglu_handle hd, int variant) {
  if (!hd || variant < 0 || variant > 3) return MGLU_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> g(hd->mu);
  hd->variant = variant;
  return MGLU_OK;
}

mglu_status mglu_set_debug(mglu_handle hd, int flags) {
  if (!hd || (flags & ~MGLU_DEBUG_FLIP_MASK_BIT)) return MGLU_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> g(hd->mu);
  hd->debug = flags;
  return MGLU_OK;
}

int mglu_last_launch_count(mglu_handle hd) { return hd ? hd->last_launches : -1; }
int mglu_last_path(mglu_handle hd) { return hd ? hd->last_path : -1; }

}  // extern "C"

// the forward on an explicit path (AUTO resolved here); shared by mglu_forward and
// mglu_forward_routed
// AUTO: the path mglu_forward takes for this handle and batch
static int auto_path(const mglu_ctx* hd, int64_t B) {
  int path;
  // measured crossovers at the Llama-3-8B FFN shape (profiles/r02/tcrow_sweep.txt): the
  // register-masked HMMA kernel for B <= 4 (one 8-column MMA tile), the tcgen05 GEMV for
  // 5 <= B <= 32 on wide layers as its row split (stream-K up to 16 on narrow ones),
  // the tcgen05 tile GEMM above; SIMT for fp32 and shapes the others refuse
  // (n_m = 8 on large layers: the HMMA kernel's 9 MMAs per step make it compute-bound, and the
  //  stream-K tcgen05 GEMV wins from B = 1: 129 vs 138 us at d=8192 h=28672; on small shards
  //  (h < 8192) the HMMA kernel stays ahead)
  // (the row split's upper batch is 64 / 48 / 32 for n_m = 1 / 2 / >= 4: fewer masked operands per
  //  unit keep it ahead of the tile GEMM longer -- profiles/r02/nm12_paths.txt;
  //  n_m = 8 on large layers keeps stream-K up to its B <= 32 limit: config 5 B = 32 264.9 vs 275.3 us
  //  for the tile GEMM; at B <= 4 the HMMA kernel ties or wins: config 5 135.8 vs 136.5, config 3
  //  38.3 vs 42.8 us -- profiles/r02/nm8_paths.txt)
  const bool nm8_big = hd->n_m == 8 && hd->h >= 8192;
  if (B <= kAutoMmaMaxB && mma_can_serve(hd, B))
    path = MGLU_PATH_MMA;
  else if (B <= (hd->n_m == 1 ? 64 : hd->n_m == 2 ? 48 : kAutoRowMaxB) && sk_can_serve(hd, B) && auto_row_split(hd, B))
    path = MGLU_PATH_TCROW;
  else if ((B <= kAutoSkMaxB || nm8_big) && sk_can_serve(hd, B))
    path = MGLU_PATH_TCDEC;
  else if (mma_can_serve(hd, B))
    path = MGLU_PATH_MMA;
  else if (tc_can_serve(hd, B))
    path = MGLU_PATH_TCGEN05;
  else
    path = MGLU_PATH_SIMT;
  return path;
}

// mglu_forward_host with page-locked, device-mapped host buffers: the copies are small kernels in
// the PDL chain instead of cudaMemcpyAsync (which the forward kernel could not overlap): the
// copy-in grid releases its dependent at once, so the forward's producer streams W while x
// crosses PCIe (the forward reads x only after griddepcontrol.wait); the copy-out grid launches
// during the forward's tail and waits for it before reading y.
__global__ void stage_in_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t n) {
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t n16 = n / 16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  for (int64_t i = n16 * 16 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void stage_out_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");      // y is the predecessor's output
  const int64_t n16 = n / 16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  for (int64_t i = n16 * 16 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
// device alias of a page-locked, mapped host buffer (nullptr for pageable / unregistered memory)
static void* mapped_alias(const void* host) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, host) != cudaSuccess) { (void)cudaGetLastError(); return nullptr; }
  if (a.type != cudaMemoryTypeHost || !a.devicePointer) return nullptr;
  return a.devicePointer;
}
static unsigned stage_grid(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(64, (n / 16 + 255) / 256));
}

// test hook: flip one bit of the caller's packed codes (mglu_set_debug)
__global__ void flip_bit_kernel(uint8_t* p, uint8_t m) { p[0] ^= m; }

static mglu_status forward_on_path(mglu_handle hd, const void* x, int64_t B, const void* Wt,
                                   const void* packed, void* out, int path, const Call& cl) {
  mglu_status s = check_ptrs(hd, x, B, Wt, packed, cl.z ? (const void*)cl.z : out);
  if (s != MGLU_OK) return s;
  hd->last_launches = 0;
  if (B == 0) return MGLU_OK;
  if (hd->n_m == 0) {                                       // dense projection (FFN W_o): MMA path only
    if (!mma_can_serve(hd, B) || (path != MGLU_PATH_AUTO && path != MGLU_PATH_MMA))
      return set_err(hd, MGLU_ERR_UNSUPPORTED, "dense (n_m = 0) handles: MMA path, bf16, 1 <= B <= 8, d % 128 == 0");
    path = MGLU_PATH_MMA;
  }
  if (path == MGLU_PATH_AUTO) path = auto_path(hd, B);
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != hd->device) cudaSetDevice(hd->device);
  cudaError_t e = cudaSuccess;
  int launches = 0;
  const bool fault = (hd->debug & MGLU_DEBUG_FLIP_MASK_BIT) && packed && hd->n_m > 0;
  if (fault) flip_bit_kernel<<<1, 1, 0, cl.st>>>((uint8_t*)const_cast<void*>(packed), 1);
  if (path == MGLU_PATH_MMA) {
    if (!mma_can_serve(hd, B)) {
      if (prev != hd->device) cudaSetDevice(prev);
      return set_err(hd, MGLU_ERR_UNSUPPORTED, "MMA path needs bf16, 1 <= B <= 8 (B <= 4 for n_m >= 4), d % 128 == 0");
    }
    e = mma_nm(hd, x, (int)B, Wt, packed, out, cl);
    launches = 1;
  } else if (path == MGLU_PATH_TCGEN05) {
    if (!tc_can_serve(hd, B)) {
      if (prev != hd->device) cudaSetDevice(prev);
      return set_err(hd, MGLU_ERR_UNSUPPORTED, "tcgen05 path needs bf16 and d * n_m % 128 == 0");
    }
    e = tc_nm(hd, x, B, Wt, packed, out, cl);
    launches = 1;
  } else if (path == MGLU_PATH_TCDEC || path == MGLU_PATH_TCROW) {
    if (!sk_can_serve(hd, B)) {
      if (prev != hd->device) cudaSetDevice(prev);
      return set_err(hd, MGLU_ERR_UNSUPPORTED,
                     "tcgen05 decode path needs bf16, 1 <= B <= 64 (32 for n_m = 8), d % 64 == 0, d * n_m % 128 == 0");
    }
    Call c2 = cl;
    c2.row_split = path == MGLU_PATH_TCROW;
    e = sk_nm(hd, x, B, Wt, packed, out, c2);
    launches = 1;
  } else {
    if (cl.z)
      e = hd->dtype == MGLU_BF16 ? simt_nm<__nv_bfloat16, true>(hd, x, (int)B, Wt, packed, nullptr, cl.z, cl)
                                 : simt_nm<float, true>(hd, x, (int)B, Wt, packed, nullptr, cl.z, cl);
    else
      e = hd->dtype == MGLU_BF16 ? simt_nm<__nv_bfloat16, false>(hd, x, (int)B, Wt, packed, out, nullptr, cl)
                                 : simt_nm<float, false>(hd, x, (int)B, Wt, packed, out, nullptr, cl);
    launches = 1;
  }
  if (fault) flip_bit_kernel<<<1, 1, 0, cl.st>>>((uint8_t*)const_cast<void*>(packed), 1);
  if (prev != hd->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(hd, e, "mglu_forward launch");
  hd->last_path = path;
  hd->last_launches = launches;
  return MGLU_OK;
}

extern "C" {

mglu_status mglu_forward(mglu_handle hd, const void* x, int64_t B, const void* Wt,
                         const void* packed, void* out, void* stream) {
  if (!hd) return MGLU_ERR_INVALID_ARG;
  int path;
  {
    std::lock_guard<std::mutex> g(hd->mu);
    path = hd->path;
  }
  Call cl;
  cl.st = (cudaStream_t)stream;
  return forward_on_path(hd, x, B, Wt, packed, out, path, cl);
}

mglu_status mglu_router_topk(mglu_handle hd, const void* x, int64_t B, const void* Wr, int K, float* G,
                             void* stream) {
  if (!hd) return MGLU_ERR_INVALID_ARG;
  if (B < 0 || !x || !Wr || !G) return set_err(hd, MGLU_ERR_INVALID_ARG, "null pointer or B < 0");
  if (K < 1 || K > hd->n_m) return set_err(hd, MGLU_ERR_INVALID_ARG, "K must be in [1, n_m]");
  if (hd->dtype != MGLU_BF16) return set_err(hd, MGLU_ERR_UNSUPPORTED, "router: bf16 handles only");
  if (!fast_nm(hd->n_m)) return set_err(hd, MGLU_ERR_UNSUPPORTED, "router: n_m in {1, 2, 4, 8}");
  if (!aligned16(x) || !aligned16(Wr) || !aligned16(G)) return set_err(hd, MGLU_ERR_MISALIGNED, "16-byte alignment");
  hd->last_launches = 0;
  if (B == 0) return MGLU_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != hd->device) cudaSetDevice(hd->device);
  const dim3 grid((unsigned)B), block(256);              // one CTA per token
  cudaStream_t st = (cudaStream_t)stream;
  const auto* xb = (const __nv_bfloat16*)x;
  const auto* wr = (const __nv_bfloat16*)Wr;
  cudaError_t e;
  switch (hd->n_m) {
    case 1: e = launch_pdl(mglu::router_topk_kernel<1>, grid, block, 0, st, xb, (int)B, (int)hd->d, wr, K, G); break;
    case 2: e = launch_pdl(mglu::router_topk_kernel<2>, grid, block, 0, st, xb, (int)B, (int)hd->d, wr, K, G); break;
    case 4: e = launch_pdl(mglu::router_topk_kernel<4>, grid, block, 0, st, xb, (int)B, (int)hd->d, wr, K, G); break;
    default: e = launch_pdl(mglu::router_topk_kernel<8>, grid, block, 0, st, xb, (int)B, (int)hd->d, wr, K, G); break;
  }
  if (prev != hd->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(hd, e, "mglu_router_topk launch");
  hd->last_launches = 1;
  return MGLU_OK;
}

mglu_status mglu_forward_routed(mglu_handle hd, const void* x, int64_t B, const void* Wt, const void* packed,
                                const float* G, int K, void* out, void* stream) {
  mglu_status s = check_ptrs(hd, x, B, Wt, packed, out);
  if (s != MGLU_OK) return s;
  if (!G) return set_err(hd, MGLU_ERR_INVALID_ARG, "null gate weights");
  if (K < 0 || K > hd->n_m) return set_err(hd, MGLU_ERR_INVALID_ARG, "K must be in [0, n_m]");
  if (!aligned16(G)) return set_err(hd, MGLU_ERR_MISALIGNED, "gate weights must be 16-byte aligned");
  int path;
  {
    std::lock_guard<std::mutex> g(hd->mu);
    path = hd->path;
  }
  // the routed weights reach every launcher in the call arguments; the MMA path also skips the
  // masks no token selected, the tensor-core paths weigh every mask in their epilogues
  if (path == MGLU_PATH_AUTO && K > 0 && mma_can_serve(hd, B)) path = MGLU_PATH_MMA;   // it skips masks
  Call cl;
  cl.st = (cudaStream_t)stream;
  cl.G = G;
  cl.K = K;
  return forward_on_path(hd, x, B, Wt, packed, out, path, cl);
}

mglu_status mglu_ffn_forward(mglu_handle up, mglu_handle down, const void* x, int64_t B, const void* Wt,
                             const void* packed, const void* Wo, void* y_mid, void* out, void* stream) {
  if (!up || !down) return MGLU_ERR_INVALID_ARG;
  mglu_status s = check_ptrs(up, x, B, Wt, packed, y_mid);
  if (s != MGLU_OK) return s;
  if (!Wo || !out) return set_err(up, MGLU_ERR_INVALID_ARG, "null W_o / out");
  if (y_mid == out || y_mid == x || out == x)
    return set_err(up, MGLU_ERR_INVALID_ARG, "x, y_mid and out must be distinct buffers (phase 2 reads y_mid while writing out)");
  if (!aligned16(Wo) || !aligned16(out)) return set_err(up, MGLU_ERR_MISALIGNED, "W_o / out must be 16-byte aligned");
  if (down->n_m != 0 || down->d != up->h || down->device != up->device || down->dtype != MGLU_BF16)
    return set_err(up, MGLU_ERR_INVALID_ARG, "down must be a dense (n_m = 0) bf16 handle with d = up.h on up's device");
  if (B == 0) return MGLU_OK;
  if (!fast_nm(up->n_m) || B > 4 || !mma_can_serve(up, B) || !mma_can_serve(down, B) ||
      (up->n_m == 8 && up->act != MGLU_ACT_SWISH))
    return set_err(up, MGLU_ERR_UNSUPPORTED,
                   "fused FFN: bf16, n_m in {1, 2, 4, 8} (Swish at n_m = 8), 1 <= B <= 4, d % 128 == 0 and h % 128 == 0");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != up->device) cudaSetDevice(up->device);
  const cudaError_t e = ffn_nm(up, down, x, (int)B, Wt, packed, Wo, y_mid, out, (cudaStream_t)stream);
  if (prev != up->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(up, e, "mglu_ffn_forward launch");
  up->last_path = MGLU_PATH_MMA;
  up->last_launches = 1;
  return MGLU_OK;
}

mglu_status mglu_forward_routed_planes(mglu_handle hd, const void* x, int64_t B, const void* Wt, const void* planes,
                                       const float* G, int K, void* out, void* stream) {
  mglu_status s = check_ptrs(hd, x, B, Wt, planes, out);
  if (s != MGLU_OK) return s;
  if (!G) return set_err(hd, MGLU_ERR_INVALID_ARG, "null gate weights");
  if (K < 1 || K > hd->n_m) return set_err(hd, MGLU_ERR_INVALID_ARG, "K must be in [1, n_m]");
  if (!aligned16(G)) return set_err(hd, MGLU_ERR_MISALIGNED, "gate weights must be 16-byte aligned");
  int path, variant;
  {
    std::lock_guard<std::mutex> g(hd->mu);
    path = hd->path;
    variant = hd->variant;
  }
  if (!mma_can_serve(hd, B) || B > 4 || hd->act != MGLU_ACT_SWISH || variant != 0 || hd->n_m < 1 ||
      (path != MGLU_PATH_AUTO && path != MGLU_PATH_MMA))
    return set_err(hd, MGLU_ERR_UNSUPPORTED,
                   "plane-major routed forward: MMA path, bf16, Swish, standard variant, 1 <= B <= 4, d % 128 == 0");
  Call cl;
  cl.st = (cudaStream_t)stream;
  cl.G = G;
  cl.K = K;
  cl.planes = true;
  return forward_on_path(hd, x, B, Wt, planes, out, MGLU_PATH_MMA, cl);
}

mglu_status mglu_forward_partials(mglu_handle hd, const void* x, int64_t B, const void* Wt,
                                  const void* packed, float* z, void* stream) {
  if (!hd) return MGLU_ERR_INVALID_ARG;
  if (hd->n_m == 0) return set_err(hd, MGLU_ERR_UNSUPPORTED, "partials need masks (n_m >= 1)");
  if (!z) return set_err(hd, MGLU_ERR_INVALID_ARG, "null z");
  int path;
  {
    std::lock_guard<std::mutex> g(hd->mu);
    path = hd->path;
  }
  // AUTO: the SIMT kernel (Alg. 1 as written); an explicit path: that kernel, whose epilogue writes
  // s_i and t - s_i instead of y (each fast path's own value streams, for the parity tests)
  if (path == MGLU_PATH_AUTO) path = MGLU_PATH_SIMT;
  Call cl;
  cl.st = (cudaStream_t)stream;
  cl.z = z;
  return forward_on_path(hd, x, B, Wt, packed, nullptr, path, cl);
}

}  // extern "C"

// ------------------------------------------------------------------ training path (row f4)
template <typename T, int NM>
static cudaError_t backward_kernels(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* packed,
                                    const float* dy, float* dx, float* dW, float* dlogits, const float* z, float* E,
                                    cudaStream_t st) {
  const int d = (int)hd->d, h = (int)hd->h;
  const int64_t n = (int64_t)B * h;
  mglu::coef_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)hd->num_sms * 16), 256, 0, st>>>(
      z, dy, B, h, NM, hd->act, E);
  if (dW || dlogits)
    mglu::dw_kernel<T, NM><<<dim3((unsigned)((d + mglu::kBwK - 1) / mglu::kBwK), (unsigned)((h + mglu::kBwJ - 1) / mglu::kBwJ)),
                             256, 0, st>>>((const T*)x, (const T*)Wt, (const uint32_t*)packed, E, B, d, h, dW, dlogits);
  if (dx)
    mglu::dx_kernel<T, NM><<<dim3((unsigned)((d + mglu::kBwK - 1) / mglu::kBwK), (unsigned)((B + mglu::kBwB - 1) / mglu::kBwB)),
                             256, 0, st>>>((const T*)Wt, (const uint32_t*)packed, E, B, d, h, dx);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t backward_nm(mglu_ctx* hd, const void* x, int B, const void* Wt, const void* packed, const float* dy,
                               float* dx, float* dW, float* dlogits, const float* z, float* E, cudaStream_t st) {
  switch (hd->n_m) {
    case 1: return backward_kernels<T, 1>(hd, x, B, Wt, packed, dy, dx, dW, dlogits, z, E, st);
    case 2: return backward_kernels<T, 2>(hd, x, B, Wt, packed, dy, dx, dW, dlogits, z, E, st);
    case 4: return backward_kernels<T, 4>(hd, x, B, Wt, packed, dy, dx, dW, dlogits, z, E, st);
    case 8: return backward_kernels<T, 8>(hd, x, B, Wt, packed, dy, dx, dW, dlogits, z, E, st);
    default: return cudaErrorInvalidValue;
  }
}

extern "C" {

mglu_status mglu_backward(mglu_handle hd, const void* x, int64_t B, const void* Wt, const void* packed,
                                     const float* dy, float* dx, float* dW, float* dlogits, void* stream) {
  if (!hd) return MGLU_ERR_INVALID_ARG;
  if (!x || !Wt || !packed || !dy || B < 0) return set_err(hd, MGLU_ERR_INVALID_ARG, "null pointer or B < 0");
  if (!fast_nm(hd->n_m)) return set_err(hd, MGLU_ERR_UNSUPPORTED, "backward: n_m in {1, 2, 4, 8}");
  if (B > (int64_t)1 << 30) return set_err(hd, MGLU_ERR_INVALID_ARG, "B too large");
  hd->last_launches = 0;
  if (B == 0) return MGLU_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != hd->device) cudaSetDevice(hd->device);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t zf = (size_t)B * 2 * hd->n_m * hd->h, ef = (size_t)B * (hd->n_m + 1) * hd->h;
  const size_t need = (zf + ef) * sizeof(float);
  if (hd->bw_ws_bytes < need) {
    if (hd->bw_ws) { cudaStreamSynchronize(st); cudaFree(hd->bw_ws); hd->bw_ws = nullptr; hd->bw_ws_bytes = 0; }
    if (cudaMalloc(&hd->bw_ws, need) != cudaSuccess) {
      if (prev != hd->device) cudaSetDevice(prev);
      return set_err(hd, MGLU_ERR_OOM, "backward workspace");
    }
    hd->bw_ws_bytes = need;
  }
  float* z = hd->bw_ws;
  float* E = hd->bw_ws + zf;
  // the forward streams s_i, v_i from the forward kernels' partials mode (the path AUTO would take)
  int path;
  {
    std::lock_guard<std::mutex> g(hd->mu);
    path = hd->path;
  }
  if (path == MGLU_PATH_AUTO) path = auto_path(hd, B);
  Call cl;
  cl.st = st;
  cl.z = z;
  mglu_status s = forward_on_path(hd, x, B, Wt, packed, nullptr, path, cl);
  if (s != MGLU_OK) { if (prev != hd->device) cudaSetDevice(prev); return s; }
  const cudaError_t e = hd->dtype == MGLU_BF16
                            ? backward_nm<__nv_bfloat16>(hd, x, (int)B, Wt, packed, dy, dx, dW, dlogits, z, E, st)
                            : backward_nm<float>(hd, x, (int)B, Wt, packed, dy, dx, dW, dlogits, z, E, st);
  if (prev != hd->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(hd, e, "mglu_backward launch");
  hd->last_launches = 2 + (dW || dlogits ? 1 : 0) + (dx ? 1 : 0);
  return MGLU_OK;
}

mglu_status mglu_forward_host(mglu_handle hd, const void* x_host, int64_t B, const void* Wt,
                              const void* packed, void* out_host, void* stream) {
  if (!hd) return MGLU_ERR_INVALID_ARG;
  if (B < 0 || !x_host || !out_host || !Wt || (!packed && hd->n_m))
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
  void* xin = mapped_alias(x_host);
  void* yout = mapped_alias(out_host);
  if (xin && aligned16(xin))
    e = launch_pdl(stage_in_kernel, dim3(stage_grid((int64_t)xb)), dim3(256), 0, st, (const uint8_t*)xin,
                   (uint8_t*)hd->x_stage, (int64_t)xb);
  else
    e = cudaMemcpyAsync(hd->x_stage, x_host, xb, cudaMemcpyHostToDevice, st);
  if (prev != hd->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(hd, e, "H2D x");
  mglu_status s = mglu_forward(hd, hd->x_stage, B, Wt, packed, hd->y_stage, stream);
  if (s != MGLU_OK) return s;
  cudaSetDevice(hd->device);
  if (yout && aligned16(yout))
    e = launch_pdl(stage_out_kernel, dim3(stage_grid((int64_t)yb)), dim3(256), 0, st, (const uint8_t*)hd->y_stage,
                   (uint8_t*)yout, (int64_t)yb);
  else
    e = cudaMemcpyAsync(out_host, hd->y_stage, yb, cudaMemcpyDeviceToHost, st);
  if (prev != hd->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(hd, e, "D2H y");
  return MGLU_OK;
}

// ------------------------------------------------------------------ packing
// Layout (reading R3, include/mglu.h): row j, 32-column group g, mask i -> little-endian u32 word
// (j*(d/32) + g)*n_m + i; column 32g + e at bit (e >> 1) + 16*(e & 1).
mglu_status mglu_pack_masks_host(const uint8_t* bits, int n_m, int64_t h, int64_t d, uint8_t* packed) {
  if (!bits || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m) || d % 32) return MGLU_ERR_UNSUPPORTED;
  const int64_t hd = h * d;
  for (int64_t q = 0; q < (int64_t)n_m * hd; ++q)
    if (bits[q] > 1) return MGLU_ERR_INVALID_ARG;
  pack_words(n_m, h, d, packed, [&](int i, int64_t j, int64_t k) { return (uint32_t)bits[i * hd + j * d + k]; });
  return MGLU_OK;
}

mglu_status mglu_pack_logits_host(const float* logits, int n_m, int64_t h, int64_t d, uint8_t* packed) {
  if (!logits || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m) || d % 32) return MGLU_ERR_UNSUPPORTED;
  const int64_t hd = h * d;
  pack_words(n_m, h, d, packed, [&](int i, int64_t j, int64_t k) {
    return logits[i * hd + j * d + k] > 0.0f ? 1u : 0u;      // strict (R4)
  });
  return MGLU_OK;
}

mglu_status mglu_unpack_masks_host(const uint8_t* packed, int n_m, int64_t h, int64_t d, uint8_t* bits) {
  if (!bits || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m) || d % 32) return MGLU_ERR_UNSUPPORTED;
  const int64_t hd = h * d, groups = d / 32;
  for (int64_t j = 0; j < h; ++j)
    for (int64_t k = 0; k < d; ++k)
      for (int i = 0; i < n_m; ++i) {
        const uint32_t w = get_le32(packed + ((j * groups + k / 32) * n_m + i) * 4);
        bits[i * hd + j * d + k] = (uint8_t)((w >> mglu::code_bit_of((int)(k % 32))) & 1u);
      }
  return MGLU_OK;
}

// ------------------------------------------------------------------ per-element code streams
static bool valid_code_width(int w, int n_m) {
  return (w == 1 || w == 2 || w == 4 || w == 8 || w == 16) && n_m >= 1 && n_m <= w && valid_nm(n_m);
}
// field (element e) of a w-bit little-endian stream; w divides 8 or is 16, so a field never
// straddles a byte boundary except for w = 16 (two whole bytes)
static uint32_t code_field(const uint8_t* c, int w, int64_t e) {
  if (w == 16) return (uint32_t)c[2 * e] | ((uint32_t)c[2 * e + 1] << 8);
  const int64_t bit = e * w;
  return (c[bit >> 3] >> (bit & 7)) & ((1u << w) - 1u);
}

size_t mglu_code_stream_bytes(int64_t d, int64_t h, int w) {
  if (d < 0 || h < 0 || !(w == 1 || w == 2 || w == 4 || w == 8 || w == 16)) return 0;
  return (size_t)((h * d * w + 7) / 8);
}

mglu_status mglu_codes_to_bits_host(const uint8_t* codes, int w, int n_m, int64_t h, int64_t d, uint8_t* bits) {
  if (!codes || !bits || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_code_width(w, n_m)) return MGLU_ERR_UNSUPPORTED;
  const int64_t hd = h * d;
  for (int64_t e = 0; e < hd; ++e)
    if (code_field(codes, w, e) >> n_m) return MGLU_ERR_INVALID_ARG;      // high-bit contamination
  for (int64_t e = 0; e < hd; ++e) {
    const uint32_t f = code_field(codes, w, e);
    for (int i = 0; i < n_m; ++i) bits[i * hd + e] = (uint8_t)((f >> i) & 1u);   // mask i+1 = bit i
  }
  return MGLU_OK;
}

mglu_status mglu_pack_codes_host(const uint8_t* codes, int w, int n_m, int64_t h, int64_t d, uint8_t* packed) {
  if (!codes || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_code_width(w, n_m) || d % 32) return MGLU_ERR_UNSUPPORTED;
  const int64_t hd = h * d;
  for (int64_t e = 0; e < hd; ++e)
    if (code_field(codes, w, e) >> n_m) return MGLU_ERR_INVALID_ARG;
  pack_words(n_m, h, d, packed, [&](int i, int64_t j, int64_t k) { return (code_field(codes, w, j * d + k) >> i) & 1u; });
  return MGLU_OK;
}

mglu_status mglu_unpack_codes_host(const uint8_t* packed, int n_m, int64_t h, int64_t d, int w, uint8_t* codes) {
  if (!codes || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_code_width(w, n_m) || d % 32) return MGLU_ERR_UNSUPPORTED;
  const int64_t groups = d / 32;
  memset(codes, 0, mglu_code_stream_bytes(d, h, w));
  for (int64_t j = 0; j < h; ++j)
    for (int64_t k = 0; k < d; ++k) {
      uint32_t f = 0;
      for (int i = 0; i < n_m; ++i)
        f |= ((get_le32(packed + ((j * groups + k / 32) * n_m + i) * 4) >> mglu::code_bit_of((int)(k % 32))) & 1u) << i;
      const int64_t e = j * d + k;
      if (w == 16) { codes[2 * e] = (uint8_t)f; codes[2 * e + 1] = (uint8_t)(f >> 8); }
      else codes[(e * w) >> 3] |= (uint8_t)(f << ((e * w) & 7));
    }
  return MGLU_OK;
}

mglu_status mglu_pack_planes_host(const uint8_t* packed, int n_m, int64_t h, int64_t d, uint8_t* planes) {
  if (!packed || !planes || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m) || d % 32) return MGLU_ERR_UNSUPPORTED;
  const int64_t G = d / 32;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(packed);
  uint32_t* dst = reinterpret_cast<uint32_t*>(planes);
  for (int64_t j = 0; j < h; ++j)
    for (int64_t g = 0; g < G; ++g)
      for (int i = 0; i < n_m; ++i) dst[((int64_t)i * h + j) * G + g] = src[(j * G + g) * n_m + i];
  return MGLU_OK;
}

mglu_status mglu_pack_planes_device(const uint8_t* packed, int n_m, int64_t h, int64_t d, uint8_t* planes, void* stream) {
  if (!packed || !planes || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m) || d % 32) return MGLU_ERR_UNSUPPORTED;
  if (!aligned16(packed) || !aligned16(planes)) return MGLU_ERR_MISALIGNED;
  const int64_t n = h * (d / 32) * n_m;
  if (n == 0) return MGLU_OK;
  mglu::planes_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const uint32_t*>(packed), n_m, h, d / 32, reinterpret_cast<uint32_t*>(planes));
  return device_launch_check(cudaGetLastError());
}

mglu_status mglu_pack_masks_device(const uint8_t* bits, int n_m, int64_t h, int64_t d, uint8_t* packed,
                                   void* stream) {
  if (!bits || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m) || d % 32) return MGLU_ERR_UNSUPPORTED;
  if (!aligned16(packed)) return MGLU_ERR_MISALIGNED;
  const int64_t nwords = h * (d / 32) * n_m;
  if (nwords == 0) return MGLU_OK;
  mglu::pack_kernel<uint8_t><<<grid_for(nwords), 256, 0, (cudaStream_t)stream>>>(bits, n_m, h, d, (uint32_t*)packed);
  return device_launch_check(cudaGetLastError());
}

mglu_status mglu_pack_logits_device(const float* logits, int n_m, int64_t h, int64_t d, uint8_t* packed,
                                    void* stream) {
  if (!logits || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m) || d % 32) return MGLU_ERR_UNSUPPORTED;
  if (!aligned16(packed)) return MGLU_ERR_MISALIGNED;
  const int64_t nwords = h * (d / 32) * n_m;
  if (nwords == 0) return MGLU_OK;
  mglu::pack_kernel<float><<<grid_for(nwords), 256, 0, (cudaStream_t)stream>>>(logits, n_m, h, d, (uint32_t*)packed);
  return device_launch_check(cudaGetLastError());
}

mglu_status mglu_unpack_masks_device(const uint8_t* packed, int n_m, int64_t h, int64_t d, uint8_t* bits,
                                     void* stream) {
  if (!bits || !packed || h < 0 || d < 0) return MGLU_ERR_INVALID_ARG;
  if (!valid_nm(n_m) || d % 32) return MGLU_ERR_UNSUPPORTED;
  if (!aligned16(packed)) return MGLU_ERR_MISALIGNED;
  const int64_t hd = h * d;
  if (hd == 0) return MGLU_OK;
  mglu::unpack_kernel<<<grid_for(hd), 256, 0, (cudaStream_t)stream>>>((const uint32_t*)packed, n_m, h, d, bits);
  return device_launch_check(cudaGetLastError());
}

}  // extern "C"
