// gemm_tc.cuh -- tcgen05/TMEM masked GEMM (prefill / large-B regime).  Placeholder until the
// kernel lands: tc_can_serve() is false, so AUTO never selects it and a forced
// MGLU_PATH_TCGEN05 returns MGLU_ERR_UNSUPPORTED.
#pragma once
#include "common.cuh"

namespace mglu {

struct TcState {};

inline bool tc_can_serve(int64_t, int64_t, int, int64_t) { return false; }
inline void tc_release(TcState&) {}
inline cudaError_t tc_forward(TcState&, int64_t, int64_t, int, int, const void*, int64_t, const void*,
                              const void*, void*, cudaStream_t, int* launches) {
  *launches = 0;
  return cudaErrorNotSupported;
}

}  // namespace mglu
