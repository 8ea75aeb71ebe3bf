// gemm_tc.cuh -- tcgen05/TMEM masked GEMM: the prefill / large-batch regime (a8).  MGLU_PATH_TCGEN05.
//
// The paper's kernel is batch 1 only; for B tokens Eq. 3 needs (n_m + 1) GEMMs that share
// x: t = X Wt^T and, per mask, the gated product.  As in the decode regime the masked operand is
// the sign-flipped weight sigma_i (.) W (sigma = +1 on the gate side, -1 on the value side), so
// the tensor core accumulates u_i = s_i - v_i and the epilogue uses s_i = (t + u_i) / 2.
//
// One CTA computes a 128-row (h) x BN-token tile.  Warp roles (192 threads):
//   warp 4   TMA producer: W tile [128 x BK] and x tile [BN x BK] (K-major, swizzled) per stage;
//   warps 0-3 masker: thread m reads its row of the W tile, builds the n_m sign-flipped rows from
//            the row's mask words (one IMAD + one LOP3 per bf16 pair and mask) and stores them in
//            the same swizzled K-major layout (the masked operands live in shared memory);
//   warp 5   MMA issuer (one thread): per k16 step, (n_m + 1) tcgen05.mma kind::f16 into
//            (n_m + 1) TMEM accumulators of BN fp32 columns each; tcgen05.commit frees the stage;
//   warps 0-3 epilogue: tcgen05.ld of row m's accumulators (TMEM lane m), Eq. 3 on registers,
//            bf16 stores y[token][row] (32 consecutive rows per warp store = coalesced).
// TMEM: (n_m + 1) * BN <= 512 columns fixes BN = 256 / 128 / 64 / 32 for n_m = 1 / 2 / 4 / 8.
#pragma once
#include "common.cuh"
#include "mma_mask.cuh"
#include "tcgen05.cuh"
#include "tma.cuh"

namespace mglu {

template <int NM> __host__ __device__ constexpr int tc_bn() { return NM == 1 ? 256 : NM == 2 ? 128 : NM == 4 ? 64 : 32; }
template <int NM> __host__ __device__ constexpr int tc_bk() { return NM == 8 ? 32 : 64; }
template <int NM> __host__ __device__ constexpr int tc_tmem_cols() {
  return (NM + 1) * tc_bn<NM>() <= 256 ? 256 : 512;
}
template <int NM> __host__ __device__ constexpr int tc_stage_bytes() {
  // W tile + x tile + n_m masked tiles, all [rows][BK] bf16
  return 128 * tc_bk<NM>() * 2 + tc_bn<NM>() * tc_bk<NM>() * 2 + NM * 128 * tc_bk<NM>() * 2;
}
constexpr int kTcThreads = 192;

struct TcParams {
  const uint32_t* codes;     // packed mask words (R3 layout)
  __nv_bfloat16* out;        // [B][h]
  int B, d, h;
  int stages;
};

template <int NM, int ACT>
__global__ void __launch_bounds__(kTcThreads, 1)
gemm_tc_kernel(const TcParams p, const __grid_constant__ CUtensorMap mW, const __grid_constant__ CUtensorMap mX) {
  constexpr int BN = tc_bn<NM>(), BK = tc_bk<NM>();
  constexpr int SPAN = BK * 2;                         // bytes per tile row (= swizzle span)
  constexpr int WT = 128 * SPAN, XT = BN * SPAN;       // tile bytes
  constexpr int SB = tc_stage_bytes<NM>();
  constexpr int GPK = BK / 32;                         // 32-column mask groups per k-block
  constexpr uint32_t IDESC = idesc_bf16_f32(128, BN);
  constexpr int TMEM_COLS = tc_tmem_cols<NM>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // swizzle atoms (and the descriptors' base offset 0) need 1024-byte aligned tiles
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = p.stages;
  uint8_t* ring = smem;                                // per stage: W | x | masked[NM]
  uint64_t* tma_full = reinterpret_cast<uint64_t*>(smem + (size_t)S * SB);
  uint64_t* mask_full = tma_full + S;
  uint64_t* empty = mask_full + S;
  uint64_t* acc_full = empty + S;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * 128;
  const int d = p.d;
  const int nkb = (d + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&tma_full[s], 1);
      mbar_init(&mask_full[s], 128);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(tmem_base_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_slot;

  if (warp == 4) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      prefetch_tmap(&mW);
      prefetch_tmap(&mX);
      pdl_wait();                                                  // x may come from the predecessor
      int s = 0;
      uint32_t ph = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = ring + (size_t)s * SB;
        mbar_arrive_expect_tx(&tma_full[s], (uint32_t)(WT + XT));
        tma_load_2d(st, &mW, kb * BK, m0, &tma_full[s]);
        tma_load_2d(st + WT, &mX, kb * BK, n0, &tma_full[s]);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 5) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&mask_full[s], ph);
        tc_fence_after();
        const uint32_t base = smem_u32(ring + (size_t)s * SB);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint32_t koff = kk * 32;                           // 16 bf16 along K
          const uint64_t bdesc = smem_desc_kmajor(base + WT + koff, SPAN);
          const uint32_t acc = (kb | kk) ? 1u : 0u;
          tc_mma_ss(tmem, smem_desc_kmajor(base + koff, SPAN), bdesc, IDESC, acc);      // t
#pragma unroll
          for (int i = 0; i < NM; ++i)                                                  // u_i
            tc_mma_ss(tmem + (1 + i) * BN, smem_desc_kmajor(base + WT + XT + i * WT + koff, SPAN), bdesc,
                      IDESC, acc);
        }
        tc_commit(&empty[s]);                                      // frees the stage when done
        if (++s == S) { s = 0; ph ^= 1; }
      }
      tc_commit(acc_full);
    }
  } else {
    // ---------------------------------------------------------------- masker (then epilogue)
    const int m = threadIdx.x;                                     // tile row 0..127
    const int grow = m0 + m;
    const int mrow = grow < p.h ? grow : p.h - 1;                  // rows past h: any valid row
    const uint32_t* crow = p.codes + (size_t)mrow * (d / 32) * NM;
    const uint32_t row_off = (uint32_t)((m >> 3) * (8 * SPAN) + (m & 7) * SPAN);
    uint32_t cw[GPK * NM], cn[GPK * NM];
#pragma unroll
    for (int q = 0; q < GPK * NM; ++q) cn[q] = ((q / NM) * 32 < d) ? ld_nc_u32(crow + q) : 0u;
    int s = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
#pragma unroll
      for (int q = 0; q < GPK * NM; ++q) cw[q] = cn[q];
      if (kb + 1 < nkb) {                                          // prefetch the next block's words
        const int g_next = (kb + 1) * GPK;
#pragma unroll
        for (int q = 0; q < GPK * NM; ++q)
          cn[q] = (g_next * 32 + (q / NM) * 32 < d) ? ld_nc_u32(crow + (size_t)g_next * NM + q) : 0u;
      }
      mbar_wait(&empty[s], ph ^ 1);                                // MMA done with this slot
      mbar_wait(&tma_full[s], ph);                                 // W tile landed
      uint8_t* st = ring + (size_t)s * SB;
#pragma unroll
      for (int c = 0; c < BK / 8; ++c) {                           // 16-byte chunks of the row
        // TMA / UMMA swizzle: 16-byte chunk bits [4, 4+log2(SPAN/16)) ^= address bits [7, ...)
        const uint32_t lin = row_off + (uint32_t)c * 16;
        const uint32_t off = lin ^ (((lin >> 7) & (uint32_t)(SPAN / 16 - 1)) << 4);
        const uint4 w = *reinterpret_cast<const uint4*>(st + off);
        const int g = c >> 2, qb = 4 * (c & 3);                    // group, first pair's bit
#pragma unroll
        for (int i = 0; i < NM; ++i) {
          const uint32_t word = cw[g * NM + i];
          uint4 o;
          o.x = sign_flip(w.x, word, 1u << (15 - qb));
          o.y = sign_flip(w.y, word, 1u << (14 - qb));
          o.z = sign_flip(w.z, word, 1u << (13 - qb));
          o.w = sign_flip(w.w, word, 1u << (12 - qb));
          *reinterpret_cast<uint4*>(st + WT + XT + i * WT + off) = o;
        }
      }
      fence_async_smem();
      mbar_arrive(&mask_full[s]);
      if (++s == S) { s = 0; ph ^= 1; }
    }

    // ---------------------------------------------------------------- epilogue
    mbar_wait(acc_full, 0);
    tc_fence_after();
    pdl_wait();                                                    // out may be read upstream
    const uint32_t lane_base = tmem + ((uint32_t)(32 * warp) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t tv[16], uv[16];
      float y[16];
      tmem_ld16(lane_base + c0, tv);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j) y[j] = 0.f;
#pragma unroll 1
      for (int i = 0; i < NM; ++i) {
        tmem_ld16(lane_base + (1 + i) * BN + c0, uv);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float t = __uint_as_float(tv[j]);
          const float sgate = 0.5f * (t + __uint_as_float(uv[j]));          // s_i = (t + u_i) / 2
          y[j] = fmaf(act_g<ACT>(sgate), t - sgate, y[j]);                 // g(s_i) (t - s_i)
        }
      }
      if (grow < p.h) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int tok = n0 + c0 + j;
          if (tok < p.B) p.out[(size_t)tok * p.h + grow] = __float2bfloat16_rn(y[j]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  pdl_launch_dependents();
  if (warp == 0) tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace mglu
