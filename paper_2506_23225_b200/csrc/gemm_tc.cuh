// gemm_tc.cuh -- tcgen05/TMEM masked GEMM: the prefill / large-batch regime.
//
// The paper's kernel is batch 1 only; for B tokens Eq. 3 needs (n_m + 1) GEMMs sharing x:
// t = X Wt^T and, per mask, a masked product.  As in the decode regime the masked operand is the
// sign-flipped weight sigma_i (.) W (sigma = +1 where M_i = 1, -1 where M_i = 0), so the tensor core
// accumulates u_i = s_i - v_i and the epilogue takes s_i = (t + u_i) / 2 (exact rescaling).
//
// One CTA computes a 128-row (h) x BN-token tile over the whole reduction (d), in stages of 64
// reduction columns:
//   * TMA (warp 8) stages x [BN x 64], W [128 x 64] (both K-major, 128-byte swizzle) and the
//     tile rows' mask words into a shared-memory ring -- 128-byte requests, deep prefetch.
//   * The masker (warps 0-7, two groups of 128 threads; thread = tile row = TMEM lane) reads its
//     row's W and mask words from shared memory, builds the n_m sign-flipped rows in registers
//     (one IMAD + one LOP3 per bf16 pair and mask) and tcgen05.st's the n_m + 1 operands
//     {W, sigma_i (.) W} into a TMEM A slot (TS form: the tensor core reads A from TMEM, so the
//     masked operands never touch shared memory).  Group g fills the A-stages js = g (mod 2).
//   * The MMA warp (warp 9, warp-uniform, one elected lane issues) runs n_m + 1 kind::f16 MMAs per
//     k16 step into n_m + 1 fp32 TMEM accumulators of BN columns: (n_m + 1) * BN + A slots <= 512.
//   * Epilogue (warps 0-7): tcgen05.ld of the accumulators, Eq. 3 in registers, bf16 stores.
#pragma once
#include "common.cuh"
#include "mma_mask.cuh"
#include "tcgen05.cuh"
#include "tma.cuh"

namespace mglu {

// tile shape per mask count: BN tokens; 2 TMEM A slots of KA reduction columns per operand; MPC
// masks per CTA.  n_m = 8 would leave BN = 32 (nine accumulators): instead a cluster of two CTAs
// splits the masks 4 + 4 (each also forms t), and the pair sums its partial outputs over DSMEM.
template <int NM> struct TcCfg;
template <> struct TcCfg<1> { static constexpr int BN = 224, KA = 32, MPC = 1; };
template <> struct TcCfg<2> { static constexpr int BN = 128, KA = 32, MPC = 2; };

#ifndef MGLU_TC_ODD_SLOTS
#define MGLU_TC_ODD_SLOTS 0
#endif
// n_m = 4 (and each CTA of the n_m = 8 pair): 80-token tiles with 16-column A-stages -- five
// accumulators of 80 columns leave two 40-column A slots; the tensor work per masked operand is 25 %
// larger than at 64 tokens with 32-column stages (2 slots of 80): config 4 8.12 vs 9.07 ms
// (profiles/r02/prefill_tiles.txt)
#ifndef MGLU_TC_BN4
#define MGLU_TC_BN4 80
#endif
template <> struct TcCfg<4> { static constexpr int BN = MGLU_TC_BN4, KA = 32, MPC = 4; };
template <> struct TcCfg<8> { static constexpr int BN = MGLU_TC_BN4, KA = 32, MPC = 4; };
// n_m = 16: a cluster of four CTAs, four masks each; 32-token tiles keep
// the three partner buffers of the DSMEM reduction beside a 4-stage ring
template <> struct TcCfg<16> { static constexpr int BN = 32, KA = 32, MPC = 4; };

constexpr int kTcThreads = 320;
constexpr int kTcMaskWarps = 8;
constexpr int kTcK = 64;                        // reduction columns per shared stage
// TMEM A slots: 4 when the accumulators leave room (small token tiles: deeper masker run-ahead
// hides the slot round trip), else 2 -- always even, so every slot belongs to one masker group
#ifndef MGLU_TC_SS_T
#define MGLU_TC_SS_T 0   // 1: t's MMA reads W straight from shared memory (SS); slots hold the masked copies only
#endif
template <int NM> __host__ __device__ constexpr int tc_slot_ops() { return TcCfg<NM>::MPC + (MGLU_TC_SS_T ? 0 : 1); }
// A-stage width of a BN-token tile: 32 columns when two such slots fit beside the accumulators, else 16
template <int NM, int BN> __host__ __device__ constexpr int tc_ka() {
  return (TcCfg<NM>::MPC + 1) * BN + 2 * tc_slot_ops<NM>() * TcCfg<NM>::KA / 2 <= 512 ? TcCfg<NM>::KA : 16;
}
template <int NM, int BN> __host__ __device__ constexpr int tc_slots() {
  constexpr int acc = (TcCfg<NM>::MPC + 1) * BN, slot = tc_slot_ops<NM>() * tc_ka<NM, BN>() / 2;
  constexpr int fit = (512 - acc) / slot;
  return fit >= 4 ? 4 : (MGLU_TC_ODD_SLOTS && fit == 3) ? 3 : 2;
}

// mask words per row per stage as loaded by TMA: 2 groups x n_m words, at least 16 bytes
template <int NM> __host__ __device__ constexpr int tc_code_words() { return 2 * NM < 4 ? 4 : 2 * NM; }
// BN = token tile: TcCfg<NM>::BN for prefill, 16 / 32 / 64 for small batches (decode regime)
template <int BN> __host__ __device__ constexpr int tc_x_bytes() { return BN * kTcK * 2; }
template <int NM, int BN> __host__ __device__ constexpr int tc_stage_bytes() {
  return tc_x_bytes<BN>() + 128 * kTcK * 2 + 128 * tc_code_words<NM>() * 4;
}
template <int NM> __host__ __device__ constexpr int tc_split() { return NM / TcCfg<NM>::MPC; }
// DSMEM buffers of the mask-split reduction on cluster rank 0: each partner's fp32 partial outputs [BN][128]
template <int NM, int BN> __host__ __device__ constexpr int tc_red_bytes() { return (tc_split<NM>() - 1) * BN * 128 * 4; }
template <int NM> __host__ __device__ constexpr int tc_tmem_used() {
  return (TcCfg<NM>::MPC + 1) * TcCfg<NM>::BN + 2 * (TcCfg<NM>::MPC + 1) * tc_ka<NM, TcCfg<NM>::BN>() / 2;
}
static_assert(tc_tmem_used<1>() <= 512 && tc_tmem_used<2>() <= 512 && tc_tmem_used<4>() <= 512 &&
              tc_tmem_used<8>() <= 512 && tc_tmem_used<16>() <= 512, "TMEM budget");

struct TcParams {
  __nv_bfloat16* out;        // [B][h]
  const float* G;            // Top-K routed gate weights [B][n_m] (nullptr: every weight 1)
  int variant;               // partial-mask ablation variant (0 = Eq. 3)
  int act;                   // g when the kernel is the kRuntimeAct instantiation
  int B, d, h;
  int stages;
  float* z;                  // non-null: write Alg. 1's z [B][2 n_m][h] (s_i, t - s_i) instead of y
};

template <int NM, int ACT, int BN>
__global__ void __launch_bounds__(kTcThreads, 1)
gemm_tc_kernel(const TcParams p, const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mW,
               const __grid_constant__ CUtensorMap mC) {
  constexpr int KA = tc_ka<NM, BN>(), SA = tc_slots<NM, BN>();
  constexpr int NSL = tc_slot_ops<NM>();                  // operands stored per A slot
  constexpr int SS = MGLU_TC_SS_T;                         // t from shared memory
  static_assert((TcCfg<NM>::MPC + 1) * BN + SA * NSL * KA / 2 <= 512, "TMEM budget");
  constexpr int MPC = TcCfg<NM>::MPC, NSPLIT = tc_split<NM>();
  constexpr int NOP = MPC + 1;                             // operands: W and this CTA's sign-flipped copies
  constexpr int XB = tc_x_bytes<BN>(), WB = 128 * kTcK * 2, CW = tc_code_words<NM>();
  constexpr int SB = tc_stage_bytes<NM, BN>();
  constexpr int KPS = KA / 16;                             // k16 steps per A-stage
  constexpr int APS = kTcK / KA;                           // A-stages per shared stage (2 or 4)
  constexpr int WW = KA / 2;                               // bf16 pairs per row and A-stage
  constexpr uint32_t IDESC = idesc_bf16_f32(128, BN);
  constexpr uint32_t A_COL0 = NOP * BN;                    // first TMEM column of the A slots
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = p.stages;
  float* red = reinterpret_cast<float*>(smem + (size_t)S * SB);           // mask-split partials (rank 0)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * SB + tc_red_bytes<NM, BN>());
  uint64_t* empty = full + S;
  uint64_t* a_full = empty + S;
  uint64_t* a_empty = a_full + SA;
  uint64_t* acc_full = a_empty + SA;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);   // provably warp-uniform
  const int lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * 128;
  const int moff = (int)blockIdx.z * MPC;                  // first mask of this CTA (cluster rank z)
  const int d = p.d;
  const int nk16 = d >> 4;                                 // d % 32 == 0
  const int nks = (d + kTcK - 1) / kTcK;                   // shared stages
  const int nas = d / KA;                                  // A-stages

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + 32 * kTcMaskWarps);         // MMA commit + every masker thread
    }
    for (int s = 0; s < SA; ++s) { mbar_init(&a_full[s], 128); mbar_init(&a_empty[s], 1); }
    mbar_init(acc_full, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if constexpr (NSPLIT > 1) {
    // the pair CTA writes partials into this CTA's shared memory (DSMEM): both must have started
    // (a distributed-shared-memory access needs its target CTA running -- compute-sanitizer racecheck)
    cluster_arrive();
    cluster_wait();
  }

  constexpr int HALF = BN / 2;                             // epilogue tokens per masker group
  float yp[HALF / 8][8];                                   // this thread's partial outputs
  if (warp == kTcMaskWarps) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      prefetch_tmap(&mX);
      prefetch_tmap(&mW);
      prefetch_tmap(&mC);
      pdl_wait();                                          // x may come from the predecessor
      int s = 0;
      uint32_t ph = 0;
      for (int ks = 0; ks < nks; ++ks) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + (size_t)s * SB;
        mbar_arrive_expect_tx(&full[s], (uint32_t)SB);
        tma_load_2d(st, &mX, ks * kTcK, n0, &full[s]);
        tma_load_2d(st + XB, &mW, ks * kTcK, m0, &full[s]);
        tma_load_2d(st + XB + WB, &mC, (ks * 2 * NM) / CW * CW, m0, &full[s]);   // box never straddles the row end
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == kTcMaskWarps + 1) {
    // ---------------------------------------------------------------- MMA issuer (whole warp)
    const uint64_t bdesc0 = smem_desc_kmajor(smem_u32(smem), 128);
    int s = 0;
    uint32_t ph = 0;
    for (int ks = 0; ks < nks; ++ks) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint64_t bdesc_s = bdesc0 + (uint64_t)((s * SB) >> 4);
#pragma unroll
      for (int kk = 0; kk < kTcK / 16; ++kk) {
        const int j = ks * (kTcK / 16) + kk;               // k16 step
        if (j < nk16) {
          const int js = j / KPS;                          // A-stage
          const int sa = js % SA;
          if (kk % KPS == 0) {
            mbar_wait(&a_full[sa], (uint32_t)(js / SA) & 1u);
            tc_fence_after();
          }
          if (elect_one()) {
            const uint64_t bdesc = bdesc_s + (uint64_t)(kk * 2);          // +32 bytes along K
            const uint32_t a0 = tmem + A_COL0 + (uint32_t)(sa * NSL * WW + (kk % KPS) * 8);
            const uint32_t acc = j > 0 ? 1u : 0u;
            if constexpr (SS) {
              const uint64_t adesc = smem_desc_kmajor(smem_u32(smem) + XB, 128) + (uint64_t)((s * SB) >> 4) + (uint64_t)(kk * 2);
              tc_mma_ss(tmem, adesc, bdesc, IDESC, acc);                                 // t: W from smem
            }
#pragma unroll
            for (int op = SS; op < NOP; ++op) tc_mma_ts(tmem + op * BN, a0 + (op - SS) * WW, bdesc, IDESC, acc);
            if (kk % KPS == KPS - 1) tc_commit(&a_empty[sa]);
          }
          __syncwarp();
        }
      }
      if (elect_one()) tc_commit(&empty[s]);               // x no longer needed
      __syncwarp();
      if (++s == S) { s = 0; ph ^= 1; }
    }
    if (elect_one()) tc_commit(acc_full);
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- masker
    const int g = warp >> 2;                               // A-stages js = g (mod 2)
    const int m = (warp & 3) * 32 + lane;                  // tile row = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t a_lane = tmem + lane_off + A_COL0;
    const uint32_t wrow_off = (uint32_t)(XB + m * 128);    // row m of the W tile (128-byte rows)
    int s = 0;
    uint32_t ph = 0;
    int js = 0;
    for (int ks = 0; ks < nks; ++ks) {
      mbar_wait(&full[s], ph);
      const uint8_t* st = smem + (size_t)s * SB;
#pragma unroll
      for (int a = 0; a < APS; ++a, ++js) {
        if ((a & 1) != g || js >= nas) continue;
        // this A-stage's W: KA columns = KA/8 16-byte chunks of the 128-byte row (SW128 layout)
        uint32_t w[WW];
#pragma unroll
        for (int c = 0; c < KA / 8; ++c) {
          const uint32_t chunk = (uint32_t)(a * (KA / 8) + c) ^ (uint32_t)(m & 7);
          const uint4 v = *reinterpret_cast<const uint4*>(st + wrow_off + chunk * 16);
          w[4 * c] = v.x; w[4 * c + 1] = v.y; w[4 * c + 2] = v.z; w[4 * c + 3] = v.w;
        }
        uint32_t cw[MPC];
        const int grp = (a * KA) >> 5;                     // code group within the stage
        const int wofs = (ks * 2 * NM) % CW;               // stage's first word within the loaded box
        // the code box is swizzled like its row width (bank-conflict-free 16-byte reads)
        lds_words_swz<MPC>(st + XB + WB, (uint32_t)(m * CW * 4 + (wofs + grp * NM + moff) * 4), CW * 4, cw);
        const int pair0 = (a * KA) & 31 ? 8 : 0;           // first pair of the A-stage in its group
        uint32_t op[NOP][WW];
#pragma unroll
        for (int q = 0; q < WW; ++q) op[0][q] = w[q];
#pragma unroll
        for (int i = 0; i < MPC; ++i) {
#pragma unroll
          for (int q = 0; q < WW; ++q)                     // pair pair0 + q: bits (pair, pair + 16)
            op[1 + i][q] = sign_flip(w[q], cw[i], 1u << (15 - pair0 - q));
        }
        const int sa = js % SA;
        mbar_wait(&a_empty[sa], ((uint32_t)(js / SA) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t a0 = a_lane + (uint32_t)(sa * NSL * WW);
#pragma unroll
        for (int o = SS; o < NOP; ++o) {
          if constexpr (WW == 16) tmem_st16(a0 + (o - SS) * WW, op[o]);
          else tmem_st8(a0 + (o - SS) * WW, *reinterpret_cast<uint32_t(*)[8]>(&op[o][0]));
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&a_full[sa]);
      }
      mbar_arrive(&empty[s]);                              // W / code rows of this stage consumed
      if (++s == S) { s = 0; ph ^= 1; }
    }

    // ---------------------------------------------------------------- epilogue
    mbar_wait(acc_full, 0);
    tc_fence_after();
    pdl_wait();                                            // out may be read upstream
    const uint32_t lane_base = tmem + lane_off;
    static_assert(HALF % 8 == 0, "BN / 2 must be a multiple of 8");
#ifdef MGLU_TC_EPI_SKIP   // timing ablation (wrong results): no epilogue at all
    if (true) {
    } else
#endif
    if (p.z) {
      // partials (debug / parity of a5, a6): this CTA's masks' s_i and t - s_i, no reduction.  A
      // separate loop: a partials branch inside the y loop below cost the BN = 64 tile 2x (measured)
      for (int ch = 0; ch < HALF / 8; ++ch) {
        const int c0 = g * HALF + ch * 8;
        uint32_t tv[8], uv[8];
        tmem_ld8(lane_base + c0, tv);
        for (int i = 0; i < MPC; ++i) {
          tmem_ld8(lane_base + (1 + i) * BN + c0, uv);
          tmem_ld_wait();
          for (int q = 0; q < 8; ++q) {
            const int tq = n0 + c0 + q;
            const float t = __uint_as_float(tv[q]), sg = 0.5f * (t + __uint_as_float(uv[q]));
            if (tq < p.B && m0 + m < p.h) {
              float* zt = p.z + (size_t)tq * 2 * NM * p.h + m0 + m;
              zt[(size_t)(moff + i) * p.h] = sg;
              zt[(size_t)(NM + moff + i) * p.h] = t - sg;
            }
          }
        }
      }
    } else
#pragma unroll
    for (int ch = 0; ch < HALF / 8; ++ch) {
      const int c0 = g * HALF + ch * 8;
      uint32_t tv[8], uv[MPC][8];
      tmem_ld8(lane_base + c0, tv);
#pragma unroll
      for (int i = 0; i < MPC; ++i) tmem_ld8(lane_base + (1 + i) * BN + c0, uv[i]);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float t = __uint_as_float(tv[q]);
        const int tq = n0 + c0 + q;                        // token of this column
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < MPC; ++i) {
          const float sg = 0.5f * (t + __uint_as_float(uv[i][q]));       // s_i = (t + u_i) / 2
          const float gate = (p.variant & 1) ? t : sg;                    // ablation variants
          const float value = (p.variant & 2) ? t : t - sg;
          const float wgt = p.G ? (tq < p.B ? p.G[(size_t)tq * NM + moff + i] : 0.f) : 1.f;   // routed (App. B)
#ifdef MGLU_TC_EPI_ABL   // timing ablation (wrong results): no activation in the epilogue
          acc = fmaf(wgt * gate, value, acc);
#else
          acc = fmaf(wgt * act_fast<ACT>(gate, p.act), value, acc);              // g(s_i) (t - s_i)
#endif
        }
        yp[ch][q] = acc;
      }
      if constexpr (NSPLIT > 1) {
        if (blockIdx.z > 0) {                              // partial of this rank's masks -> rank 0's buffer
          float* rb = red + (size_t)(blockIdx.z - 1) * BN * 128;
#pragma unroll
          for (int q = 0; q < 8; ++q) st_cluster_f32(rb + (c0 + q) * 128 + m, 0, yp[ch][q]);
        }
      } else {
        const int grow = m0 + m;
#ifdef MGLU_TC_EPI_NOSTORE   // timing ablation (wrong results): the epilogue without its global stores
        if (grow < 0) {
#elif defined(MGLU_TC_EPI_MATHONLY)   // timing ablation: the math kept (consumed), stores almost never
        if (yp[ch][0] + yp[ch][1] + yp[ch][2] + yp[ch][3] + yp[ch][4] + yp[ch][5] + yp[ch][6] + yp[ch][7] == 1234.5f) {
#else
        if (grow < p.h) {
#endif
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int tok = n0 + c0 + q;
            if (tok < p.B) p.out[(size_t)tok * p.h + grow] = __float2bfloat16_rn(yp[ch][q]);
          }
        }
      }
    }
  }
  if constexpr (NSPLIT > 1) {
    cluster_arrive();                                      // partials delivered (release / acquire)
    cluster_wait();
  }
  if (NSPLIT > 1 && warp < kTcMaskWarps && blockIdx.z == 0 && !p.z) {
    const int g = warp >> 2;
    const int m = (warp & 3) * 32 + lane;
    const int grow = m0 + m;
    if (grow < p.h) {
#pragma unroll
      for (int ch = 0; ch < HALF / 8; ++ch) {
        const int c0 = g * HALF + ch * 8;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int tok = n0 + c0 + q;
          float y = yp[ch][q];
#pragma unroll
          for (int r = 1; r < NSPLIT; ++r) y += red[(size_t)(r - 1) * BN * 128 + (c0 + q) * 128 + m];   // rank order
          if (tok < p.B) p.out[(size_t)tok * p.h + grow] = __float2bfloat16_rn(y);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  pdl_launch_dependents();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace mglu
