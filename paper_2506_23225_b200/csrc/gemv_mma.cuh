// gemv_mma.cuh -- TMA-fed, register-masked tensor-core fused masked GEMV (decode regime, bf16,
// 1 <= B <= 8).  MGLU_PATH_MMA.
//
// The FlashMGLU forward of Alg. 1 for small B, re-designed for sm_100a:
//  * a2: W (rows of Wt) and the packed codes stream HBM -> shared memory exactly once per call
//    (P:245).  Each CTA owns a contiguous, row-balanced range of Wt rows (no split-K across
//    CTAs, no atomics: reading R9).  Its rows are processed in rounds of up to 64 rows; a stage of
//    a round is one 3-D TMA box of W (64-column blocks x rows, 128B-swizzled) plus one box of the
//    codes, landing in a multi-stage mbarrier ring fed by one producer thread.
//  * a3/a4: 16 consumer warps.  A round of T 8-row tiles gives each tile WPT = 16 / T warps, each
//    owning 128 columns of every stage, so the last (ragged) round keeps all warps busy.  The n_m
//    masked operands are built in registers from the mask words as sign-flipped copies
//    sigma_i (.) W (one IMAD + one LOP3 per bf16 pair and mask, see sign_flip) and fed, with the
//    unmasked W, to mma.sync m16n8k16 (bf16 in, fp32 accumulate) with x as the B operand:
//    t = x W and u_i = x (sigma_i (.) W) = s_i - v_i in one pass, so
//    s_i = (t + u_i) / 2 = x (M_i (.) W) and v_i = t - s_i.  Products are exact in fp32.
//  * a5: k is reduced in each warp's MMA accumulators over the row, then across the WPT warps of
//    a tile through shared memory in a fixed order at the end of the round (deterministic);
//  * a6/a7: value_i = t - s_i and y = sum_i g(s_i) value_i (Eq. 3) run on registers and y is
//    stored once as bf16.
//
// Pair-role mapping (why one 16-byte LDS feeds one A fragment): the order of the reduction over
// k is free.  MMA row g (< 8) carries the EVEN bf16 pairs of real row pi(g) and MMA row g + 8 the
// ODD pairs of the same row; the B operand carries x's even pairs in column 2b and odd pairs in
// column 2b + 1 for token b.  Thread (g, c)'s A fragment {A[g][2c..], A[g+8][2c..], A[g][2c+8..],
// A[g+8][2c+8..]} is then the four consecutive pairs 4c..4c+3 of a 32-column step of row pi(g),
// and y(row pi(g), token b) = D[g][2b] + D[g+8][2b+1], both held by thread (g, b).  The tile row
// order pi(g) = g/2 + 4 (g mod 2) makes the swizzled 16-byte reads bank-conflict free.
//
// PDL: the producer starts streaming W/codes (constant weights) before griddepcontrol.wait; x and
// out are touched only after it.
#pragma once
#include "common.cuh"
#include "mma_mask.cuh"
#include "tma.cuh"

namespace mglu {

#ifndef MGLU_DEC_CONSUMERS
#define MGLU_DEC_CONSUMERS 16
#endif
constexpr int kDecConsumers = MGLU_DEC_CONSUMERS;      // consumer warps (4 per SM sub-partition)
constexpr int kDecThreads = (kDecConsumers + 1) * 32;  // + 1 producer warp
constexpr int kDecFullTiles = kDecConsumers / 2;       // 8-row tiles of a full round (2 warps each)
constexpr int kDecFullRows = 8 * kDecFullTiles;        // 64
constexpr int kDecWBytes = kDecConsumers * 2048;       // W region of a stage slot (max over rounds)

// mask bytes of one 128-column block of a row: 4 groups x n_m words (TMA box inner span = swizzle span)
template <int NM> __host__ __device__ constexpr int dec_code_span() { return 16 * NM; }   // 0: dense (n_m = 0)
// stage slot = W region + codes region (rows x WPT blocks x 16 NM bytes <= 128 * consumers * NM)
template <int NM> __host__ __device__ constexpr int dec_stage_bytes() { return kDecWBytes + 128 * kDecConsumers * NM; }

// round geometry: T tiles of 8 rows, WPT warps per tile, stage width 128 * WPT columns
__host__ __device__ constexpr int dec_wpt(int tiles) { return kDecConsumers / tiles; }

struct DecParams {
  const __nv_bfloat16* x;
  __nv_bfloat16* out;
  const float* G;            // Top-K routed gate weights [B][n_m] (nullptr: plain Eq. 3)
  int variant;               // partial-mask ablation variant (0 = Eq. 3; 1 NG, 2 NV, 3 NM)
  int act;                   // g when the kernel is the kRuntimeAct instantiation
  int B, d, h;
  int rows_base, rows_rem;   // CTA c owns rows_base + (c < rows_rem) rows
  int stages;                // ring depth
  int xpar;                  // u32 words per parity array of one token's x in smem (+ pad)
  int rem_a, rem_b;          // last-round rows of CTAs owning rows_base / rows_base + 1 rows
};

// swizzled byte offset within a 1024-aligned region of `rb`-byte rows (rb in {16..128})
__device__ __forceinline__ uint32_t swz(uint32_t lin, uint32_t rb) {
  return lin ^ (((lin >> 7) & (rb / 16 - 1)) << 4);
}

template <int NM, int ACT, int NB, int KSEL>
__global__ void __launch_bounds__(kDecThreads, 1)
gemv_mma_kernel(const DecParams p,
                const __grid_constant__ CUtensorMap mW64, const __grid_constant__ CUtensorMap mC64,
                const __grid_constant__ CUtensorMap mWa, const __grid_constant__ CUtensorMap mCa,
                const __grid_constant__ CUtensorMap mWb, const __grid_constant__ CUtensorMap mCb) {
  constexpr int SPAN = dec_code_span<NM>();
  constexpr int SB = dec_stage_bytes<NM>();
  constexpr int NACC = NB * ((KSEL > 0 ? KSEL : NM) + 1);
  extern __shared__ __align__(1024) uint8_t smem[];
  const int S = p.stages;
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * SB);
  uint64_t* empty = full + S;
  float* part = reinterpret_cast<float*>(empty + S);     // [16 warps][32 lanes][NACC]
  uint32_t* xs = reinterpret_cast<uint32_t*>(part + kDecConsumers * 32 * NACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int r0 = cta * p.rows_base + min(cta, p.rows_rem);
  const int nrows = p.rows_base + (cta < p.rows_rem ? 1 : 0);
  const int d = p.d;
  const int nfull = nrows / kDecFullRows, rem = nrows - nfull * kDecFullRows;
  const int nks_full = (d + 255) / 256;
  const int t_rem = (rem + 7) >> 3;
  const int wpt_rem = rem ? dec_wpt(t_rem) : 1;
  const int nks_rem = rem ? (d + 128 * wpt_rem - 1) / (128 * wpt_rem) : 0;
  const int nstages = nfull * nks_full + nks_rem;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kDecConsumers);
    }
    mbar_fence_init();
  }
  __syncthreads();
  pdl_launch_dependents();

  if (warp == kDecConsumers) {
    // ------------------------------------------------------------ producer (one thread)
    if (lane == 0) {
      // full rounds: boxes of 64 rows x (4 W blocks | 2 code blocks); the last round: boxes of
      // exactly `rem` rows x (2 WPT W blocks | WPT code blocks) -> two TMA ops per stage always,
      // no over-read of the neighbouring CTA's rows (one descriptor pair per CTA row count)
      const CUtensorMap* mWr = rem == p.rem_a ? &mWa : &mWb;
      const CUtensorMap* mCr = rem == p.rem_a ? &mCa : &mCb;
      prefetch_tmap(&mW64);
      if (NM > 0) prefetch_tmap(&mC64);
      if (rem) { prefetch_tmap(mWr); if (NM > 0) prefetch_tmap(mCr); }
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nstages; ++i) {
        const bool is_full = i < nfull * nks_full;
        const int rho = is_full ? i / nks_full : nfull;
        const int ks = is_full ? i - rho * nks_full : i - nfull * nks_full;
        const int rows = is_full ? kDecFullRows : rem;
        const int wpt = is_full ? 2 : wpt_rem;
        const int k0 = ks * 128 * wpt;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* wst = ring + (size_t)s * SB;
        mbar_arrive_expect_tx(&full[s], (uint32_t)(rows * wpt * (2 * 128 + SPAN)));
        tma_load_3d_hint(wst, is_full ? &mW64 : mWr, 0, r0 + rho * kDecFullRows, k0 / 64, &full[s], pol);
        if constexpr (NM > 0)
          tma_load_3d_hint(wst + kDecWBytes, is_full ? &mC64 : mCr, 0, r0 + rho * kDecFullRows, k0 / 128, &full[s], pol);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g = lane >> 2, c = lane & 3;
  const int B = p.B;
  const int prow = (g >> 1) + 4 * (g & 1);                 // pi(g): tile-local real row
  // pair q of this thread's 8 columns = group columns 8c + 2q, 8c + 2q + 1 -> layout bits
  // 4c + q and 16 + 4c + q; multiplying by 2^(15 - 4c - q) moves them to bits 15 and 31
  uint32_t mul[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) mul[q] = 1u << (15 - 4 * c - q);

  pdl_wait();                                              // x is the predecessor's output
  {
    // x -> smem split by bf16-pair parity: xs[b][parity][pair/2], zero-padded past d
    // token B is an all-zero row: lanes whose MMA column has no token read it unconditionally
    const int npair = p.xpar * 2 - 16;
    for (int v = threadIdx.x; v < (B + 1) * npair; v += kDecConsumers * 32) {
      const int b = v / npair, q = v - b * npair;
      uint32_t val = 0u;
      if (b < B && 2 * q < d) val = reinterpret_cast<const uint32_t*>(p.x + (size_t)b * d)[q];
      xs[(size_t)(2 * b + (q & 1)) * p.xpar + (q >> 1)] = val;
    }
  }
  // KSEL > 0: Top-K routed forward (Appendix B).  Only the masks some token of the batch selected
  // (nonzero G) are evaluated: up to KSEL of them, gathered into slots sel[0..KSEL) (uniform
  // across the CTA); unused slots repeat slot 0 with valid = false (computed, weighted 0).
  constexpr int NSLOT = KSEL > 0 ? KSEL : NM;              // masked accumulators
  int sel[NSLOT > 0 ? NSLOT : 1];
  uint32_t valid = (1u << NSLOT) - 1u;
#pragma unroll
  for (int k = 0; k < NSLOT; ++k) sel[k] = k;
  if constexpr (KSEL > 0) {
    uint32_t active = 0u;
    for (int q = 0; q < B * NM; ++q) active |= (p.G[q] != 0.0f ? 1u : 0u) << (q % NM);
    valid = 0u;
    int n = 0;
#pragma unroll
    for (int i = 0; i < NM; ++i)
      if (((active >> i) & 1u) && n < KSEL) { sel[n] = i; valid |= 1u << n; ++n; }
#pragma unroll
    for (int k = 0; k < NSLOT; ++k)
      if (!((valid >> k) & 1u)) sel[k] = sel[0];
  }
  named_bar_sync(1, kDecConsumers * 32);

  float acc[NB][NSLOT + 1][4];   // [0] = t; NM = 0 (dense projection): t only
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
#pragma unroll
    for (int a = 0; a <= NSLOT; ++a)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[nb][a][v] = 0.f;

  int s = 0;
  uint32_t ph = 0;
  int i = 0;
  for (int rho = 0; rho < nfull + (rem ? 1 : 0); ++rho) {
    const bool is_full = rho < nfull;
    const int rows = is_full ? kDecFullRows : rem;
    const int ntile = is_full ? kDecFullTiles : t_rem;
    const int wpt = is_full ? 2 : wpt_rem;
    const int nks = is_full ? nks_full : nks_rem;
    const int tl = warp / wpt, kp = warp - tl * wpt;        // tile and column part of this warp
    const bool live = tl < ntile;                           // warp-uniform
    const int srow = tl * 8 + prow;                         // row within the round's box
    // per-round shared-memory offsets (bytes, relative to a stage slot) of this thread's operands
    // for the four 32-column steps st of a stage: the stage loop then only adds the slot base
    uint32_t woff[4], coff[4];
#pragma unroll
    for (int st = 0; st < 4; ++st) {
      // A: pairs 4c..4c+3 of step st = one swizzled 16-byte read of W block (2 kp + st/2)
      woff[st] = swz((uint32_t)(((2 * kp + (st >> 1)) * rows + srow) * 128 + (32 * (st & 1) + 8 * c) * 2), 128);
      // the step's 32-column group (group st of code block kp): n_m words (16-byte chunks swizzled)
      if constexpr (NM > 0) coff[st] = (uint32_t)kDecWBytes + swz((uint32_t)((kp * rows + srow) * SPAN + st * 4 * NM), SPAN);
      else coff[st] = 0u;
    }
    // routed: the selected masks' words (one 4-byte read per slot and step)
    uint32_t csel[KSEL > 0 ? KSEL : 1][4];
    if constexpr (KSEL > 0) {
#pragma unroll
      for (int k = 0; k < KSEL; ++k)
#pragma unroll
        for (int st = 0; st < 4; ++st)
          csel[k][st] = (uint32_t)kDecWBytes + swz((uint32_t)((kp * rows + srow) * SPAN + (st * NM + sel[k]) * 4), SPAN);
    }
    // x: word index of pair 4c of step 0 of stage 0 for this lane's token column (token B = zeros)
    uint32_t xoff[NB];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const int tok = min(nb * 4 + (g >> 1), B);
      xoff[nb] = (uint32_t)((2 * tok + (g & 1)) * p.xpar + kp * 32 + 2 * c) * 4u;
    }
    for (int ks = 0; ks < nks; ++ks, ++i) {
      mbar_wait(&full[s], ph);
      if (live) {
        // slot base as a provably warp-uniform value: the LDS addresses become [per-thread + uniform]
        const uint8_t* wst = ring + __shfl_sync(0xffffffffu, s * SB, 0);
        const uint8_t* xst = reinterpret_cast<const uint8_t*>(xs) + __shfl_sync(0xffffffffu, ks * wpt * 128, 0);
#pragma unroll
        for (int st = 0; st < 4; ++st) {
          const uint4 wq = *reinterpret_cast<const uint4*>(wst + woff[st]);
          uint32_t mw[NSLOT > 0 ? NSLOT : 1];
          if constexpr (KSEL > 0) {
#pragma unroll
            for (int k = 0; k < KSEL; ++k) mw[k] = *reinterpret_cast<const uint32_t*>(wst + csel[k][st]);
          } else if constexpr (NM > 0)
#pragma unroll
          for (int q = 0; q < (NM + 3) / 4; ++q) {
            // n_m = 8: the second 16-byte chunk is the next one in the swizzled span
            const uint8_t* cp = wst + (q == 0 ? coff[st] : (coff[st] ^ 16u));
            if constexpr (NM == 1) mw[0] = *reinterpret_cast<const uint32_t*>(cp);
            else if constexpr (NM == 2) { const uint2 u = *reinterpret_cast<const uint2*>(cp); mw[0] = u.x; mw[1] = u.y; }
            else {
              const uint4 u = *reinterpret_cast<const uint4*>(cp);
              mw[4 * q] = u.x; mw[4 * q + 1] = u.y; mw[4 * q + 2] = u.z; mw[4 * q + 3] = u.w;
            }
          }
          // B: x pairs (4c + parity, 4c + 2 + parity) of the step for this lane's column(s)
          uint32_t xb[NB][2];
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            const uint2 u = *reinterpret_cast<const uint2*>(xst + xoff[nb] + st * 32);
            xb[nb][0] = u.x; xb[nb][1] = u.y;
          }
          // t += x W
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) mma_16816(acc[nb][0], wq.x, wq.y, wq.z, wq.w, xb[nb][0], xb[nb][1]);
          // u_i += x (sigma_i (.) W): pair q of the thread's 8 columns is register q of the quad
#pragma unroll
          for (int ii = 0; ii < NSLOT; ++ii) {
            const uint32_t a0 = sign_flip(wq.x, mw[ii], mul[0]), a1 = sign_flip(wq.y, mw[ii], mul[1]);
            const uint32_t a2 = sign_flip(wq.z, mw[ii], mul[2]), a3 = sign_flip(wq.w, mw[ii], mul[3]);
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) mma_16816(acc[nb][1 + ii], a0, a1, a2, a3, xb[nb][0], xb[nb][1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == S) { s = 0; ph ^= 1; }
    }

    // a5: (even pairs, even column) + (odd pairs, odd column) -> one value per (row, token)
    // and accumulator; parts kp >= 1 hand theirs to part 0 through smem (fixed order).  The round
    // ends at the same stage for every warp, so one consumer-wide barrier pair serves all tiles.
    float v[NB][NSLOT + 1];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int a = 0; a <= NSLOT; ++a) {
        v[nb][a] = acc[nb][a][0] + acc[nb][a][3];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[nb][a][q] = 0.f;
      }
    if (live && kp > 0) {
      float* pw = part + ((size_t)warp * 32 + lane) * NACC;
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int a = 0; a <= NSLOT; ++a) pw[nb * (NSLOT + 1) + a] = v[nb][a];
    }
    named_bar_sync(1, kDecConsumers * 32);                  // the producer keeps streaming meanwhile
    if (live && kp == 0) {
      for (int q = 1; q < wpt; ++q) {
        const float* pq = part + ((size_t)(warp + q) * 32 + lane) * NACC;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int a = 0; a <= NSLOT; ++a) v[nb][a] += pq[nb * (NSLOT + 1) + a];
      }
      const int row = rho * kDecFullRows + tl * 8 + prow;
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int tok = nb * 4 + c;
        if (tok < B && row < nrows) {
          float sv[NSLOT > 0 ? NSLOT : 1];
#pragma unroll
          for (int ii = 0; ii < NSLOT; ++ii) sv[ii] = 0.5f * (v[nb][0] + v[nb][1 + ii]);   // s_i = (t + u_i) / 2
          float y;
          if constexpr (NM == 0) {
            y = v[nb][0];                                   // dense projection x W (FFN W_o, row f1)
          } else if constexpr (KSEL > 0) {                         // routed: slot k is mask sel[k], weight G
            y = 0.f;
            const float* gw = p.G + (size_t)tok * NM;
#pragma unroll
            for (int k = 0; k < KSEL; ++k)
              if ((valid >> k) & 1u) y = fmaf(gw[sel[k]] * act_g<ACT>(sv[k], p.act), v[nb][0] - sv[k], y);
          } else {
            y = mglu_epilogue_v<ACT, NM>(v[nb][0], sv, p.G ? p.G + (size_t)tok * NM : nullptr, p.variant, p.act);   // Eq. 3 / routed / variant
          }
          p.out[(size_t)tok * p.h + r0 + row] = __float2bfloat16_rn(y);
        }
      }
    }
    named_bar_sync(1, kDecConsumers * 32);                  // partials are rewritten next round
  }
}

}  // namespace mglu
