// gemv_tc.cuh -- decode / small-batch regime on the 5th-generation tensor cores: a persistent,
// stream-K balanced, TMA-fed masked GEMV.  MGLU_PATH_TCDEC (AUTO for 5 <= B <= 24).
//
// What it computes is Eq. 3 per token row, by Alg. 1's single pass: W and
// the packed codes stream HBM -> SM exactly once per call, the unmasked product
// t = x W and the n_m gated sums are accumulated together and value_i = t - s_i.  As in the
// other tensor-core regimes the masked operand is the sign-flipped weight sigma_i (.) W (sigma = +1
// where M_i = 1, -1 where M_i = 0): the tensor core accumulates u_i = s_i - v_i and the epilogue
// takes s_i = (t + u_i) / 2 (exact rescaling of the same fp32 sums).
//
// Work decomposition (why stream-K): the layer is cut into 128-row tiles (one tcgen05 M = 128 tile,
// TMEM lane = W row) and each tile's reduction into units of KS columns.  The MT * (d / KS) units
// are split into gridDim.x = #SM contiguous, equal ranges (tile-major), so every SM streams the same
// number of bytes whatever h is (h / 128 tiles rarely divide 148 SMs).  A tile cut by a range
// boundary is finished by the CTA that owns its FIRST unit: the other CTAs touching it publish their
// fp32 partial accumulators (t, u_1..u_nm) to a global workspace and raise a flag; the owner adds
// them in CTA order (a fixed order -- repeats are bit-identical) and applies the fused Eq. 3
// epilogue.  The partial-publishing segment is always a CTA's first and the waiting one its last,
// so contributors publish early.  No atomics on data, no split-K pass (reading R9).
//
// Roles (warp-specialised, one CTA per SM):
//   * warps [0, 4 MG): MG masker groups of 4 warps (one per TMEM lane quarter, thread = tile row).
//     Group g owns the KA-column A-stages a = g (mod MG) of every unit: it reads its row's W and
//     mask words from shared memory and writes W itself plus the n_m sign-flipped copies (one IMAD +
//     one LOP3 per bf16 pair and mask, see sign_flip) into a TMEM A slot with tcgen05.st, then
//     arrives on the slot's a_full.  Every MMA therefore reads A from TMEM (the TS form: probes
//     showed an M=128, N=16 MMA with A in shared memory costs ~4x one with A in TMEM).
//   * warp 4 MG: TMA producer -- W (3-D box: KS/64 blocks x 128 rows x 64 columns, 128B swizzle),
//     the tile rows' mask words and x (KS/64 blocks x BN tokens x 64 columns) into an mbarrier ring.
//     W and the codes stream before griddepcontrol.wait (PDL: constant weights), x after it.
//   * warp 4 MG + 1: MMA issuer -- per A-stage (n_m + 1) x KA/16 MMAs (M = 128, N = BN, K = 16,
//     bf16 -> fp32) into an accumulator set of (n_m + 1) x BN TMEM columns (double-buffered when it
//     fits), committing the slot back to the maskers and the stage back to the producer.
//   * warps 4 MG + 2 .. 4 MG + 5: epilogue -- tcgen05.ld of the accumulators, partial publishing or
//     owner fix-up, Eq. 3, bf16 stores.
// Variants measured on the way (a per-group MMA issue, wider masker groups, SS operands, 64- and
// 128-column units) are logged in profiles/r01_tcdec_experiments.txt.
#pragma once
#include "common.cuh"
#include "mma_mask.cuh"
#include "tcgen05.cuh"
#include "tma.cuh"

namespace mglu {

// reduction columns per unit (= shared-memory stage) and per TMEM A-stage, by mask count (measured,
// profiles/r01_tcdec_experiments.txt: 256 / 64 for n_m <= 4; n_m = 8 keeps its stages small,
// 128 / 16, for ring depth and TMEM room)
template <int NM> __host__ __device__ constexpr int sk_ks() { return NM == 8 ? 128 : 256; }
template <int NM> __host__ __device__ constexpr int sk_ka() { return NM == 8 ? 16 : 64; }
#ifndef MGLU_SK_EPI_CH
#define MGLU_SK_EPI_CH 4 // epilogue tokens per chunk (8 and 16 measured slower, profiles/r01_tcdec_experiments.txt §11)
#endif
#ifndef MGLU_SK_NOFIXUP
#define MGLU_SK_NOFIXUP 0  // timing ablation only (wrong results): no partial stores / owner fix-up
#endif
#ifndef MGLU_SK_ACC2_SLOTS
#define MGLU_SK_ACC2_SLOTS 2  // A slots per masker group that must fit beside two accumulator sets
#endif
#ifndef MGLU_SK_SS_T
#define MGLU_SK_SS_T 0   // 1: t's MMA reads W from shared memory (SS); TMEM slots hold the masked copies only
#endif

struct SkParams {
  __nv_bfloat16* out;   // [B][h]
  const float* G;       // Top-K routed gate weights [B][n_m] (nullptr: every weight 1)
  int variant;          // partial-mask ablation variant (0 = Eq. 3)
  float* ws;            // partials [gridDim.x][NOP][B][128]
  uint32_t* flags;      // [gridDim.x], 0 between calls
  int B, d, h, act;
  int upt;              // units per tile = ceil(d / KS)
  float* z;             // non-null: write Alg. 1's z [B][2 n_m][h] (s_i, t - s_i) instead of y
  int units_base, units_rem;   // CTA c owns units_base + (c < units_rem) units
  int stages;
};

__device__ __forceinline__ int sk_unit0(const SkParams& p, int c) {
  return c * p.units_base + min(c, p.units_rem);
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}


// geometry of one instantiation: NM masks, BN token columns, MG masker groups of 4 warps
template <int NM, int BN, int MG> struct SkCfg {
  static constexpr int NOP = NM + 1;
  static constexpr int KS = sk_ks<NM>();
  static constexpr int KA = sk_ka<NM>();
  static constexpr int TOP = MGLU_SK_SS_T ? 0 : 1;   // W copies in a TMEM slot
  static constexpr int SLOT = (NM + TOP) * KA / 2;
  static constexpr int ACC = NOP * BN;
  static constexpr int NACC = 2 * ACC + MGLU_SK_ACC2_SLOTS * MG * SLOT <= 512 ? 2 : 1;
  static constexpr int SA_FIT = (512 - NACC * ACC) / SLOT / MG * MG;
  static constexpr int SA = SA_FIT > 4 * MG ? 4 * MG : SA_FIT;
  static constexpr int WPS = KS / 32 * NM;
  static constexpr int CW = WPS < 4 ? 4 : WPS;
  static constexpr int WB = KS / 64 * 128 * 128;
  static constexpr int XB = KS / 64 * BN * 128;
  static constexpr int CB = 128 * CW * 4;
  static constexpr int SB = (WB + XB + CB + 1023) / 1024 * 1024;
  static constexpr int THREADS = (4 * MG + 6) * 32;
  static constexpr bool ok = SA >= MG && KS / KA >= MG && (KS / KA) % MG == 0;
};

template <int NM, int BN, int MG>
__global__ void __launch_bounds__(SkCfg<NM, BN, MG>::THREADS, 1)
gemv_tc_kernel(const SkParams p, const __grid_constant__ CUtensorMap mW, const __grid_constant__ CUtensorMap mX,
                const __grid_constant__ CUtensorMap mC) {
  using C = SkCfg<NM, BN, MG>;
  constexpr int NOP = C::NOP, KA = C::KA, SLOT = C::SLOT, SA = C::SA, NACC = C::NACC, ACC = C::ACC;
  constexpr int WPS = C::WPS, CW = C::CW, WB = C::WB, XB = C::XB, SB = C::SB;
  constexpr int KS = C::KS, APS = KS / KA, WW = KA / 2;
  constexpr uint32_t IDESC = idesc_bf16_f32(128, BN);
  constexpr uint32_t A_COL0 = NACC * ACC;
  constexpr int kTma = 4 * MG, kMma = 4 * MG + 1, kEpi0 = 4 * MG + 2;
  static_assert(C::ok, "TMEM budget");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * SB);
  uint64_t* empty = full + S;
  uint64_t* a_full = empty + S;
  uint64_t* a_empty = a_full + SA;
  uint64_t* acc_full = a_empty + SA;
  uint64_t* acc_empty = acc_full + NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + NACC);

  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);
  const int lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int u0 = sk_unit0(p, cta);
  const int u1 = u0 + p.units_base + (cta < p.units_rem ? 1 : 0);
  const int upt = p.upt;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < SA; ++s) { mbar_init(&a_full[s], 4); mbar_init(&a_empty[s], 1); }
    for (int s = 0; s < NACC; ++s) { mbar_init(&acc_full[s], 1); mbar_init(&acc_empty[s], 4); }
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();

  if (warp == kTma) {
    if (lane == 0) {
      prefetch_tmap(&mW);
      prefetch_tmap(&mC);
      prefetch_tmap(&mX);
      const uint64_t pol = policy_evict_first();
      const int n = u1 - u0;
      const int pre = n < S ? n : S;
      for (int i = 0; i < pre; ++i) {
        const int u = u0 + i, tile = u / upt, ks = u - tile * upt;
        uint8_t* st = smem + (size_t)i * SB;
        mbar_arrive_expect_tx(&full[i], (uint32_t)(WB + XB + C::CB));
        tma_load_3d_hint(st, &mW, 0, tile * 128, ks * (KS / 64), &full[i], pol);
        tma_load_2d_hint(st + WB + XB, &mC, (ks * WPS) / CW * CW, tile * 128, &full[i], pol);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) {
        const int ks = (u0 + i) % upt;
        tma_load_3d(smem + (size_t)i * SB + WB, &mX, 0, 0, ks * (KS / 64), &full[i]);
      }
      int s = pre % S;
      uint32_t ph = pre == S ? 1u : 0u;
      for (int i = pre; i < n; ++i) {
        const int u = u0 + i, tile = u / upt, ks = u - tile * upt;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + (size_t)s * SB;
        mbar_arrive_expect_tx(&full[s], (uint32_t)(WB + XB + C::CB));
        tma_load_3d_hint(st, &mW, 0, tile * 128, ks * (KS / 64), &full[s], pol);
        tma_load_3d(st + WB, &mX, 0, 0, ks * (KS / 64), &full[s]);
        tma_load_2d_hint(st + WB + XB, &mC, (ks * WPS) / CW * CW, tile * 128, &full[s], pol);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == kMma) {
    int s = 0, js = 0, set = 0;
    uint32_t ph = 0;
    uint32_t use_a = 0u, use_b = 0u;                   // completed uses of accumulator set 0 / 1
    for (int u = u0; u < u1; ++u) {
      const bool seg_first = u == u0 || u % upt == 0;
      const bool seg_last = u == u1 - 1 || u % upt == upt - 1;
      if (seg_first) {
        mbar_wait(&acc_empty[set], ((set ? use_b : use_a) & 1u) ^ 1u);
        tc_fence_after();
      }
      const uint32_t st = smem_u32(smem + (size_t)s * SB);
      const uint32_t dacc = tmem + (uint32_t)(set * ACC);
#pragma unroll
      for (int a = 0; a < APS; ++a, ++js) {
        const int sa = js % SA;
        mbar_wait(&a_full[sa], (uint32_t)(js / SA) & 1u);   // implies full[s]: the maskers waited it
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < KA / 16; ++kk) {
            const int k16 = a * (KA / 16) + kk;
            const uint64_t bdesc = smem_desc_kmajor(st + WB + (k16 >> 2) * BN * 128, 128) + (uint64_t)((k16 & 3) * 2);
            const uint32_t accum = (seg_first && k16 == 0) ? 0u : 1u;
            const uint32_t asl = tmem + A_COL0 + (uint32_t)(sa * SLOT + kk * 8);
            if constexpr (C::TOP == 0) {
              const uint64_t adesc = smem_desc_kmajor(st + (k16 >> 2) * 16384, 128) + (uint64_t)((k16 & 3) * 2);
              tc_mma_ss(dacc, adesc, bdesc, IDESC, accum);
            }
#pragma unroll
            for (int o = 1 - C::TOP; o < NOP; ++o)
              tc_mma_ts(dacc + (uint32_t)(o * BN), asl + (uint32_t)((o - 1 + C::TOP) * WW), bdesc, IDESC, accum);
          }
          tc_commit(&a_empty[sa]);
          if (a == APS - 1) tc_commit(&empty[s]);
          if (a == APS - 1 && seg_last) tc_commit(&acc_full[set]);
        }
        __syncwarp();
      }
      if (seg_last) { if (set) ++use_b; else ++use_a; if (NACC == 2) set ^= 1; }
      if (++s == S) { s = 0; ph ^= 1; }
    }
  } else if (warp < 4 * MG) {
    const int g = warp >> 2;
    const int m = (warp & 3) * 32 + lane;
    const uint32_t a_lane = tmem + ((uint32_t)((warp & 3) * 32) << 16) + A_COL0;
    int s = 0, js = 0;
    uint32_t ph = 0;
    for (int u = u0; u < u1; ++u) {
      const int ks = u % upt;
      mbar_wait(&full[s], ph);
      const uint8_t* st = smem + (size_t)s * SB;
      const int wofs = (ks * WPS) % CW;
#pragma unroll
      for (int a = 0; a < APS; ++a, ++js) {
        if (a % MG != g) continue;
        const int col = a * KA;
        uint32_t w[WW];
#pragma unroll
        for (int c = 0; c < KA / 8; ++c) {
          const uint32_t chunk = (uint32_t)(((col & 63) >> 3) + c) ^ (uint32_t)(m & 7);
          const uint4 v = *reinterpret_cast<const uint4*>(st + (col >> 6) * 16384 + m * 128 + chunk * 16);
          w[4 * c] = v.x; w[4 * c + 1] = v.y; w[4 * c + 2] = v.z; w[4 * c + 3] = v.w;
        }
        // mask words of the A-stage's 32-column groups (swizzled code box: conflict-free reads)
        constexpr int NG = KA >= 32 ? KA / 32 : 1, PPG = KA >= 32 ? 16 : KA / 2;
        uint32_t cw[NG][NM];
#pragma unroll
        for (int gi = 0; gi < NG; ++gi)
          lds_words_swz<NM>(st + WB + XB, (uint32_t)(m * CW * 4 + (wofs + ((col >> 5) + gi) * NM) * 4), CW * 4, cw[gi]);
        const int pair0 = (col & 31) >> 1;
        const int sa = js % SA;
        mbar_wait(&a_empty[sa], ((uint32_t)(js / SA) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t a0 = a_lane + (uint32_t)(sa * SLOT);
        if constexpr (C::TOP) tmem_st_n<WW>(a0, w);
#pragma unroll
        for (int i = 0; i < NM; ++i) {
          uint32_t op[WW];
#pragma unroll
          for (int q = 0; q < WW; ++q)                     // pair q: group q / PPG, bits (p, p + 16)
            op[q] = sign_flip(w[q], cw[q / PPG][i], 1u << (15 - pair0 - (q % PPG)));
          tmem_st_n<WW>(a0 + (uint32_t)((C::TOP + i) * WW), op);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[sa]);
      }
      if (++s == S) { s = 0; ph ^= 1; }
    }
  } else if (warp >= kEpi0) {
    const int quarter = warp & 3;
    const int m = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const int B = p.B;
    constexpr int CH = MGLU_SK_EPI_CH;                 // tokens per epilogue chunk (multiple of 4)
    static_assert(CH % 4 == 0 && BN % CH == 0, "epilogue chunk");
    const int nch = (B + CH - 1) / CH;
    pdl_wait();
    int set = 0;
    uint32_t use_a = 0u, use_b = 0u;                   // completed uses of accumulator set 0 / 1
    int u = u0;
    while (u < u1) {
      const int tile = u / upt;
      const int tile_end = (tile + 1) * upt;
      const int seg_end = u1 < tile_end ? u1 : tile_end;
      const bool owner = u == tile * upt;
      const bool whole = owner && seg_end == tile_end;
      mbar_wait(&acc_full[set], (set ? use_b : use_a) & 1u);
      tc_fence_after();
      const uint32_t abase = lane_base + (uint32_t)(set * ACC);
      const int grow = tile * 128 + m;
      int ncon = 0;
      if (owner && !whole && !MGLU_SK_NOFIXUP) {
        while (cta + 1 + ncon < (int)gridDim.x && sk_unit0(p, cta + 1 + ncon) < tile_end) ++ncon;
        for (int k = 1; k <= ncon; ++k) {
          uint32_t polls = 0;
          while (ld_acquire_u32(p.flags + cta + k) == 0u) {
            if (++polls == (1u << 26)) __trap();
            __nanosleep(64);
          }
        }
      }
      for (int ch = 0; ch < nch; ++ch) {
        float f[NOP][CH];
        {
          uint32_t v[NOP][CH];                         // all loads of the chunk in flight, one wait
#pragma unroll
          for (int o = 0; o < NOP; ++o)
#pragma unroll
            for (int c4 = 0; c4 < CH / 4; ++c4)
              tmem_ld4(abase + (uint32_t)(o * BN + ch * CH + c4 * 4), *reinterpret_cast<uint32_t(*)[4]>(&v[o][c4 * 4]));
          tmem_ld_wait();
#pragma unroll
          for (int o = 0; o < NOP; ++o)
#pragma unroll
            for (int q = 0; q < CH; ++q) f[o][q] = __uint_as_float(v[o][q]);
        }
        if (!owner) {
          if (MGLU_SK_NOFIXUP) continue;
          float* wsp = p.ws + (size_t)cta * NOP * B * 128 + m;
#pragma unroll
          for (int o = 0; o < NOP; ++o)
#pragma unroll
            for (int q = 0; q < CH; ++q) {
              const int tok = ch * CH + q;
              if (tok < B) __stcg(wsp + ((size_t)o * B + tok) * 128, f[o][q]);
            }
          continue;
        }
        for (int k = 1; k <= ncon; ++k) {
          const float* wsp = p.ws + (size_t)(cta + k) * NOP * B * 128 + m;
#pragma unroll
          for (int o = 0; o < NOP; ++o)
#pragma unroll
            for (int q = 0; q < CH; ++q) {
              const int tok = ch * CH + q;
              if (tok < B) f[o][q] += __ldcg(wsp + ((size_t)o * B + tok) * 128);
            }
        }
        if (grow < p.h) {
#pragma unroll
          for (int q = 0; q < CH; ++q) {
            const int tok = ch * CH + q;
            if (tok < B && p.z) {                          // partials (debug / parity of a5, a6)
              const float t = f[0][q];
              float* zt = p.z + (size_t)tok * 2 * NM * p.h + grow;
#pragma unroll
              for (int i = 0; i < NM; ++i) {
                const float sg = 0.5f * (t + f[1 + i][q]);
                zt[(size_t)i * p.h] = sg;
                zt[(size_t)(NM + i) * p.h] = t - sg;
              }
            } else if (tok < B) {
              const float t = f[0][q];
              float y = 0.f;
#pragma unroll
              for (int i = 0; i < NM; ++i) {
                const float sg = 0.5f * (t + f[1 + i][q]);
                const float gate = (p.variant & 1) ? t : sg;                // ablation variants
                const float value = (p.variant & 2) ? t : t - sg;
                const float wgt = p.G ? p.G[(size_t)tok * NM + i] : 1.f;    // routed (Appendix B)
                y = fmaf(wgt * act_rt(p.act, gate), value, y);
              }
              p.out[(size_t)tok * p.h + grow] = __float2bfloat16_rn(y);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[set]);
      if (!owner) {
        __threadfence();
        named_bar_sync(15, 128);
        if (warp == kEpi0 && lane == 0) st_release_u32(p.flags + cta, 1u);
      } else if (ncon) {
        named_bar_sync(15, 128);
        if (warp == kEpi0)
          for (int k = lane; k < ncon; k += 32) p.flags[cta + 1 + k] = 0u;
      }
      if (set) ++use_b; else ++use_a;
      if (NACC == 2) set ^= 1;
      u = seg_end;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace mglu
