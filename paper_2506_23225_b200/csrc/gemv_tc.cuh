// gemv_tc.cuh -- batched-decode regime on the 5th-generation tensor cores: a persistent, stream-K
// balanced, TMA-fed masked GEMV.  MGLU_PATH_TCDEC (AUTO for 5 <= B <= 64, and n_m = 8 on large
// layers from B = 1).
//
// What it computes is Eq. 3 per token row, by Alg. 1's single pass: W and
// the packed codes stream HBM -> SM exactly once per call, the unmasked product
// t = x W and the n_m gated sums are accumulated together and value_i = t - s_i.  As in the
// other tensor-core regimes the masked operand is the sign-flipped weight sigma_i (.) W (sigma = +1
// where M_i = 1, -1 where M_i = 0): the tensor core accumulates u_i = s_i - v_i and the epilogue
// takes s_i = (t + u_i) / 2 (exact rescaling of the same fp32 sums).
//
// Work decomposition (why stream-K): the layer is cut into 128-row tiles (one tcgen05 M = 128 tile,
// TMEM lane = W row) and each tile's reduction into units of KS = 128 columns.  The MT * (d / KS)
// units are split into gridDim.x = #SM contiguous, equal ranges (tile-major), so every SM streams
// the same number of bytes whatever h is (h / 128 tiles rarely divide 148 SMs).  A CTA's range is
// cut into segments at tile boundaries; a tile cut by a range boundary ("shared") is reduced by its
// LAST ARRIVER: every contributor publishes its fp32 partial accumulators (t, u_1..u_nm) to a
// workspace and bumps the tile's ticket counter (one atomic on a counter, none on data); the CTA
// that takes the last ticket adds all partials in CTA order (a fixed order: repeats are
// bit-identical) and runs the fused Eq. 3 epilogue.  Nobody waits for anybody (no spin on another
// CTA: forward progress whatever runs concurrently), and each CTA processes its (at most two)
// shared segments FIRST, so shared tiles complete early and their reduction overlaps the streaming
// of the CTA's whole tiles (reading R9: no split-K pass, no atomics on data).
//
// Pipelines (warp-specialised, one CTA per SM):
//   * W ring: per unit one 3-D TMA box of W (2 64-column blocks x 128 rows, 128B swizzle) + one box
//     of the tile rows' mask words.  Masker warps copy their share of a stage into registers and hand
//     the slot back at once (a slot is held only for the shared-memory load latency, so nearly the
//     whole ring stays in flight -- the same lesson as the HMMA decode kernel).
//   * x ring: per unit the BN-token x box (2 blocks x BN rows x 64 columns), released by the MMA
//     commit (the tensor core reads it as the B operand).  W streams before griddepcontrol.wait
//     (PDL: constant weights), x after it.
//   * warps [0, 4 MG): MG masker groups of 4 warps (one per TMEM lane quarter, thread = tile row).
//     Group g owns the KA = 32-column A-stages a = g (mod MG) of every unit: it writes W itself
//     plus the n_m sign-flipped copies (one IMAD + one LOP3 per bf16 pair and mask, see sign_flip)
//     into a TMEM A slot with tcgen05.st and arrives on the slot's a_full.  Every MMA therefore
//     reads A from TMEM (the TS form: an M = 128, N = 16 MMA with A in shared memory costs ~4x).
//   * warps 4 MG and 4 MG + 1: TMA producers of the W ring and of the x ring (separate warps: two
//     spinning lanes of one warp would serialise behind each other).
//   * warp 4 MG + 2: MMA issuer -- per A-stage (n_m + 1) x 2 MMAs (M = 128, N = BN, K = 16, bf16 ->
//     fp32) into an accumulator set of (n_m + 1) x BN TMEM columns (double-buffered when it fits).
//   * warps 4 MG + 3 .. 4 MG + 6: epilogue -- tcgen05.ld of the accumulators, publish / last-arriver
//     reduction, Eq. 3 (or the partials z), bf16 stores.
#pragma once
#include "common.cuh"
#include "mma_mask.cuh"
#include "tcgen05.cuh"
#include "tma.cuh"

namespace mglu {

#ifndef MGLU_SK_ABL
#define MGLU_SK_ABL 0   // timing ablations (wrong results): 1 no sign flips, 2 no masked-copy stores, 3 t's MMA only
#endif
#ifndef MGLU_SK_EPI_CH
#define MGLU_SK_EPI_CH 4 // epilogue tokens per chunk (8 and 16 measured slower, profiles/r01_tcdec_experiments.txt §11)
#endif

struct SkParams {
  __nv_bfloat16* out;   // [B][h]
  const float* G;       // Top-K routed gate weights [B][n_m] (nullptr: every weight 1)
  float* z;             // non-null: write Alg. 1's z [B][2 n_m][h] (s_i, t - s_i) instead of y
  int variant;          // partial-mask ablation variant (0 = Eq. 3)
  float* ws;            // published partials [gridDim.x][2 segment slots][NOP][B][128]
  uint32_t* tickets;    // [tiles] arrival counters, 0 between calls (the last arriver re-arms)
  int B, d, h, act;
  int upt;              // units per tile = ceil(d / KS)
  int units_base, units_rem;   // stream-K: CTA c owns units_base + (c < units_rem) units
  int row_mode;         // 1: row split -- CTA c owns tiles [c tpc, (c + 1) tpc) over the whole d
  int tpc;              // row split: tiles per CTA
  int tr_base, tr_rem;  // row split: tile t has tr_base + (t < tr_rem) rows (<= 128), contiguous
  int wstages, xstages;
  int wblk, wsb;        // bytes of one 64-column W block of a stage (16384: 128 rows) and of a stage
};

// one segment of a CTA's work: a run of units [klo, khi) of one tile of `rows` W rows from row0
struct SkSeg {
  int tile, row0, rows, klo, khi;
  bool shared;          // stream-K tile cut by a CTA range boundary (last-arriver reduction)
  bool big;             // row split: the tile has tr_base + 1 rows (selects the TMA box)
};

__device__ __forceinline__ int sk_unit0(const SkParams& p, int c) {
  return c * p.units_base + min(c, p.units_rem);
}
// CTA owning unit u (inverse of sk_unit0)
__device__ __forceinline__ int sk_cta_of(const SkParams& p, int u) {
  const int big = p.units_rem * (p.units_base + 1);
  return u < big ? u / (p.units_base + 1) : p.units_rem + (u - big) / p.units_base;
}

// geometry of one instantiation: NM masks, BN token columns, MG masker groups of 4 warps
template <int NM, int BN, int MG> struct SkCfg {
  static constexpr int NOP = NM + 1;
  static constexpr int KS = 128;                          // unit width (columns)
  // A-stage width: one 32-column mask group (16 at n_m = 8 measured slower: 169 vs 129 us on config 5)
#ifndef MGLU_SK_KA
#define MGLU_SK_KA 32
#endif
#ifndef MGLU_SK_KA8
#define MGLU_SK_KA8 32
#endif
  static constexpr int KA = NM >= 8 ? MGLU_SK_KA8 : MGLU_SK_KA;
  static constexpr int APS = KS / KA;                     // A-stages per unit
  static constexpr int SLOT = NOP * KA / 2;               // TMEM columns of an A slot (W + n_m copies)
  static constexpr int ACC = NOP * BN;                    // TMEM columns of an accumulator set
  // accumulator sets and A slots, when the CTA has several segments (stream-K, or a row split of
  // several tiles per CTA: double-buffered accumulators) or one (a single set, one slot more).
  // A-stage J of the CTA uses slot J % SA whatever the masker group, so SA need not divide by MG.
  static constexpr int NACC = 2 * ACC + 2 * MG * SLOT <= 512 ? 2 : 1;
  static constexpr int SA_CAP = 4 * MG + 2;
  static constexpr int SA_FIT = (512 - NACC * ACC) / SLOT;
  static constexpr int SA = SA_FIT > SA_CAP ? SA_CAP : SA_FIT;
  static constexpr int SA1_FIT = (512 - ACC) / SLOT;                 // one accumulator set
  static constexpr int SA1 = SA1_FIT > SA_CAP ? SA_CAP : SA1_FIT;
  static constexpr int CWORDS = KS / 32 * NM;             // mask words of a row per unit
  static constexpr int WB = KS / 64 * 128 * 128;          // W box bytes
  static constexpr int CB = 128 * CWORDS * 4;             // code box bytes
  static constexpr int WSB = (WB + CB + 1023) / 1024 * 1024;
  static constexpr int XB = (KS / 64 * BN * 128 + 1023) / 1024 * 1024;
  static constexpr int THREADS = (4 * MG + 7) * 32;
  static constexpr bool ok = SA >= MG && APS % MG == 0;
  static constexpr int SA_MAX = SA1 > SA ? SA1 : SA;
};

// TMEM -> registers: the NOP accumulators of token chunk ch (CH tokens) of this thread's row
template <int NOP, int BN, int CH>
__device__ __forceinline__ void sk_ld_chunk(uint32_t abase, int ch, float (&f)[NOP][CH]) {
  uint32_t (&v)[NOP][CH] = *reinterpret_cast<uint32_t(*)[NOP][CH]>(&f);   // loaded in place
#pragma unroll
  for (int o = 0; o < NOP; ++o)
#pragma unroll
    for (int c4 = 0; c4 < CH / 4; ++c4)
      tmem_ld4(abase + (uint32_t)(o * BN + ch * CH + c4 * 4), *reinterpret_cast<uint32_t(*)[4]>(&v[o][c4 * 4]));
  tmem_ld_wait();                                          // all loads of the chunk in flight, one wait
}

// Eq. 3 epilogue (a6, a7) of token chunk ch of tile row `grow` from its summed accumulators f[0] = t,
// f[1 + i] = u_i (s_i = (t + u_i) / 2), or Alg. 1's z when p.z is set
template <int NM, int CH, int ACT>
__device__ __forceinline__ void sk_epi_store_g(const SkParams& p, const float (&f)[NM + 1][CH], int ch, int grow) {
#pragma unroll
  for (int q = 0; q < CH; ++q) {
    const int tok = ch * CH + q;
    if (tok >= p.B) continue;
    const float t = f[0][q];
    if (p.z) {                                             // partials (debug / parity of a5, a6)
      float* zt = p.z + (size_t)tok * 2 * NM * p.h + grow;
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        const float sg = 0.5f * (t + f[1 + i][q]);
        zt[(size_t)i * p.h] = sg;
        zt[(size_t)(NM + i) * p.h] = t - sg;
      }
      continue;
    }
    float y = 0.f;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      const float sg = 0.5f * (t + f[1 + i][q]);
      const float gate = (p.variant & 1) ? t : sg;              // ablation variants
      const float value = (p.variant & 2) ? t : t - sg;
      const float wgt = p.G ? p.G[(size_t)tok * NM + i] : 1.f;  // routed (Appendix B)
      y = fmaf(wgt * act_fast<ACT>(gate, p.act), value, y);
    }
    p.out[(size_t)tok * p.h + grow] = __float2bfloat16_rn(y);
  }
}
// g resolved once per chunk, not per output: Swish (the default) inline, the others through act_rt
template <int NM, int CH>
__device__ __forceinline__ void sk_epi_store(const SkParams& p, const float (&f)[NM + 1][CH], int ch, int grow) {
  if (p.act == kSwish) sk_epi_store_g<NM, CH, kSwish>(p, f, ch, grow);
  else sk_epi_store_g<NM, CH, kRuntimeAct>(p, f, ch, grow);
}

// ONE: the CTA has a single segment (row split, one tile per CTA): one accumulator set and the TMEM
// it frees as A slots
template <int NM, int BN, int MG, bool ONE>
__global__ void __launch_bounds__(SkCfg<NM, BN, MG>::THREADS, 1)
gemv_tc_kernel(const SkParams p, const __grid_constant__ CUtensorMap mW, const __grid_constant__ CUtensorMap mX,
               const __grid_constant__ CUtensorMap mC, const __grid_constant__ CUtensorMap mWb,
               const __grid_constant__ CUtensorMap mCb) {
  using C = SkCfg<NM, BN, MG>;
  constexpr int NOP = C::NOP, KA = C::KA, APS = C::APS, SLOT = C::SLOT;
  constexpr int ACC = C::ACC, CWORDS = C::CWORDS, WB = C::WB, XB = C::XB, KS = C::KS;
  constexpr int WW = KA / 2;                               // 32-bit words (bf16 pairs) of an A-stage row
  constexpr int APG = APS / MG;                            // A-stages per unit of one masker group
#ifndef MGLU_SK_LG1
#define MGLU_SK_LG1 1   // one A-stage in registers at a time: 1-1.5 % faster than two at B = 8..32 (profiles/r02/tc_gemv_experiments.txt)
#endif
  constexpr int LG = (NM >= 8 || MGLU_SK_LG1) ? 1 : APG;   // A-stages a masker holds in registers at once
  constexpr uint32_t IDESC = idesc_bf16_f32(128, BN);
  constexpr int CH = MGLU_SK_EPI_CH;                   // tokens per epilogue chunk (multiple of 4)
  static_assert(CH % 4 == 0 && BN % CH == 0, "epilogue chunk");
  constexpr int NACC = ONE ? 1 : C::NACC, SA = ONE ? C::SA1 : C::SA;
  constexpr uint32_t A_COL0 = (uint32_t)(NACC * ACC);
  constexpr int kTma = 4 * MG, kTmaX = 4 * MG + 1, kMma = 4 * MG + 2, kEpi0 = 4 * MG + 3;
  static_assert(C::ok, "TMEM budget");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int SW = p.wstages, SX = p.xstages;
  uint8_t* wring = smem;
  const int WSBr = p.wsb, WBLK = p.wblk, WCODE = KS / 64 * p.wblk;   // stage layout (host: SkCfg / row split)
  uint8_t* xring = smem + (size_t)SW * WSBr;
  uint64_t* w_full = reinterpret_cast<uint64_t*>(xring + (size_t)SX * XB);
  uint64_t* w_empty = w_full + SW;
  uint64_t* x_full = w_empty + SW;
  uint64_t* x_empty = x_full + SX;
  uint64_t* a_full = x_empty + SX;
  uint64_t* a_empty = a_full + SA;
  uint64_t* acc_full = a_empty + SA;
  uint64_t* acc_empty = acc_full + NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + NACC);
  uint32_t* last_flag = tmem_slot + 1;

  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);
  const int lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int upt = p.upt;
  // stream-K: segments of [u0, u1) cut at tile boundaries, processed as: first, last, then the middle
  // ones (the first and last are the only ones that can be shared with a neighbour CTA).
  // row split: the CTA's tpc tiles in order, each over all of d (no sharing, no reduction).
  const int u0 = p.row_mode ? 0 : sk_unit0(p, cta);
  const int u1 = p.row_mode ? 0 : u0 + p.units_base + (cta < p.units_rem ? 1 : 0);
  const int t_first = u0 / upt, t_last = u1 > u0 ? (u1 - 1) / upt : t_first;
  const int nseg = p.row_mode ? p.tpc : (u1 > u0 ? t_last - t_first + 1 : 0);
  auto seg = [&](int k) {
    SkSeg s;
    if (p.row_mode) {
      s.tile = cta * p.tpc + k;
      s.big = s.tile < p.tr_rem;
      s.row0 = s.tile * p.tr_base + min(s.tile, p.tr_rem);
      s.rows = p.tr_base + (s.big ? 1 : 0);
      s.klo = 0;
      s.khi = upt;
      s.shared = false;
    } else {
      s.tile = k == 0 ? t_first : k == 1 ? t_last : t_first + k - 1;
      s.big = false;
      s.row0 = s.tile * 128;
      s.rows = 128;
      s.klo = max(u0, s.tile * upt) - s.tile * upt;
      s.khi = min(u1, (s.tile + 1) * upt) - s.tile * upt;
      s.shared = s.klo > 0 || s.khi < upt;
    }
    return s;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < SW; ++s) { mbar_init(&w_full[s], 1); mbar_init(&w_empty[s], 4 * MG); }
    for (int s = 0; s < SX; ++s) { mbar_init(&x_full[s], 1); mbar_init(&x_empty[s], 1); }
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
    if (lane == 0) {                                       // W ring (constant weights: before the PDL wait)
      prefetch_tmap(&mW);
      prefetch_tmap(&mC);
      if (p.row_mode) { prefetch_tmap(&mWb); prefetch_tmap(&mCb); }
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (int k = 0; k < nseg; ++k) {
        const SkSeg sg = seg(k);
        const CUtensorMap* mw = sg.big ? &mW : &mWb;
        const CUtensorMap* mc = sg.big ? &mC : &mCb;
        for (int ks = sg.klo; ks < sg.khi; ++ks) {
          mbar_wait(&w_empty[s], ph ^ 1);
          uint8_t* st = wring + (size_t)s * WSBr;
          if (p.row_mode) {
            // boxes of exactly the tile's rows, each 64-column block at its 128-row slot (the
            // maskers' layout does not depend on the row count; rows past it are never used)
            mbar_arrive_expect_tx(&w_full[s], (uint32_t)(sg.rows * (KS * 2 + CWORDS * 4)));
#pragma unroll
            for (int b = 0; b < KS / 64; ++b)
              tma_load_2d_hint(st + b * WBLK, mw, ks * KS + b * 64, sg.row0, &w_full[s], pol);
            tma_load_2d_hint(st + WCODE, mc, ks * CWORDS, sg.row0, &w_full[s], pol);
          } else {
            mbar_arrive_expect_tx(&w_full[s], (uint32_t)(WB + C::CB));
            tma_load_3d_hint(st, &mW, 0, sg.row0, ks * (KS / 64), &w_full[s], pol);
            tma_load_2d_hint(st + WB, &mC, ks * CWORDS, sg.row0, &w_full[s], pol);
          }
          if (++s == SW) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == kTmaX) {
    if (lane == 0) {                                       // x ring (the predecessor's output)
      prefetch_tmap(&mX);
      pdl_wait();
      int s = 0;
      uint32_t ph = 0;
      for (int k = 0; k < nseg; ++k) {
        const SkSeg sg = seg(k);
        for (int ks = sg.klo; ks < sg.khi; ++ks) {
          mbar_wait(&x_empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&x_full[s], (uint32_t)(KS / 64 * BN * 128));
          tma_load_3d(xring + (size_t)s * XB, &mX, 0, 0, ks * (KS / 64), &x_full[s]);
          if (++s == SX) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == kMma) {
    int sx = 0, js = 0, set = 0;
    uint32_t phx = 0;
    uint32_t use_a = 0u, use_b = 0u;                       // completed uses of accumulator set 0 / 1
    for (int k = 0; k < nseg; ++k) {
      const SkSeg sg = seg(k);
      const int lo = sg.klo, hi = sg.khi;
      mbar_wait(&acc_empty[set], ((set ? use_b : use_a) & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t dacc = tmem + (uint32_t)(set * ACC);
      for (int u = lo; u < hi; ++u) {
        mbar_wait(&x_full[sx], phx);
        tc_fence_after();
        const uint32_t xst = smem_u32(xring + (size_t)sx * XB);
#pragma unroll
        for (int a = 0; a < APS; ++a, ++js) {
          const int sa = js % SA;
          mbar_wait(&a_full[sa], (uint32_t)(js / SA) & 1u);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < KA / 16; ++kk) {
              const int k16 = a * (KA / 16) + kk;         // 16-column step within the unit
              const uint64_t bdesc = smem_desc_kmajor(xst + (k16 >> 2) * BN * 128, 128) + (uint64_t)((k16 & 3) * 2);
              const uint32_t accum = (u == lo && k16 == 0) ? 0u : 1u;
              const uint32_t asl = tmem + A_COL0 + (uint32_t)(sa * SLOT + kk * 8);
#pragma unroll
              for (int o = 0; o < (MGLU_SK_ABL == 3 ? 1 : NOP); ++o)
                tc_mma_ts(dacc + (uint32_t)(o * BN), asl + (uint32_t)(o * WW), bdesc, IDESC, accum);
            }
            tc_commit(&a_empty[sa]);
            if (a == APS - 1) tc_commit(&x_empty[sx]);
            if (a == APS - 1 && u == hi - 1) tc_commit(&acc_full[set]);
          }
          __syncwarp();
        }
        if (++sx == SX) { sx = 0; phx ^= 1; }
      }
      if (set) ++use_b; else ++use_a;
      if (NACC == 2) set ^= 1;
    }
  } else if (warp < 4 * MG) {
    // ------------------------------------------------ maskers: thread = tile row m
    const int g = warp >> 2;
    const int m = (warp & 3) * 32 + lane;
    const uint32_t a_lane = tmem + ((uint32_t)((warp & 3) * 32) << 16) + A_COL0;
    int s = 0, js = 0;
    uint32_t ph = 0;
    for (int k = 0; k < nseg; ++k) {
      const SkSeg sg = seg(k);
      for (int u = sg.klo; u < sg.khi; ++u) {
        mbar_wait(&w_full[s], ph);
        const uint8_t* st = wring + (size_t)s * WSBr;
        // this group's A-stages of the unit go to registers (LG at a time) and the slot goes back to
        // the producer as soon as the last of them is loaded
#pragma unroll
        for (int j0 = 0; j0 < APG; j0 += LG) {
          uint32_t w[LG][WW];
          uint32_t cw[LG][NM];
#pragma unroll
          for (int j = 0; j < LG; ++j) {
            const int col = (g + (j0 + j) * MG) * KA;
#pragma unroll
            for (int c = 0; c < KA / 8; ++c) {
              const uint32_t chunk = (uint32_t)(((col & 63) >> 3) + c) ^ (uint32_t)(m & 7);
              const uint4 v = *reinterpret_cast<const uint4*>(st + (col >> 6) * WBLK + m * 128 + chunk * 16);
              w[j][4 * c] = v.x; w[j][4 * c + 1] = v.y; w[j][4 * c + 2] = v.z; w[j][4 * c + 3] = v.w;
            }
            // the 32-column group's n_m words (swizzled code box: conflict-free reads)
            lds_words_swz<NM>(st + WCODE, (uint32_t)(m * CWORDS * 4 + (col >> 5) * NM * 4), CWORDS * 4, cw[j]);
          }
          if (j0 + LG == APG) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&w_empty[s]);
          }
#pragma unroll
          for (int j = 0; j < LG; ++j, js += MG) {
            const int sa = (js + g) % SA;
            mbar_wait(&a_empty[sa], ((uint32_t)((js + g) / SA) & 1u) ^ 1u);
            tc_fence_after();
            const uint32_t a0 = a_lane + (uint32_t)(sa * SLOT);
            tmem_st_n<WW>(a0, w[j]);
#pragma unroll
            for (int i = 0; i < (MGLU_SK_ABL == 2 ? 0 : NM); ++i) {
              uint32_t op[WW];
              // pair q of the A-stage is pair q0 + q of its 32-column group: bits (q0 + q, q0 + q + 16)
              // of the group's word; shifting the word right by q0 keeps the bits that reach the bf16
              // sign positions exactly those two
              const uint32_t word = cw[j][i] >> (((g + (j0 + j) * MG) * KA & 31) >> 1);
#pragma unroll
              for (int q = 0; q < WW; ++q)
                op[q] = MGLU_SK_ABL == 1 ? (w[j][q] ^ word) : sign_flip(w[j][q], word, 1u << (15 - q));
              tmem_st_n<WW>(a0 + (uint32_t)((1 + i) * WW), op);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_full[sa]);
          }
        }
        if (++s == SW) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp >= kEpi0) {
    // ------------------------------------------------ epilogue: thread = tile row m
    const int quarter = warp & 3;
    const int m = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const int B = p.B;
    const int nch = (B + CH - 1) / CH;
    const size_t slot_f = (size_t)NOP * B * 128;       // floats of one published partial
    pdl_wait();
    int set = 0;
    uint32_t use_a = 0u, use_b = 0u;
    for (int k = 0; k < nseg; ++k) {
      const SkSeg sg = seg(k);
      const int tile = sg.tile;
      const bool shared = sg.shared;
      mbar_wait(&acc_full[set], (set ? use_b : use_a) & 1u);
      tc_fence_after();
      const uint32_t abase = lane_base + (uint32_t)(set * ACC);
      const int grow = sg.row0 + m;
      const bool row_ok = m < sg.rows && grow < p.h;
      // contributors of a shared tile: CTAs [c_lo, c_hi]; this CTA's slot: 0 if the tile is its first
      const int c_lo = shared ? sk_cta_of(p, tile * upt) : cta;
      const int c_hi = shared ? sk_cta_of(p, min((tile + 1) * upt, p.units_base * (int)gridDim.x + p.units_rem) - 1) : cta;
      auto slot_of = [&](int c) { return sk_unit0(p, c) / upt == tile ? 0 : 1; };
      bool last = !shared;
      if (shared) {
        // publish this CTA's partial, then take a ticket
        float* wsp = p.ws + ((size_t)cta * 2 + slot_of(cta)) * slot_f + m;
        for (int ch = 0; ch < nch; ++ch) {
          float v[NOP][CH];
          sk_ld_chunk<NOP, BN, CH>(abase, ch, v);
#pragma unroll
          for (int o = 0; o < NOP; ++o)
#pragma unroll
            for (int q = 0; q < CH; ++q) {
              const int tok = ch * CH + q;
              if (tok < B) __stcg(wsp + ((size_t)o * B + tok) * 128, v[o][q]);
            }
        }
        __threadfence();
        named_bar_sync(15, 128);
        if (warp == kEpi0 && lane == 0) {
          const uint32_t old = atomicAdd(p.tickets + tile, 1u);
          const uint32_t is_last = old == (uint32_t)(c_hi - c_lo) ? 1u : 0u;
          if (is_last) p.tickets[tile] = 0u;              // re-arm for the next call (stream order)
          *last_flag = is_last;
        }
        named_bar_sync(15, 128);
        last = *last_flag != 0u;
        if (last) __threadfence();                          // acquire the other contributors' partials
      }
      if (last) {
        // the row split's final tile is shared out over every lane-owning warp (the maskers are idle
        // by then): this team takes its share of the token chunks
        int ch0 = 0, ch1 = nch;
        if (p.row_mode && k == nseg - 1) { ch0 = MG * nch / (MG + 1); }
        for (int ch = ch0; ch < ch1; ++ch) {
          float f[NOP][CH];
          if (!shared) {
            sk_ld_chunk<NOP, BN, CH>(abase, ch, f);
          } else {
            // every contributor's published partial (this CTA's included), added in CTA order
#pragma unroll
            for (int o = 0; o < NOP; ++o)
#pragma unroll
              for (int q = 0; q < CH; ++q) f[o][q] = 0.f;
            for (int c = c_lo; c <= c_hi; ++c) {
              const float* wsp = p.ws + ((size_t)c * 2 + slot_of(c)) * slot_f + m;
#pragma unroll
              for (int o = 0; o < NOP; ++o)
#pragma unroll
                for (int q = 0; q < CH; ++q) {
                  const int tok = ch * CH + q;
                  if (tok < B) f[o][q] += __ldcg(wsp + ((size_t)o * B + tok) * 128);
                }
            }
          }
          if (row_ok) sk_epi_store<NM, CH>(p, f, ch, grow);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[set]);
      if (set) ++use_b; else ++use_a;
      if (NACC == 2) set ^= 1;
    }
  }
  // row split: the maskers' share of the final tile's epilogue (after their last A-stage)
  if (p.row_mode && warp < 4 * MG && nseg > 0) {
    const int k = nseg - 1;
    const int set = NACC == 2 ? (k & 1) : 0;
    const int quarter = warp & 3, g = warp >> 2;
    const int m = quarter * 32 + lane;
    const int nch = (p.B + CH - 1) / CH;
    pdl_wait();
    mbar_wait(&acc_full[set], (uint32_t)((NACC == 2 ? k >> 1 : k) & 1));
    tc_fence_after();
    const SkSeg sg = seg(k);
    const int grow = sg.row0 + m;
    const uint32_t abase = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(set * ACC);
    for (int ch = g * nch / (MG + 1); ch < (g + 1) * nch / (MG + 1); ++ch) {
      float f[NOP][CH];
      sk_ld_chunk<NOP, BN, CH>(abase, ch, f);
      if (m < sg.rows && grow < p.h) sk_epi_store<NM, CH>(p, f, ch, grow);
    }
    tc_fence_before();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace mglu
