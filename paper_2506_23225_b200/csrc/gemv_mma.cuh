// gemv_mma.cuh -- TMA-fed, register-masked tensor-core fused masked GEMV (decode regime, bf16,
// 1 <= B <= 8).  MGLU_PATH_MMA.
//
// The FlashMGLU forward of Alg. 1 for small B, re-designed for sm_100a:
//  * a2: W (rows of Wt) and the packed codes stream HBM -> shared memory exactly once per call
//    (P:245).  Each CTA owns a contiguous range of whole 8-row tiles of Wt (tile-balanced; no
//    split-K across CTAs, no atomics: reading R9), processed in rounds
//    of T = 8, 4, 2 or 1 tiles (full rounds of 8, then the remainder's binary digits); a stage of
//    a round is one 3-D TMA box of W (64-column blocks x 8T rows, 128B-swizzled) plus one box of
//    the codes, landing in a multi-stage mbarrier ring fed by one producer thread.  A consumer
//    warp copies its share of a stage into registers and hands the slot back BEFORE its MMAs:
//    a slot is held only for the shared-memory load latency, so nearly the whole ring is in
//    flight (streaming at HBM rate needs ~130 KB in flight per SM at ~5000-cycle loaded latency,
//    tools/probes/probe_sk.cu; holding slots through the MMAs cost ~15 % of the bandwidth).
//  * a3/a4: 16 consumer warps.  A round of T tiles gives each tile WPT = 16 / T warps, each owning
//    128 columns of every stage: every stage is 16384 elements and every warp's share of it is
//    8 rows x 128 columns in every round, so no round is ragged.  The n_m
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

constexpr int kDecConsumers = 16;                      // consumer warps (4 per SM sub-partition)
constexpr int kDecThreads = (kDecConsumers + 1) * 32;  // + 1 producer warp
constexpr int kDecWBytes = kDecConsumers * 2048;       // W region of a stage slot (16384 bf16)

// mask bytes of one 128-column block of a row: 4 groups x n_m words (TMA box inner span = swizzle span)
template <int NM> __host__ __device__ constexpr int dec_code_span() { return 16 * NM; }   // 0: dense (n_m = 0)
// stage slot = W region + codes region (16384 elements: 128 row-blocks x 16 n_m bytes)
template <int NM> __host__ __device__ constexpr int dec_stage_bytes() { return kDecWBytes + 128 * kDecConsumers * NM; }
// plane-major codes (routed, row f2): a stage holds W and the KSEL selected planes' words only
// (16384 elements x 1 bit = 2 KB per plane)
constexpr int kDecPlaneBytes = 2048;
template <int NM, int KSEL, bool PL> __host__ __device__ constexpr int dec_stage_bytes_pl() {
  return PL ? kDecWBytes + KSEL * kDecPlaneBytes : dec_stage_bytes<NM>();
}

struct DecParams {
  const __nv_bfloat16* x;
  __nv_bfloat16* out;
  const float* G;            // Top-K routed gate weights [B][n_m] (nullptr: plain Eq. 3)
  int variant;               // partial-mask ablation variant (0 = Eq. 3; 1 NG, 2 NV, 3 NM)
  int act;                   // g when the kernel is the kRuntimeAct instantiation
  int B, d, h;
  int tiles_base, tiles_rem; // CTA c < ncta owns tiles_base + (c < tiles_rem) 8-row tiles
  int ncta;                  // CTAs of this pass (the fused FFN grid may be wider: the rest own none)
  int stages;                // ring depth
  int xpar;                  // u32 words per parity array of one token's x in smem (+ pad)
  int l2pf;                  // stages beyond the ring prefetched into L2 once, at the CTA's start
  int light_drop;            // stages fewer in flight for the CTAs owning tiles_base tiles
  float* z;                  // KSEL = -1 instantiation: Alg. 1's z [B][2 n_m][h] (s_i, t - s_i) instead of y
};

// One TMA descriptor pair per round type ti (T = 8 >> ti tiles of 8 rows, WPT = 2 << ti warps per
// tile, stage width KS = 256 << ti columns): W boxes of 64 columns x 8T rows x 2 WPT blocks
// (SW128) and code boxes of 16 n_m bytes x 8T rows x WPT blocks.  Every stage of every round type
// is the same 8T x KS = 16384 elements, so every stage slot is exactly full.
struct DecMaps {
  CUtensorMap w[4];
  CUtensorMap c[4];
};

// Top-K routed forward: the masks some token of the batch selected (nonzero G), at most KSEL of
// them, lowest index first, in slots 0..nsel-1; unused slots repeat slot 0 (static register
// indexing: __fns finds the bit, no local-memory array)
template <int NM, int KSEL>
__device__ __forceinline__ int dec_select(const float* G, int B, int (&sel)[KSEL]) {
  uint32_t active = 0u;
  for (int q = 0; q < B * NM; ++q) active |= (G[q] != 0.0f ? 1u : 0u) << (q % NM);
  const int nsel = min(__popc(active), KSEL);
#pragma unroll
  for (int k = 0; k < KSEL; ++k) sel[k] = k < nsel ? (int)__fns(active, 0, k + 1) : 0;
#pragma unroll
  for (int k = 0; k < KSEL; ++k)
    if (k >= nsel) sel[k] = sel[0];
  return nsel;
}

// swizzled byte offset within a 1024-aligned region of `rb`-byte rows (rb in {16..128})
__device__ __forceinline__ uint32_t swz(uint32_t lin, uint32_t rb) {
  return lin ^ (((lin >> 7) & (rb / 16 - 1)) << 4);
}

// stages of one round of type ti over a reduction of d columns
__host__ __device__ __forceinline__ int dec_round_stages(int ti, int d) { return (d + (256 << ti) - 1) >> (8 + ti); }

// Round schedule of a CTA owning `ntiles` 8-row tiles: ntiles / 8 full rounds (ti = 0), then one
// round per set bit of ntiles % 8, largest first (4 tiles: ti = 1, 2: ti = 2, 1: ti = 3).  Every
// round keeps all 16 consumer warps on 8 rows x 128 columns per stage, so per-warp work is the
// same in every round (no ragged round).  Stage i -> (round type, first row of the round, stage
// within the round).
__device__ __forceinline__ void dec_stage_of(int i, int nfull, int rem, int d, int& ti, int& row0, int& ks) {
  const int n0 = dec_round_stages(0, d);
  if (i < nfull * n0) {
    const int r = i / n0;
    ti = 0; row0 = 64 * r; ks = i - r * n0;
    return;
  }
  int j = i - nfull * n0;
  row0 = 64 * nfull;
  ti = 3; ks = j;
#pragma unroll
  for (int b = 2; b >= 0; --b) {
    if (!((rem >> b) & 1)) continue;
    const int t = 3 - b, n = dec_round_stages(t, d);
    if (j < n) { ti = t; ks = j; return; }
    j -= n;
    row0 += 8 << b;
  }
}

// PL (routed only, KSEL > 0): the codes are PLANE-MAJOR -- plane i is [h][d/32] words, the same
// pair-split bit order within a word (mglu_pack_planes_*) -- and a stage loads only the planes the
// batch selected, so a routed call reads W plus K (not n_m) bits per element (row f2).
// maps.c[ti] then views the planes as one [n_m h][d/32] word tensor with boxes of 8T rows x KS/32
// words; the selection needs G, so this producer starts after griddepcontrol.wait.
// a CTA's share of a layer: whole 8-row tiles [tile0, tile0 + ntiles) processed in rounds
struct DecGeo {
  int r0, nrows, nfull, rem, nstages, d;
};
__device__ __forceinline__ DecGeo dec_geo(const DecParams& p, int cta) {
  DecGeo g;
  const int tile0 = cta * p.tiles_base + min(cta, p.tiles_rem);
  const int ntiles = cta < p.ncta ? p.tiles_base + (cta < p.tiles_rem ? 1 : 0) : 0;
  g.r0 = 8 * tile0;
  g.nrows = min(8 * ntiles, p.h - g.r0);
  g.d = p.d;
  g.nfull = ntiles >> 3;
  g.rem = ntiles & 7;
  g.nstages = g.nfull * dec_round_stages(0, g.d);
#pragma unroll
  for (int b = 0; b < 3; ++b)
    if ((g.rem >> b) & 1) g.nstages += dec_round_stages(3 - b, g.d);
  return g;
}

// one thread: the TMA producer of the CTA's stages (ring position s / ph carried across calls:
// the fused FFN kernel streams its two phases through one ring)
template <int NM, int ACT, int NB, int KSEL, bool PL, int SB>
__device__ __forceinline__ void dec_produce(const DecParams& p, const DecMaps& maps, uint8_t* ring, uint64_t* full,
                                            uint64_t* empty, int S, const DecGeo& geo, int& s, uint32_t& ph) {
  static_assert(!PL || KSEL > 0, "plane-major codes: routed calls only");
  constexpr int SPAN = dec_code_span<NM>();
  constexpr int NACC = NB * ((KSEL > 0 ? KSEL : NM) + 1);
  (void)SPAN; (void)NACC;
  const int r0 = geo.r0, nrows = geo.nrows, nfull = geo.nfull, rem = geo.rem, nstages = geo.nstages, d = geo.d;
  (void)nrows; (void)nstages;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      prefetch_tmap(&maps.w[t]);
      if (NM > 0) prefetch_tmap(&maps.c[t]);
    }
    const uint64_t pol = policy_evict_first();
    int psel[PL ? KSEL : 1];
    int pn = 0;
    if constexpr (PL) {
      // the ring's first stages of W (constant weights) stream before the PDL wait: their
      // barriers expect the W bytes now, the selected planes' bytes and the arrival after it
      const int pre = min(S, nstages);
      for (int i = 0; i < pre; ++i) {
        int ti, row0, ks;
        dec_stage_of(i, nfull, rem, d, ti, row0, ks);
        mbar_expect_tx(&full[i], (uint32_t)(16384 * 2));
        tma_load_3d_hint(ring + (size_t)i * SB, &maps.w[ti], 0, r0 + row0, ks * (256 << ti) / 64, &full[i], pol);
      }
      pdl_wait();                                          // G comes from the router launch
      pn = dec_select<NM, KSEL>(p.G, p.B, psel);
      for (int i = 0; i < pre; ++i) {
        int ti, row0, ks;
        dec_stage_of(i, nfull, rem, d, ti, row0, ks);
        mbar_arrive_expect_tx(&full[i], (uint32_t)(pn * kDecPlaneBytes));
#pragma unroll
        for (int k = 0; k < KSEL; ++k)
          if (k < pn) tma_load_2d_hint(ring + (size_t)i * SB + kDecWBytes + k * kDecPlaneBytes, &maps.c[ti],
                                       ks * (256 << ti) / 32, psel[k] * p.h + r0 + row0, &full[i], pol);
      }
    }
    for (int i = 0; i < nstages; ++i) {
      int ti, row0, ks;
      dec_stage_of(i, nfull, rem, d, ti, row0, ks);
      const int k0 = ks * (256 << ti);
      if constexpr (PL) {
        if (i < S) { if (++s == S) { s = 0; ph ^= 1; } continue; }   // issued above
      }
      mbar_wait(&empty[s], ph ^ 1);
      uint8_t* wst = ring + (size_t)s * SB;
      if constexpr (PL) {
        // W + the selected planes' words of the stage's rows (8T rows x KS/32 words each)
        mbar_arrive_expect_tx(&full[s], (uint32_t)(16384 * 2 + pn * kDecPlaneBytes));
        tma_load_3d_hint(wst, &maps.w[ti], 0, r0 + row0, k0 / 64, &full[s], pol);
#pragma unroll
        for (int k = 0; k < KSEL; ++k)
          if (k < pn) tma_load_2d_hint(wst + kDecWBytes + k * kDecPlaneBytes, &maps.c[ti], k0 / 32,
                                       psel[k] * p.h + r0 + row0, &full[s], pol);
        if (++s == S) { s = 0; ph ^= 1; }
        continue;
      }
      mbar_arrive_expect_tx(&full[s], (uint32_t)(16384 * 2 + 16384 / 128 * SPAN));
      tma_load_3d_hint(wst, &maps.w[ti], 0, r0 + row0, k0 / 64, &full[s], pol);
      if constexpr (NM > 0) tma_load_3d_hint(wst + kDecWBytes, &maps.c[ti], 0, r0 + row0, k0 / 128, &full[s], pol);
      if (i == S - 1) {
        // ring filled: the next l2pf stages go to L2 once, so HBM keeps streaming while the
        // consumers wait for the previous grid (PDL) and for x
        for (int f = S; f < min(nstages, S + p.l2pf); ++f) {
          int fti, frow, fks;
          dec_stage_of(f, nfull, rem, d, fti, frow, fks);
          const int fk0 = fks * (256 << fti);
          tma_prefetch_3d(&maps.w[fti], 0, r0 + frow, fk0 / 64);
          if constexpr (NM > 0) tma_prefetch_3d(&maps.c[fti], 0, r0 + frow, fk0 / 128);
        }
      }
      if (++s == S) { s = 0; ph ^= 1; }
    }
}

// the 16 consumer warps: x staging, the rounds of MMAs over the stages, the epilogue
template <int NM, int ACT, int NB, int KSEL, bool PL, int SB>
__device__ __forceinline__ void dec_consume(const DecParams& p, uint8_t* ring, uint64_t* full, uint64_t* empty,
                                            float* part, uint32_t* xs, int S, const DecGeo& geo, int& s, uint32_t& ph) {
  static_assert(!PL || KSEL > 0, "plane-major codes: routed calls only");
  constexpr int SPAN = dec_code_span<NM>();
  constexpr int NACC = NB * ((KSEL > 0 ? KSEL : NM) + 1);
  (void)SPAN; (void)NACC;
  // 32-column steps loaded per register group: all 4 of a stage, or 2 / 1 where the staged
  // operands would not fit beside the accumulators (n_m = 8; two token groups with n_m >= 4).
  // (17 warps per CTA leave 96 registers per thread: one SM sub-partition holds 5 of them.)
  constexpr int kGrp = (NB == 2 && (KSEL > 0 ? KSEL : NM) >= 4) ? 1 : ((KSEL > 0 ? KSEL : NM) * NB > 4) ? 2 : 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = geo.r0, nrows = geo.nrows, nfull = geo.nfull, rem = geo.rem, nstages = geo.nstages, d = geo.d;
  (void)nrows; (void)nstages;
  const int g = lane >> 2, c = lane & 3;
  const int B = p.B;
  const int prow = (g >> 1) + 4 * (g & 1);                 // pi(g): tile-local real row
  // pair q of this thread's 8 columns = group columns 8c + 2q, 8c + 2q + 1 -> layout bits
  // 4c + q and 16 + 4c + q; multiplying by 2^(15 - 4c - q) moves them to bits 15 and 31
  uint32_t mul[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) mul[q] = 1u << (15 - 4 * c - q);

  // x -> smem split by bf16-pair parity: xs[2b + parity][pair / 2], zero-padded past d.  MMA
  // columns of tokens >= B read token 0's row: their D columns are never used (finite either way).
  // The zero fill does not depend on the predecessor grid and runs before the PDL wait; x itself
  // is one 16-byte load per 8 columns, all of a thread's loads in flight together.
  const int ctid = threadIdx.x;                             // consumer thread 0..511
  constexpr int kCT = kDecConsumers * 32;
  const int dw = d / 4;                                     // u32 words of one parity array
  {
    const int padw = p.xpar - dw;
    for (int v = ctid; v < 2 * B * padw; v += kCT) {
      const int a = v / padw;
      xs[(size_t)a * p.xpar + dw + (v - a * padw)] = 0u;
    }
  }
#ifndef MGLU_ABL_NOPDLWAIT  // timing ablation (unsafe ordering): do not wait for the previous grid
  pdl_wait();                                              // x is the predecessor's output
#endif
  {
    const int nvec = d / 8;                                 // 16-byte vectors per token
    const int total = B * nvec;
    for (int base = ctid; base < total; base += 4 * kCT) {
      uint4 u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int v = base + q * kCT;
        if (v < total) {
          const int b = v / nvec, e = v - b * nvec;
          u[q] = *reinterpret_cast<const uint4*>(p.x + (size_t)b * d + 8 * e);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int v = base + q * kCT;
        if (v < total) {
          const int b = v / nvec, e = v - b * nvec;
          // pairs 4e .. 4e+3: even pairs (4e, 4e+2) -> words 2e, 2e+1 of parity 0, odd -> parity 1
          *reinterpret_cast<uint2*>(xs + (size_t)(2 * b) * p.xpar + 2 * e) = make_uint2(u[q].x, u[q].z);
          *reinterpret_cast<uint2*>(xs + (size_t)(2 * b + 1) * p.xpar + 2 * e) = make_uint2(u[q].y, u[q].w);
        }
      }
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
  int nsel = NSLOT;
  if constexpr (KSEL > 0) {
    nsel = dec_select<NM, KSEL>(p.G, B, sel);
    valid = (1u << nsel) - 1u;
  }
  named_bar_sync(1, kDecConsumers * 32);

  float acc[NB][NSLOT + 1][4];   // [0] = t; NM = 0 (dense projection): t only
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
#pragma unroll
    for (int a = 0; a <= NSLOT; ++a)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[nb][a][v] = 0.f;

  int row0 = 0;
  const int nrounds = nfull + __popc(rem);
  for (int rho = 0; rho < nrounds; ++rho) {
    // round type: full rounds first, then the remainder's set bits, largest first
    int ti = 0;
    if (rho >= nfull) {
      int k = rho - nfull;
#pragma unroll
      for (int b = 2; b >= 0; --b)
        if ((rem >> b) & 1) { if (k == 0) { ti = 3 - b; break; } --k; }
    }
    const int rows = 64 >> ti;
    const int wpt = 2 << ti;
    const int nks = dec_round_stages(ti, d);
    const int tl = warp / wpt, kp = warp - tl * wpt;        // tile and column part of this warp
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
    if constexpr (PL) {
      // plane box of slot k (slots past nsel reuse slot 0's plane): row srow, word kp * 4 + st
#pragma unroll
      for (int k = 0; k < KSEL; ++k)
#pragma unroll
        for (int st = 0; st < 4; ++st)
          csel[k][st] = (uint32_t)(kDecWBytes + (k < nsel ? k : 0) * kDecPlaneBytes + srow * (32 << ti) + (kp * 4 + st) * 4);
    } else if constexpr (KSEL > 0) {
#pragma unroll
      for (int k = 0; k < KSEL; ++k)
#pragma unroll
        for (int st = 0; st < 4; ++st)
          csel[k][st] = (uint32_t)kDecWBytes + swz((uint32_t)((kp * rows + srow) * SPAN + (st * NM + sel[k]) * 4), SPAN);
    }
    // x: word index of pair 4c of step 0 of stage 0 for this lane's token column (tokens >= B: 0)
    uint32_t xoff[NB];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const int tok = nb * 4 + (g >> 1) < B ? nb * 4 + (g >> 1) : 0;
      xoff[nb] = (uint32_t)((2 * tok + (g & 1)) * p.xpar + kp * 32 + 2 * c) * 4u;
    }
    for (int ks = 0; ks < nks; ++ks) {
      mbar_wait(&full[s], ph);
      // operands go to registers first and the slot goes back to the producer before the last
      // group's MMAs: a slot is held only for the shared-memory load latency (plus, where
      // registers force two load groups, the first group's MMAs), so nearly the whole ring stays
      // in flight (the HBM stream needs ~130+ KB in flight per SM)
      // slot base as a provably warp-uniform value: the LDS addresses become [per-thread + uniform]
      const uint8_t* wst = ring + __shfl_sync(0xffffffffu, s * SB, 0);
      const uint8_t* xst = reinterpret_cast<const uint8_t*>(xs) + __shfl_sync(0xffffffffu, ks * wpt * 128, 0);
#pragma unroll
      for (int g0 = 0; g0 < 4; g0 += kGrp) {
        uint4 wq[kGrp];
        uint32_t mw[kGrp][NSLOT > 0 ? NSLOT : 1];
        uint32_t xb[kGrp][NB][2];
#pragma unroll
        for (int j = 0; j < kGrp; ++j) {
          const int st = g0 + j;
          wq[j] = *reinterpret_cast<const uint4*>(wst + woff[st]);
          if constexpr (KSEL > 0) {
#pragma unroll
            for (int k = 0; k < KSEL; ++k) mw[j][k] = *reinterpret_cast<const uint32_t*>(wst + csel[k][st]);
          } else if constexpr (NM > 0) {
#pragma unroll
            for (int q = 0; q < (NM + 3) / 4; ++q) {
              // n_m = 8: the second 16-byte chunk is the next one in the swizzled span
              const uint8_t* cp = wst + (q == 0 ? coff[st] : (coff[st] ^ 16u));
              if constexpr (NM == 1) mw[j][0] = *reinterpret_cast<const uint32_t*>(cp);
              else if constexpr (NM == 2) { const uint2 u = *reinterpret_cast<const uint2*>(cp); mw[j][0] = u.x; mw[j][1] = u.y; }
              else {
                const uint4 u = *reinterpret_cast<const uint4*>(cp);
                mw[j][4 * q] = u.x; mw[j][4 * q + 1] = u.y; mw[j][4 * q + 2] = u.z; mw[j][4 * q + 3] = u.w;
              }
            }
          }
          // B: x pairs (4c + parity, 4c + 2 + parity) of the step for this lane's column(s)
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            const uint2 u = *reinterpret_cast<const uint2*>(xst + xoff[nb] + st * 32);
            xb[j][nb][0] = u.x; xb[j][nb][1] = u.y;
          }
        }
        if (g0 + kGrp == 4) {                                 // the stage's last loads are issued
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
#pragma unroll
        for (int j = 0; j < kGrp; ++j) {
#ifdef MGLU_ABL_NOMMA   // timing ablation (wrong results): operands loaded, no tensor-core work
          acc[0][0][0] += __uint_as_float(wq[j].x ^ wq[j].y ^ wq[j].z ^ wq[j].w ^ mw[j][0] ^ xb[j][0][0] ^ xb[j][0][1]);
          continue;
#endif
          // t += x W
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) mma_16816(acc[nb][0], wq[j].x, wq[j].y, wq[j].z, wq[j].w, xb[j][nb][0], xb[j][nb][1]);
#ifdef MGLU_ABL_NOMASK  // timing ablation (wrong results): t only
          acc[0][1][0] += __uint_as_float(mw[j][0] ^ mw[j][NSLOT - 1]);
          continue;
#endif
          // u_i += x (sigma_i (.) W): pair q of the thread's 8 columns is register q of the quad
#pragma unroll
          for (int ii = 0; ii < NSLOT; ++ii) {
            const uint32_t a0 = sign_flip(wq[j].x, mw[j][ii], mul[0]), a1 = sign_flip(wq[j].y, mw[j][ii], mul[1]);
            const uint32_t a2 = sign_flip(wq[j].z, mw[j][ii], mul[2]), a3 = sign_flip(wq[j].w, mw[j][ii], mul[3]);
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) mma_16816(acc[nb][1 + ii], a0, a1, a2, a3, xb[j][nb][0], xb[j][nb][1]);
          }
        }
      }
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
    if (kp > 0) {
      float* pw = part + ((size_t)warp * 32 + lane) * NACC;
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int a = 0; a <= NSLOT; ++a) pw[nb * (NSLOT + 1) + a] = v[nb][a];
    }
    named_bar_sync(1, kDecConsumers * 32);                  // the producer keeps streaming meanwhile
    if (kp == 0) {
      for (int q = 1; q < wpt; ++q) {
        const float* pq = part + ((size_t)(warp + q) * 32 + lane) * NACC;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int a = 0; a <= NSLOT; ++a) v[nb][a] += pq[nb * (NSLOT + 1) + a];
      }
      const int row = row0 + tl * 8 + prow;
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const int tok = nb * 4 + c;
        if (tok < B && row < nrows) {
          float sv[NSLOT > 0 ? NSLOT : 1];
#pragma unroll
          for (int ii = 0; ii < NSLOT; ++ii) sv[ii] = 0.5f * (v[nb][0] + v[nb][1 + ii]);   // s_i = (t + u_i) / 2
          if constexpr (KSEL < 0) {                        // partials instantiation (debug / parity of a5, a6)
            float* zt = p.z + (size_t)tok * 2 * NM * p.h + r0 + row;
#pragma unroll
            for (int ii = 0; ii < NM; ++ii) {
              zt[(size_t)ii * p.h] = sv[ii];
              zt[(size_t)(NM + ii) * p.h] = v[nb][0] - sv[ii];
            }
            continue;
          }
          float y;
          if constexpr (NM == 0) {
            y = v[nb][0];                                   // dense projection x W (FFN W_o, row f1)
          } else if constexpr (KSEL > 0) {                         // routed: slot k is mask sel[k], weight G
            y = 0.f;
            const float* gw = p.G + (size_t)tok * NM;
#pragma unroll
            for (int k = 0; k < KSEL; ++k)
              if ((valid >> k) & 1u) y = fmaf(gw[sel[k]] * act_fast<ACT>(sv[k], p.act), v[nb][0] - sv[k], y);
          } else {
            y = mglu_epilogue_v<ACT, NM, true>(v[nb][0], sv, p.G ? p.G + (size_t)tok * NM : nullptr, p.variant, p.act);   // Eq. 3 / routed / variant
          }
          p.out[(size_t)tok * p.h + r0 + row] = __float2bfloat16_rn(y);
        }
      }
    }
    named_bar_sync(1, kDecConsumers * 32);                  // partials are rewritten next round
    row0 += rows;
  }
}

template <int NM, int ACT, int NB, int KSEL, bool PL = false>
__global__ void __launch_bounds__(kDecThreads, 1)
gemv_mma_kernel(const DecParams p, const __grid_constant__ DecMaps maps) {
  constexpr int SB = dec_stage_bytes_pl<NM, KSEL, PL>();
  constexpr int NACC = NB * ((KSEL > 0 ? KSEL : NM) + 1);
  extern __shared__ __align__(1024) uint8_t smem[];
  // ring depth: the CTAs owning one tile more than the others keep one stage more in flight, so
  // their share of the HBM bandwidth grows with their work and they do not finish last (the next
  // call's consumers wait for this grid's last CTA)
  const int S = (p.tiles_rem && (int)blockIdx.x >= p.tiles_rem) ? p.stages - p.light_drop : p.stages;
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * SB);
  uint64_t* empty = full + S;
  float* part = reinterpret_cast<float*>(empty + S);     // [16 warps][32 lanes][NACC]
  uint32_t* xs = reinterpret_cast<uint32_t*>(part + kDecConsumers * 32 * NACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kDecConsumers);
    }
    mbar_fence_init();
  }
  __syncthreads();
  pdl_launch_dependents();

  const DecGeo geo = dec_geo(p, blockIdx.x);
  if (warp == kDecConsumers) {
    int s = 0;
    uint32_t ph = 0;
    if (lane == 0) dec_produce<NM, ACT, NB, KSEL, PL, SB>(p, maps, ring, full, empty, S, geo, s, ph);
    return;
  }
  int s = 0;
  uint32_t ph = 0;
  dec_consume<NM, ACT, NB, KSEL, PL, SB>(p, ring, full, empty, part, xs, S, geo, s, ph);
}

// ---------------------------------------------------------------------------------------------
// Row f1, fused: the SwiMGLU FFN block FFN(x) = MGLU(x) W_o^T (reading R19) in ONE launch.
// Phase 1 is the decode kernel above over the up-projection's rows (y = MGLU(x), bf16, to `p1.out`);
// phase 2 the same kernel's dense form (n_m = 0) over W_o's rows with x = y.  Both phases stream
// through ONE ring: the producer issues W_o's stages right after the up-projection's, so while the
// consumers wait at the grid barrier (every CTA's y slice written) the ring fills with W_o and the
// HBM stream never stops at the layer boundary -- the part a two-launch composition loses (the
// dependent grid cannot start streaming until the first grid's CTAs leave the SMs).  y makes one
// round trip through L2 (B h bf16 values); the grid barrier needs all CTAs resident (cooperative
// launch, one CTA per SM) and resets itself (sense reversal), so repeats and graph replays work.
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// one thread per CTA; bar[0] = arrivals, bar[1] = generation (both 0 at allocation)
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nctas) {
  const unsigned gen = ld_acquire_gpu(bar + 1);
  __threadfence();
  if (atomicAdd(bar, 1u) == nctas - 1u) {
    atomicExch(bar, 0u);
    __threadfence();
    atomicAdd(bar + 1, 1u);                                 // release the waiters
  } else {
    while (ld_acquire_gpu(bar + 1) == gen) __nanosleep(64);
  }
  __threadfence();
}

template <int NM, int ACT>
__global__ void __launch_bounds__(kDecThreads, 1)
ffn_mma_kernel(const DecParams p1, const __grid_constant__ DecMaps m1, const DecParams p2,
               const __grid_constant__ DecMaps m2, unsigned* gbar) {
  constexpr int SB = dec_stage_bytes<NM>();                 // W_o stages use the same slots
  constexpr int NACC = NM + 1;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int S = p1.stages;
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * SB);
  uint64_t* empty = full + S;
  float* part = reinterpret_cast<float*>(empty + S);
  uint32_t* xs = reinterpret_cast<uint32_t*>(part + kDecConsumers * 32 * NACC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kDecConsumers);
    }
    mbar_fence_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  const DecGeo g1 = dec_geo(p1, blockIdx.x), g2 = dec_geo(p2, blockIdx.x);
  if (warp == kDecConsumers) {
    int s = 0;
    uint32_t ph = 0;
    if (lane == 0) {
      dec_produce<NM, ACT, 1, 0, false, SB>(p1, m1, ring, full, empty, S, g1, s, ph);
      dec_produce<0, kIdentity, 1, 0, false, SB>(p2, m2, ring, full, empty, S, g2, s, ph);
    }
    return;
  }
  int s = 0;
  uint32_t ph = 0;
  dec_consume<NM, ACT, 1, 0, false, SB>(p1, ring, full, empty, part, xs, S, g1, s, ph);
  __threadfence();                                          // this CTA's y slice -> visible
  named_bar_sync(1, kDecConsumers * 32);
  if (threadIdx.x == 0) grid_barrier(gbar, gridDim.x);
  named_bar_sync(1, kDecConsumers * 32);
  dec_consume<0, kIdentity, 1, 0, false, SB>(p2, ring, full, empty, part, xs, S, g2, s, ph);
}

}  // namespace mglu
