// gemm_tc.cuh -- tcgen05/TMEM masked GEMM: the prefill / large-batch regime.
//
// The paper's kernel is batch 1 only; for B tokens Eq. 3 needs (n_m + 1) GEMMs sharing x:
// t = X Wt^T and, per mask, a masked product.  As in the decode regime the masked operand is the
// sign-flipped weight sigma_i (.) W (sigma = +1 where M_i = 1, -1 where M_i = 0), so the tensor core
// accumulates u_i = s_i - v_i and the epilogue takes s_i = (t + u_i) / 2 (exact rescaling).
//
// One CTA computes a 128-row (h) x BN-token tile over the whole reduction (d).  Operands:
//   * A = the n_m + 1 weight operands {W, sigma_1 (.) W, ...} live in TENSOR MEMORY (TS form): the
//     masker warps read W rows straight from global memory (whole 32-byte sectors per thread),
//     build the sign-flipped rows in registers (one IMAD + one LOP3 per bf16 pair and mask) and
//     tcgen05.st them into a ring of SA TMEM A slots of KA columns of K each.  Shared memory
//     carries only x, so the tensor core is not starved by shared-memory bandwidth (an
//     SS form at N <= 128 needs > 128 B/clk of operand reads).
//   * B = the x tile [BN tokens x 64] (K-major, 128-byte swizzle) staged by TMA in a shared ring.
//   * D = n_m + 1 fp32 accumulators of BN columns each in TMEM:
//     (n_m + 1) * BN + SA * (n_m + 1) * KA / 2 <= 512 columns.
// Warp roles (320 threads): warps 0-7 masker (group g = warp / 4 fills the A slots of the A-stages
// js = g mod 2; warp w owns TMEM lanes 32 (w % 4) .. +31 = tile rows), then epilogue (tcgen05.ld,
// Eq. 3 in registers, bf16 stores; group g takes half the tokens); warp 8 TMA producer; warp 9 MMA
// issuer (warp-uniform loop, one elected lane issues; one a_full wait and one commit per A-stage).
#pragma once
#include "common.cuh"
#include "mma_mask.cuh"
#include "tcgen05.cuh"
#include "tma.cuh"

namespace mglu {

// tile shape per mask count: BN tokens; SA TMEM A slots of KA reduction columns per operand
template <int NM> struct TcCfg;
template <> struct TcCfg<1> { static constexpr int BN = 224, SA = 2, KA = 32; };
template <> struct TcCfg<2> { static constexpr int BN = 128, SA = 2, KA = 32; };
template <> struct TcCfg<4> { static constexpr int BN = 64, SA = 2, KA = 32; };
template <> struct TcCfg<8> { static constexpr int BN = 32, SA = 2, KA = 16; };

constexpr int kTcThreads = 320;
constexpr int kTcMaskWarps = 8;
constexpr int kTcXK = 64;                       // K per x stage (128-byte rows)
constexpr int kTcPrefetch = 2;                  // masker register prefetch depth (A-stages of its group)

template <int NM> __host__ __device__ constexpr int tc_x_stage_bytes() { return TcCfg<NM>::BN * kTcXK * 2; }
template <int NM> __host__ __device__ constexpr int tc_tmem_used() {
  return (NM + 1) * TcCfg<NM>::BN + TcCfg<NM>::SA * (NM + 1) * TcCfg<NM>::KA / 2;
}
static_assert(tc_tmem_used<1>() <= 512 && tc_tmem_used<2>() <= 512 && tc_tmem_used<4>() <= 512 &&
              tc_tmem_used<8>() <= 512, "TMEM budget");

// the n_m code words of one (row, 32-column group), vector loads, L1-allocating
template <int NM> __device__ __forceinline__ void ld_words(const uint32_t* p, uint32_t (&c)[NM]) {
  if constexpr (NM == 1) {
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(c[0]) : "l"(p));
  } else if constexpr (NM == 2) {
    asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(c[0]), "=r"(c[1]) : "l"(p));
  } else if constexpr (NM == 4) {
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]) : "l"(p));
  } else {
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]), "=r"(c[7])
                 : "l"(p));
  }
}

struct TcParams {
  const __nv_bfloat16* Wt;   // [h][d]
  const uint32_t* codes;     // packed mask words (R3 layout)
  __nv_bfloat16* out;        // [B][h]
  int B, d, h;
  int xstages;
};

// Masker group G (0/1) builds the A operands of the A-stages js = G, G + 2, ... (KA columns each)
// for the tile row this thread owns (TMEM lane): W straight from global memory (KA * 2 bytes =
// whole sectors), the row's n_m code words of the 32-column group, n_m sign flips per bf16 pair,
// n_m + 1 tcgen05.st.  A-stage js uses slot js % SA (SA even): each slot belongs to one group,
// which visits its slots in order, so the parity waits can never skip a phase.
template <int NM, int G>
__device__ __forceinline__ void tc_masker(const __nv_bfloat16* wrow, const uint32_t* crow, int nstages,
                                          uint32_t a_lane, uint64_t* a_full, uint64_t* a_empty) {
  constexpr int SA = TcCfg<NM>::SA, KA = TcCfg<NM>::KA;
  constexpr int NOP = NM + 1, WW = KA / 2;                 // u32 words (bf16 pairs) per row and stage
  static_assert(SA % 2 == 0, "A slots must split evenly between the two masker groups");
  static_assert(KA == 32 || KA == 16, "A-stage width");
  constexpr int PAIR0 = KA == 32 ? 0 : 8 * G;              // first pair of the stage in its code group
  uint32_t wb[kTcPrefetch][WW], cb[kTcPrefetch][NM];
  auto fetch = [&](int js, uint32_t (&w)[WW], uint32_t (&c)[NM]) {
    if (js < nstages) {
      ld_nc_v8_na(wrow + KA * js, *reinterpret_cast<uint32_t(*)[8]>(&w[0]));
      if constexpr (WW == 16) ld_nc_v8_na(wrow + KA * js + 16, *reinterpret_cast<uint32_t(*)[8]>(&w[8]));
      ld_words<NM>(crow + (size_t)((KA * js) >> 5) * NM, c);
    }
  };
#pragma unroll
  for (int u = 0; u < kTcPrefetch; ++u) fetch(G + 2 * u, wb[u], cb[u]);
  for (int js0 = G; js0 < nstages; js0 += 2 * kTcPrefetch) {
#pragma unroll
    for (int u = 0; u < kTcPrefetch; ++u) {
      const int js = js0 + 2 * u;
      if (js < nstages) {
        uint32_t a[NOP][WW];
#pragma unroll
        for (int q = 0; q < WW; ++q) a[0][q] = wb[u][q];
#pragma unroll
        for (int i = 0; i < NM; ++i) {
#pragma unroll
          for (int q = 0; q < WW; ++q)                     // pair PAIR0 + q: bits (pair, pair + 16)
            a[1 + i][q] = sign_flip(wb[u][q], cb[u][i], 1u << (15 - PAIR0 - q));
        }
        fetch(js + 2 * kTcPrefetch, wb[u], cb[u]);         // refill this buffer
        const int sa = js % SA;
        mbar_wait(&a_empty[sa], ((uint32_t)(js / SA) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t a0 = a_lane + (uint32_t)(sa * NOP * WW);
#pragma unroll
        for (int op = 0; op < NOP; ++op) {
          if constexpr (WW == 16) tmem_st16(a0 + op * WW, a[op]);
          else tmem_st8(a0 + op * WW, *reinterpret_cast<uint32_t(*)[8]>(&a[op][0]));
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&a_full[sa]);
      }
    }
  }
}

template <int NM, int ACT>
__global__ void __launch_bounds__(kTcThreads, 1)
gemm_tc_kernel(const TcParams p, const __grid_constant__ CUtensorMap mX) {
  constexpr int BN = TcCfg<NM>::BN, SA = TcCfg<NM>::SA, KA = TcCfg<NM>::KA;
  constexpr int NOP = NM + 1;                              // operands: W and n_m sign-flipped copies
  constexpr int XB = tc_x_stage_bytes<NM>();
  constexpr int KPS = KA / 16;                             // k16 steps per A-stage
  constexpr uint32_t IDESC = idesc_bf16_f32(128, BN);
  constexpr uint32_t A_COL0 = NOP * BN;                    // first TMEM column of the A ring
  static_assert((kTcXK / 16) % (KPS * SA) == 0, "the slot pattern repeats within an x stage");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int SX = p.xstages;
  uint8_t* xring = smem;
  uint64_t* x_full = reinterpret_cast<uint64_t*>(smem + (size_t)SX * XB);
  uint64_t* x_empty = x_full + SX;
  uint64_t* a_full = x_empty + SX;
  uint64_t* a_empty = a_full + SA;
  uint64_t* acc_full = a_empty + SA;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * 128;
  const int d = p.d;
  const int nk16 = d >> 4;                                 // d % 32 == 0
  const int nkx = (d + kTcXK - 1) / kTcXK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SX; ++s) { mbar_init(&x_full[s], 1); mbar_init(&x_empty[s], 1); }
    for (int s = 0; s < SA; ++s) { mbar_init(&a_full[s], 128); mbar_init(&a_empty[s], 1); }
    mbar_init(acc_full, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kTcMaskWarps) {
    // ---------------------------------------------------------------- TMA producer (x)
    if (lane == 0) {
      prefetch_tmap(&mX);
      pdl_wait();                                          // x may come from the predecessor
      int s = 0;
      uint32_t ph = 0;
      for (int kx = 0; kx < nkx; ++kx) {
        mbar_wait(&x_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&x_full[s], (uint32_t)XB);
        tma_load_2d(xring + (size_t)s * XB, &mX, kx * kTcXK, n0, &x_full[s]);
        if (++s == SX) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == kTcMaskWarps + 1) {
    // ---------------------------------------------------------------- MMA issuer (whole warp)
    const uint64_t bdesc0 = smem_desc_kmajor(smem_u32(xring), 128);
    int sx = 0;
    uint32_t phx = 0;
    for (int kx = 0; kx < nkx; ++kx) {
      mbar_wait(&x_full[sx], phx);
      tc_fence_after();
      const uint64_t bdesc_s = bdesc0 + (uint64_t)((sx * XB) >> 4);
#pragma unroll
      for (int kk = 0; kk < kTcXK / 16; ++kk) {
        const int j = kx * (kTcXK / 16) + kk;              // k16 step
        if (j < nk16) {
          const int js = j / KPS;                          // A-stage
          const int sa = (kk / KPS) % SA;                  // == js % SA (x stages hold whole slot cycles)
          if (kk % KPS == 0) {
            mbar_wait(&a_full[sa], (uint32_t)(js / SA) & 1u);
            tc_fence_after();
          }
          if (elect_one()) {
            const uint64_t bdesc = bdesc_s + (uint64_t)(kk * 2);          // +32 bytes along K
            const uint32_t a0 = tmem + A_COL0 + (uint32_t)(sa * NOP * (KA / 2) + (kk % KPS) * 8);
            const uint32_t acc = j > 0 ? 1u : 0u;
#pragma unroll
            for (int op = 0; op < NOP; ++op)
              tc_mma_ts(tmem + op * BN, a0 + op * (KA / 2), bdesc, IDESC, acc);
            if (kk % KPS == KPS - 1) tc_commit(&a_empty[sa]);
          }
          __syncwarp();
        }
      }
      if (elect_one()) tc_commit(&x_empty[sx]);
      __syncwarp();
      if (++sx == SX) { sx = 0; phx ^= 1; }
    }
    if (elect_one()) tc_commit(acc_full);
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- masker
    const int g = warp >> 2;
    const int m = (warp & 3) * 32 + lane;                  // tile row = TMEM lane
    const int grow = m0 + m;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    {
      const int mrow = grow < p.h ? grow : p.h - 1;        // rows past h: any valid row, discarded
      const __nv_bfloat16* wrow = p.Wt + (size_t)mrow * d;
      const uint32_t* crow = p.codes + (size_t)mrow * (d / 32) * NM;
      const uint32_t a_lane = tmem + lane_off + A_COL0;
      const int nstages = d / KA;
      if (g == 0)
        tc_masker<NM, 0>(wrow, crow, nstages, a_lane, a_full, a_empty);
      else
        tc_masker<NM, 1>(wrow, crow, nstages, a_lane, a_full, a_empty);
    }

    // ---------------------------------------------------------------- epilogue
    mbar_wait(acc_full, 0);
    tc_fence_after();
    pdl_wait();                                            // out may be read upstream
    const uint32_t lane_base = tmem + lane_off;
    constexpr int HALF = BN / 2;                           // tokens per masker group
    static_assert(HALF % 8 == 0, "BN / 2 must be a multiple of 8");
#pragma unroll 1
    for (int c0 = g * HALF; c0 < (g + 1) * HALF; c0 += 8) {
      uint32_t tv[8], uv[8];
      float y[8];
      tmem_ld8(lane_base + c0, tv);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 8; ++q) y[q] = 0.f;
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        tmem_ld8(lane_base + (1 + i) * BN + c0, uv);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float t = __uint_as_float(tv[q]);
          const float sg = 0.5f * (t + __uint_as_float(uv[q]));           // s_i = (t + u_i) / 2
          y[q] = fmaf(act_g<ACT>(sg), t - sg, y[q]);                      // g(s_i) (t - s_i)
        }
      }
      if (grow < p.h) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int tok = n0 + c0 + q;
          if (tok < p.B) p.out[(size_t)tok * p.h + grow] = __float2bfloat16_rn(y[q]);
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
