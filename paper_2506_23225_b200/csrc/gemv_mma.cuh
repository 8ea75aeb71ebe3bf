// gemv_mma.cuh -- register-masked tensor-core fused masked GEMV (decode regime, bf16, B <= 8).
//
// The FlashMGLU forward of Alg. 1 for small B, re-designed for sm_100a:
//  * a2: W (Wt rows) and the packed codes stream HBM -> registers exactly once per call (P:245,
//    P:435) with 256-bit / 64-bit coalesced L1-bypassing loads; each CTA owns a contiguous,
//    byte-balanced range of Wt rows (no split-K across CTAs, no atomics: reading R9);
//  * a3/a4: instead of per-element predicated adds, the n_m masked operands M_i (.) W are built
//    in registers (one PRMT sign-replicate + one LOP3 per bf16 pair and mask) and fed, with the
//    unmasked W, to mma.sync m16n8k16 (bf16 in, fp32 accumulate), x being the B operand.  So
//    t = x W and s_i = x (M_i (.) W) are accumulated in one pass; the products are
//    exact in fp32 and the 8-token N dimension serves B <= 8 at the same ALU cost;
//  * a5: the K range of a 16-row tile is split across the CTA's warps and reduced through shared
//    memory in a fixed order (deterministic), then
//  * a6/a7: value_i = t - s_i and y = sum_i g(s_i) value_i (Eq. 3) are applied on chip and
//    y is stored once as bf16.
//
// Logical/physical K permutation: the reduction order over k is free, so each thread loads 16
// contiguous elements per row (one 32-byte load) and feeds them to four k16 MMA steps; x is read
// with the same permutation, so every product W[j,k] x[k] is formed with the same k.
#pragma once
#include "common.cuh"

namespace mglu {

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

__device__ __forceinline__ void mma_16816(float (&acc)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// 32-bit AND-mask for the bf16 pair (elements 2Q, 2Q+1 of a thread's 16) under mask I (0-based):
// low half = 0xffff iff bit I of code(2Q), high half = 0xffff iff bit I of code(2Q+1).
// Codes of the 16 elements form a 16*NM-bit string cw[] (element e, mask I at bit NM*e + I).
// Shift the bit to the MSB of its byte, then PRMT with sign-replicate selectors (bit 3 of each
// selector nibble) copies that MSB over two bytes.
template <int NM, int Q, int I>
__device__ __forceinline__ uint32_t mask_word(const uint32_t* cw) {
  constexpr int b0 = NM * (2 * Q) + I, b1 = NM * (2 * Q + 1) + I;
  constexpr int w0 = b0 >> 5, w1 = b1 >> 5;
  constexpr int sh0 = 7 - (b0 & 7), sh1 = 7 - (b1 & 7);
  constexpr uint32_t y0 = (b0 & 31) >> 3, y1 = (b1 & 31) >> 3;
  constexpr uint32_t sel = (8u | y0) | ((8u | y0) << 4) | ((12u | y1) << 8) | ((12u | y1) << 12);
  return prmt(cw[w0] << sh0, cw[w1] << sh1, sel);
}

constexpr int kCodeWords(int nm) { return nm >= 2 ? nm / 2 : 1; }   // u32 words of 16 codes

struct MmaStage {
  uint32_t wa[8], wb[8];   // 16 bf16 of rows r and r+8 (pairs)
  uint32_t ca[4], cb[4];   // their 16 codes (16*NM bits)
};

template <int NM>
__device__ __forceinline__ void load_codes16(const uint8_t* p, uint32_t (&c)[4]) {
  if constexpr (NM == 1) { c[0] = ld_nc_u16(p); }
  else if constexpr (NM == 2) { c[0] = ld_nc_u32(p); }
  else if constexpr (NM == 4) { uint2 v = ld_nc_v2(p); c[0] = v.x; c[1] = v.y; }
  else { uint4 v = ld_nc_v4(p); c[0] = v.x; c[1] = v.y; c[2] = v.z; c[3] = v.w; }
}

__device__ __forceinline__ void ld_nc_v8(const void* p, uint32_t (&w)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}

struct MmaParams {
  const __nv_bfloat16* x;
  const __nv_bfloat16* Wt;
  const uint8_t* codes;
  __nv_bfloat16* out;
  int B, d, h;
  int rows_base, rows_rem;   // CTA c owns rows_base + (c < rows_rem) rows
  int wk_log2;               // K-split: WK = 1 << wk_log2 warps share a tile, WM = 16 / WK
  int Bp;                    // tokens padded to 1/2/4/8 (partials layout)
};

constexpr int kMmaWarps = 16;

template <int NM, int ACT>
__global__ void __launch_bounds__(kMmaWarps * 32, 1)
gemv_mma_kernel(const MmaParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, c = lane & 3;
  const int WK = 1 << p.wk_log2, WM = kMmaWarps >> p.wk_log2;
  const int wk = warp & (WK - 1), wm = warp >> p.wk_log2;
  const int d = p.d, B = p.B, Bp = p.Bp;
  const int cta = blockIdx.x;
  const int r0 = cta * p.rows_base + min(cta, p.rows_rem);
  const int nrows = p.rows_base + (cta < p.rows_rem ? 1 : 0);
  const int ntiles = (nrows + 15) >> 4;
  const int rounds = (ntiles + WM - 1) / WM;
  const int nch = d >> 6;              // 64-element chunks per row (d % 64 == 0 on this path)
  const int nkw = nch >> p.wk_log2;    // chunks per warp per tile
  const int n_items = rounds * nkw;

  const int xstride = d + 8;                                       // padded smem row (bf16)
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(smem);
  float* part = reinterpret_cast<float*>(smem + (size_t)Bp * xstride * 2);
  // part[wm][wk][a][16 rows][Bp]
  const int part_acc_stride = 16 * Bp;
  const int part_warp_stride = (NM + 1) * part_acc_stride;

  auto item_tile = [&](int i) { return (i / nkw) * WM + wm; };
  auto item_kc = [&](int i) { return wk * nkw + (i % nkw); };

  auto load_stage = [&](MmaStage& s, int i) {
    const int tile = item_tile(i);
    const int kc = item_kc(i);
    const int k = (kc << 6) + (c << 4);
    const int ra = tile * 16 + r, rb = ra + 8;                  // rows within the CTA range
    if (tile < ntiles && ra < nrows) {
      const size_t e = (size_t)(r0 + ra) * d + k;
      ld_nc_v8(p.Wt + e, s.wa);
      load_codes16<NM>(p.codes + e * NM / 8, s.ca);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) s.wa[q] = 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) s.ca[q] = 0u;
    }
    if (tile < ntiles && rb < nrows) {
      const size_t e = (size_t)(r0 + rb) * d + k;
      ld_nc_v8(p.Wt + e, s.wb);
      load_codes16<NM>(p.codes + e * NM / 8, s.cb);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) s.wb[q] = 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) s.cb[q] = 0u;
    }
  };

  float acc[NM + 1][4];
#pragma unroll
  for (int a = 0; a <= NM; ++a)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[a][v] = 0.f;

  auto compute = [&](const MmaStage& s, int i) {
    const int kc = item_kc(i);
    uint32_t xr[8];
    if (r < B) {
      const uint4* xp = reinterpret_cast<const uint4*>(xs + (size_t)r * xstride + (kc << 6) + (c << 4));
      const uint4 x0 = xp[0], x1 = xp[1];
      xr[0] = x0.x; xr[1] = x0.y; xr[2] = x0.z; xr[3] = x0.w;
      xr[4] = x1.x; xr[5] = x1.y; xr[6] = x1.z; xr[7] = x1.w;
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) xr[q] = 0u;
    }
    // t += x W  (unmasked operand)
#pragma unroll
    for (int st = 0; st < 4; ++st)
      mma_16816(acc[0], s.wa[2 * st], s.wb[2 * st], s.wa[2 * st + 1], s.wb[2 * st + 1], xr[2 * st], xr[2 * st + 1]);
    // s_i += x (M_i (.) W)
#define MGLU_MASKED_STEP(ST, I)                                                                 \
    mma_16816(acc[1 + I],                                                                       \
              s.wa[2 * ST] & mask_word<NM, 2 * ST, I>(s.ca),                                    \
              s.wb[2 * ST] & mask_word<NM, 2 * ST, I>(s.cb),                                    \
              s.wa[2 * ST + 1] & mask_word<NM, 2 * ST + 1, I>(s.ca),                            \
              s.wb[2 * ST + 1] & mask_word<NM, 2 * ST + 1, I>(s.cb), xr[2 * ST], xr[2 * ST + 1]);
#define MGLU_MASKED_ALL_STEPS(I) \
    if constexpr (I < NM) { MGLU_MASKED_STEP(0, I) MGLU_MASKED_STEP(1, I) MGLU_MASKED_STEP(2, I) MGLU_MASKED_STEP(3, I) }
    MGLU_MASKED_ALL_STEPS(0)
    MGLU_MASKED_ALL_STEPS(1)
    MGLU_MASKED_ALL_STEPS(2)
    MGLU_MASKED_ALL_STEPS(3)
    MGLU_MASKED_ALL_STEPS(4)
    MGLU_MASKED_ALL_STEPS(5)
    MGLU_MASKED_ALL_STEPS(6)
    MGLU_MASKED_ALL_STEPS(7)
#undef MGLU_MASKED_ALL_STEPS
#undef MGLU_MASKED_STEP
  };

  // end of a tile round: stash fragments, reduce across the K-split warps, epilogue, store
  auto flush = [&](int round) {
    float* pw = part + (size_t)(wm * WK + wk) * part_warp_stride;
#pragma unroll
    for (int a = 0; a <= NM; ++a) {
      float* pa = pw + a * part_acc_stride;
      const int t0 = 2 * c, t1 = 2 * c + 1;
      if (t0 < Bp) { pa[r * Bp + t0] = acc[a][0]; pa[(r + 8) * Bp + t0] = acc[a][2]; }
      if (t1 < Bp) { pa[r * Bp + t1] = acc[a][1]; pa[(r + 8) * Bp + t1] = acc[a][3]; }
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[a][v] = 0.f;
    }
    __syncthreads();
    // WM tiles x 16 rows in this round; warp w reduces rows w, w+16, ...
    const int tok = lane & 7, grp = lane >> 3;
    for (int orow = warp; orow < WM * 16; orow += kMmaWarps) {
      const int twm = orow >> 4, row = orow & 15;
      const int tile = round * WM + twm;
      float vals[NM + 1];
#pragma unroll
      for (int a = 0; a <= NM; ++a) vals[a] = 0.f;
      if (tok < Bp) {
        for (int w2 = grp; w2 < WK; w2 += 4) {          // fixed order: deterministic
          const float* pp = part + (size_t)(twm * WK + w2) * part_warp_stride + row * Bp + tok;
#pragma unroll
          for (int a = 0; a <= NM; ++a) vals[a] += pp[a * part_acc_stride];
        }
      }
#pragma unroll
      for (int a = 0; a <= NM; ++a) {
        vals[a] += __shfl_xor_sync(0xffffffffu, vals[a], 8);
        vals[a] += __shfl_xor_sync(0xffffffffu, vals[a], 16);
      }
      const int lrow = tile * 16 + row;
      if (grp == 0 && tok < B && tile < ntiles && lrow < nrows) {
        float s[NM];
#pragma unroll
        for (int i = 0; i < NM; ++i) s[i] = vals[1 + i];
        const float y = mglu_epilogue<ACT, NM>(vals[0], s);          // Eq. 3, value = t - s_i
        p.out[(size_t)tok * p.h + r0 + lrow] = __float2bfloat16_rn(y);
      }
    }
    __syncthreads();
  };

  MmaStage st0, st1, st2;
  // W and the codes do not depend on the previous kernel: start streaming before the PDL wait.
  if (n_items > 0) load_stage(st0, 0);
  if (n_items > 1) load_stage(st1, 1);
  pdl_wait();
  pdl_launch_dependents();
  // x -> shared memory (B rows, padded stride)
  {
    const int vec_per_row = d >> 3;   // 16-byte vectors
    for (int v = threadIdx.x; v < B * vec_per_row; v += blockDim.x) {
      const int b = v / vec_per_row, q = v - b * vec_per_row;
      reinterpret_cast<uint4*>(xs + (size_t)b * xstride)[q] =
          reinterpret_cast<const uint4*>(p.x + (size_t)b * d)[q];
    }
  }
  __syncthreads();

#define MGLU_ITEM(S_CUR, S_NEXT2)                                        \
  {                                                                      \
    if (i + 2 < n_items) load_stage(S_NEXT2, i + 2);                     \
    compute(S_CUR, i);                                                   \
    if ((i % nkw) == nkw - 1) flush(i / nkw);                            \
    if (++i >= n_items) break;                                           \
  }
  int i = 0;
  if (n_items > 0) {
    for (;;) {
      MGLU_ITEM(st0, st2)
      MGLU_ITEM(st1, st0)
      MGLU_ITEM(st2, st1)
    }
  }
#undef MGLU_ITEM
}

}  // namespace mglu
