/*
 * mglu.h -- C ABI of libmglu: the FlashMGLU forward pass (MoEG / SwiMGLU up-projection) on
 * B200 (sm_100a).
 *
 * What it computes (Eq. 3, "MoEG Variant"):
 *
 *     y = sum_{i=1..n_m} g( x (M_i (.) W) ) (.) ( x (Mbar_i (.) W) ),   Mbar_i = 1 - M_i
 *
 * for every token row of x, with one shared weight W and n_m binary masks M_i that are fixed at
 * inference ("At inference, all masks are fixed, and the fused masked projections execute with
 * a single kernel").  The kernels read W and the packed masks from HBM once per call
 * (P:245), accumulate the unmasked product t and the gated sums s_i in one pass
 * (Alg. 1), form the value stream as t - s_i and apply g, the product
 * and the sum over i on chip.
 *
 * Letters (reading R2, BASELINE naming): d = reduction (model) dim, h = output
 * (intermediate) dim, B = tokens.
 *
 * ---------------------------------------------------------------------------------------------
 * Layouts (all row-major, contiguous, no padding):
 *   x        [B][d]   dtype of the handle (bf16 or f32)
 *   Wt       [h][d]   dtype of the handle.  Row j is column j of the logical W (d x h), i.e.
 *                     Alg. 1's A and nn.Linear.weight.
 *   packed   h*d*n_m/8 bytes (n_m bits per weight, Table 1's n_m*hd), the pair-split
 *                     bit-plane layout of DESIGN.md reading R3: for row j, 32-column group
 *                     g = k/32 and mask i (1..n_m), one little-endian 32-bit word at byte offset
 *                     ((j*(d/32) + g)*n_m + (i-1))*4 holds M_i[j, 32g .. 32g+31], column 32g+e at
 *                     bit (e/2) + 16*(e mod 2) (even columns in the low half-word, odd columns in
 *                     the high half-word).  M_i is bit (i-1) of the element's n_m-bit code
 *                     (Alg. 1: "mask[row,k] AND (1 << (i-1))").  Rows of Wt own contiguous
 *                     byte ranges [j*d*n_m/8, (j+1)*d*n_m/8), so an h-shard of a layer is a
 *                     pointer offset into Wt and into packed.
 *   out      [B][h]   dtype of the handle; bf16 stored round-to-nearest-even from fp32.
 *   z        [B][2*n_m][h] fp32 (debug partials, Alg. 1's accumulator order P:208):
 *                     z[b][i-1][j] = gate_i = s_i,   z[b][n_m+i-1][j] = value_i = t - s_i.
 *
 * Ownership: every data pointer is BORROWED.  The caller allocates x, Wt, packed, out, z (device
 * memory unless the entry point says "host") and keeps them alive until the work queued on
 * `stream` has completed.  A handle owns only its configuration, a TMA-descriptor cache and a
 * device workspace of the batched-decode path (MGLU_PATH_TCDEC), allocated on its first call (or
 * by mglu_reserve) and grown -- with a stream synchronisation -- only when a larger batch arrives;
 * otherwise mglu_forward never allocates, never frees and never synchronises (it enqueues kernels
 * on `stream` and returns).
 *
 * Errors: every call returns mglu_status; nothing throws or aborts across the ABI.  Argument
 * errors are detected before any launch.  Launch failures return MGLU_ERR_CUDA with the CUDA
 * error string available from mglu_last_error(handle).  Faults inside a kernel surface at the
 * caller's next synchronisation, as in CUDA.
 *
 * Threading: use a handle from ONE stream at a time (one handle per concurrently running stream).
 * The handle holds per-call state: the stream-K workspace and tile tickets (MGLU_PATH_TCDEC, which
 * AUTO picks for bf16 and 5 <= B <= 16 on narrow layers, and for n_m = 8 on layers with h >= 8192
 * from B = 1; the row split MGLU_PATH_TCROW keeps none) and mglu_forward_host's device staging
 * buffers.  Calls on different handles may run
 * concurrently on any streams (the kernels never wait on another CTA, so concurrent kernels always
 * make progress).  mglu_set_path / mglu_set_variant / mglu_set_debug and the descriptor cache are
 * guarded by a mutex.
 * Streams are `cudaStream_t` passed as void* (NULL = the legacy default stream).
 */
#ifndef MGLU_H_
#define MGLU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mglu_ctx* mglu_handle;

typedef enum {
  MGLU_OK = 0,
  MGLU_ERR_INVALID_ARG = 1,   /* null pointer, negative size, bad enum, dtype mismatch       */
  MGLU_ERR_UNSUPPORTED = 2,   /* n_m not in {1,2,4,8}; d % 32 != 0; path not available for cfg*/
  MGLU_ERR_MISALIGNED = 3,    /* a data pointer not 16-byte aligned                           */
  MGLU_ERR_CUDA = 4,          /* a CUDA runtime/driver call failed; see mglu_last_error()     */
  MGLU_ERR_OOM = 5            /* workspace allocation failed                                  */
} mglu_status;

/* g of Eq. 1/3 (reading R5): Swish = z*sigmoid(z) (SiLU, beta = 1); GELU exact erf form. */
typedef enum {
  MGLU_ACT_IDENTITY = 0,
  MGLU_ACT_SWISH = 1,
  MGLU_ACT_GELU = 2,
  MGLU_ACT_RELU = 3,
  MGLU_ACT_SIGMOID = 4
} mglu_activation;

typedef enum { MGLU_BF16 = 0, MGLU_F32 = 1 } mglu_dtype;

/* Kernel regime.  AUTO picks by dtype, n_m, h and B from measured crossovers: bf16
 * B <= 4 MMA; 5..32 TCROW on layers with >= 64 rows per SM (to 48 / 64 at n_m = 2 / 1; at n_m = 8
 * only with one tile per CTA), on narrower layers TCDEC up to 15 and TCROW 16..32; n_m = 8 on
 * large layers TCDEC up to 32; larger B TCGEN05; n_m = 16 TCGEN05; fp32 SIMT; a path that refuses
 * the shape falls through.  The others force one
 * kernel (for tests and benchmarks); forcing a path that cannot serve the configuration makes
 * mglu_forward return MGLU_ERR_UNSUPPORTED. */
typedef enum {
  MGLU_PATH_AUTO = 0,
  MGLU_PATH_SIMT = 1,     /* CUDA-core fused masked GEMV (Alg. 1 without split-K), any dtype/B   */
  MGLU_PATH_MMA = 2,      /* register-masked mma.sync GEMV, bf16, streams W+codes once per 8 tok */
  MGLU_PATH_TCGEN05 = 3,  /* tcgen05/TMEM masked GEMM, bf16, prefill / large B                  */
  MGLU_PATH_TCDEC = 4,    /* tcgen05 stream-K masked GEMV, bf16, decode 1 <= B <= 64             */
  MGLU_PATH_TCROW = 5     /* tcgen05 row-split masked GEMV (same kernel, each CTA owns whole     *
                           * row tiles over all of d: no cross-CTA reduction), bf16, 1 <= B <= 64,
                           * n_m <= 8 (B <= 32 at n_m = 8)                                          */
} mglu_path;

/* Create a handle for one (d, h, n_m, act, dtype) layer on CUDA device `device`.
 *   d, h >= 1; d % 32 == 0 (the 32-column groups of the packed layout, reading R3);
 *   n_m in {1, 2, 4, 8} (every kernel), or 3, 5, 6, 7, 16 (the SIMT kernel only: SURVEY row f3,
 *   P:885-947; the packed layout is the same n_m words per 32-column group), or n_m = 0 for a
 *   DENSE projection out = x Wt^T (no masks, no activation;
 *   `packed` may be NULL) -- the FFN down-projection W_o of SURVEY row f1 (bf16, MMA path,
 *   1 <= B <= 8, d % 128 == 0, x staged in shared memory: about 4 (B + 1) d bytes must fit next to
 *   two 32 KB stages; other configurations return UNSUPPORTED or CUDA from mglu_forward).
 * Errors: INVALID_ARG (null out, bad enum, d/h < 1), UNSUPPORTED (n_m, d % 32), CUDA, OOM. */
mglu_status mglu_create(mglu_handle* out, int64_t d, int64_t h, int n_m, int act, int dtype,
                        int device);

/* Destroy a handle (frees its workspace).  NULL is a no-op returning MGLU_OK. */
mglu_status mglu_destroy(mglu_handle hd);

/* Force a kernel regime (mglu_path).  INVALID_ARG for an unknown value. */
mglu_status mglu_set_path(mglu_handle hd, int path);

/* The forward pass: out[B][h] = Eq. 3 of x[B][d] (device pointers, 16-byte aligned).
 * B == 0 is a valid empty call (returns MGLU_OK, launches nothing).
 * Errors: INVALID_ARG (null pointer, B < 0), MISALIGNED, UNSUPPORTED (forced path cannot serve
 * this B/dtype), CUDA. */
mglu_status mglu_forward(mglu_handle hd, const void* x, int64_t B, const void* Wt,
                         const void* packed, void* out, void* stream);

/* Debug/test: Alg. 1's accumulators z[B][2*n_m][h] fp32 (see Layouts) instead of y.  Same
 * single pass over W and the codes; runs the SIMT regime.  Errors as mglu_forward. */
mglu_status mglu_forward_partials(mglu_handle hd, const void* x, int64_t B, const void* Wt,
                                  const void* packed, float* z, void* stream);

/* Partial-mask ablation variants (PAPER.md "Partial Mask Ablation"):
 * 0 = Eq. 3; 1 = NG (no gate mask: g(xW) (.) x(Mbar_i W)); 2 = NV (no value mask:
 * g(x(M_i W)) (.) xW); 3 = NM (no masks: g(xW) (.) xW), each applied per mask term and summed over i
 * (the paper defines n_m = 1).  Every path applies the variant in its epilogue.
 * Errors: INVALID_ARG (null, variant). */
mglu_status mglu_set_variant(mglu_handle hd, int variant);

/* Top-K routed MGLU (Appendix B).
 * mglu_router_topk: router logits l[b] = x[b] W_r in fp32 from bf16 inputs, then
 *   G[b] = Softmax(TopK(l[b])): the K largest logits (ties -> lowest index) get the
 *   softmax weights over those K values, every other entry exactly 0.
 *   Wr [n_m][d] bf16 row-major (row i = logit i's weights, like Wt), device; G [B][n_m] fp32,
 *   device, written.  1 <= K <= n_m.  bf16 handles only.  One launch.
 *   Errors: INVALID_ARG (nulls, B < 0, K out of range), MISALIGNED, UNSUPPORTED (fp32), CUDA.
 * mglu_forward_routed: y[b][j] = sum_i G[b][i] g(s_i) (t - s_i) in one pass over W and
 *   the codes, G [B][n_m] fp32 on the device (e.g. from mglu_router_topk on the same stream; read
 *   after the predecessor completes).  K (0..n_m) promises at most K nonzero weights per token (as
 *   produced by mglu_router_topk with that K); 0 = no promise.  With K > 0 the MMA path evaluates
 *   only the masks some token of the call selected (at most min(n_m, B*K); their sign flips and MMAs,
 *   Swish only -- other activations evaluate every mask); a G violating the promise gives undefined
 *   output.  Dispatch as mglu_forward (the tensor-core paths evaluate every mask and weigh them in
 *   their epilogues).  Errors as mglu_forward, plus INVALID_ARG (K) / MISALIGNED for G. */
mglu_status mglu_router_topk(mglu_handle hd, const void* x, int64_t B, const void* Wr, int K, float* G,
                             void* stream);
mglu_status mglu_forward_routed(mglu_handle hd, const void* x, int64_t B, const void* Wt, const void* packed,
                                const float* G, int K, void* out, void* stream);

/* Row f1, fused: the SwiMGLU FFN block out = MGLU(x) Wo^T (DESIGN R19) in ONE launch.
 *   up    an MGLU handle (d, h, n_m in {1, 2, 4, 8}, any act), down a DENSE handle (h, d_out, 0);
 *   x [B][d], Wt [h][d], packed (interleaved codes), Wo [d_out][h] (nn.Linear(h, d_out).weight),
 *   y_mid [B][h] bf16 (written: MGLU(x), rounded to bf16 -- the value the down-projection reads),
 *   out [B][d_out] bf16.  Every pointer device, 16-byte aligned, borrowed.
 * The grid streams the up-projection's W and codes and then W_o through one shared-memory ring,
 * with a grid-wide barrier (cooperative launch: all CTAs resident, one per SM) between the phases;
 * the result equals up.forward followed by down.forward bit for bit.  bf16, 1 <= B <= 4,
 * d % 128 == 0 and h % 128 == 0, Swish at n_m = 8, else UNSUPPORTED; mismatched handles INVALID_ARG.  The up
 * handle keeps the barrier state (8 bytes, allocated on the first call): one stream at a time per
 * up handle.  x, y_mid and out must be distinct buffers (INVALID_ARG otherwise). */
mglu_status mglu_ffn_forward(mglu_handle up, mglu_handle down, const void* x, int64_t B, const void* Wt,
                             const void* packed, const void* Wo, void* y_mid, void* out, void* stream);

/* Top-K routed forward on PLANE-MAJOR codes (mglu_pack_planes_*): the same result as
 * mglu_forward_routed on the interleaved codes (bit-identical: same kernel arithmetic), but each
 * stage streams W and only the planes some token selected.  MMA path only: bf16, Swish, standard
 * variant, 1 <= B <= 4, d % 128 == 0, 1 <= K <= n_m; other configurations return UNSUPPORTED. */
mglu_status mglu_forward_routed_planes(mglu_handle hd, const void* x, int64_t B, const void* Wt, const void* planes,
                                       const float* G, int K, void* out, void* stream);

/* End-to-end form: x_host [B][d] and out_host [B][h] are HOST buffers (pinned for async
 * copies; pageable works but serialises).  Copies x to the handle's device staging buffer,
 * runs mglu_forward, copies y back, all enqueued on `stream` (the caller synchronises).  With
 * page-locked, device-mapped buffers the copies are small kernels chained to the forward by PDL
 * (its W streaming overlaps x's transfer, the copy-out launches during its tail); other buffers
 * use cudaMemcpyAsync.  The
 * staging buffer is allocated at the first call for a given B and reused (grown, never shrunk).
 * Errors as mglu_forward plus OOM. */
mglu_status mglu_forward_host(mglu_handle hd, const void* x_host, int64_t B, const void* Wt,
                              const void* packed, void* out_host, void* stream);

/* Number of packed-mask bytes of an (h x d) layer with n_m masks: h*d*n_m/8 (Table 1's n_m*hd
 * mask bits).  Returns 0 for invalid arguments (including d % 32 != 0). */
size_t mglu_packed_mask_bytes(int64_t d, int64_t h, int n_m);

/* Offline mask packing ("all masks are fixed"; "Combine the n_m binary masks ...").
 *   bits   [n_m][h][d] uint8, each 0 or 1 (INVALID_ARG on any other value)
 *   logits [n_m][h][d] float32; bit = (logit > 0), strict (Alg. 2; reading R4)
 *   packed mglu_packed_mask_bytes(d, h, n_m) bytes (written entirely); d % 32 == 0 else
 *          UNSUPPORTED; device variants need a 16-byte aligned packed buffer (MISALIGNED)
 * Host variants work on host memory, run synchronously and validate every bit byte; device
 * variants take device pointers, enqueue one kernel on `stream` and use bit (b & 1) of each byte
 * (a device-side value check could only be reported after a synchronisation). */
mglu_status mglu_pack_masks_host(const uint8_t* bits, int n_m, int64_t h, int64_t d,
                                 uint8_t* packed);
mglu_status mglu_pack_logits_host(const float* logits, int n_m, int64_t h, int64_t d,
                                  uint8_t* packed);
mglu_status mglu_unpack_masks_host(const uint8_t* packed, int n_m, int64_t h, int64_t d,
                                   uint8_t* bits);
/* Plane-major code layout (row f2): plane i (mask i + 1) is [h][d/32] u32 words, word
 * (i, j, g) at byte offset ((i h + j) d/32 + g) * 4, each word holding M_{i+1}[j, 32g .. 32g+31] in
 * the same pair-split bit order as the interleaved layout (R3).  Same h*d*n_m/8 bytes; a routed
 * call on it loads only the planes its tokens selected (16 + K instead of 16 + n_m bits per
 * element).  These convert an interleaved `packed` (mglu_pack_masks_*) into `planes`.
 * Errors: INVALID_ARG (null / negative), UNSUPPORTED (n_m, d % 32), MISALIGNED (device). */
mglu_status mglu_pack_planes_host(const uint8_t* packed, int n_m, int64_t h, int64_t d, uint8_t* planes);
mglu_status mglu_pack_planes_device(const uint8_t* packed, int n_m, int64_t h, int64_t d, uint8_t* planes,
                                    void* stream);
mglu_status mglu_pack_masks_device(const uint8_t* bits, int n_m, int64_t h, int64_t d,
                                   uint8_t* packed, void* stream);
mglu_status mglu_pack_logits_device(const float* logits, int n_m, int64_t h, int64_t d,
                                    uint8_t* packed, void* stream);
mglu_status mglu_unpack_masks_device(const uint8_t* packed, int n_m, int64_t h, int64_t d,
                                     uint8_t* bits, void* stream);

/* Interop with per-element codes ("Combine the n_m binary masks into a single integer code
 * per weight element"; Alg. 1's bit test `mask & (1 << (i-1))`; the listing's one uint8
 * mask per element).  A code stream holds one w-bit field per
 * element of the [h][d] layer, field (j, k) at bit offset w*(j*d + k), little-endian (bit b of the
 * stream = bit b%8 of byte b/8); mask i is bit i-1 of the field.
 *   w = n_m: the dense stream (h*d*n_m/8 bytes; n_m in {1,2,4,8,16});
 *   w = 8:   one byte per element (the paper's listing; any n_m <= 8); w = 16: two bytes (n_m <= 16).
 * Field bits at or above n_m must be zero (INVALID_ARG otherwise: "high-bit contamination",
 * SPEC S:85).  mglu_codes_to_bits_host: stream -> 0/1 masks [n_m][h][d] (any d >= 1);
 * mglu_pack_codes_host: stream -> this library's packed layout (d % 32 == 0 else UNSUPPORTED);
 * mglu_unpack_codes_host: packed layout -> stream (the inverse; unused field bits written 0).
 * Host memory, synchronous; streams are ceil(h*d*w/8) bytes. */
size_t mglu_code_stream_bytes(int64_t d, int64_t h, int w);
mglu_status mglu_codes_to_bits_host(const uint8_t* codes, int w, int n_m, int64_t h, int64_t d, uint8_t* bits);
mglu_status mglu_pack_codes_host(const uint8_t* codes, int w, int n_m, int64_t h, int64_t d, uint8_t* packed);
mglu_status mglu_unpack_codes_host(const uint8_t* packed, int n_m, int64_t h, int64_t d, int w, uint8_t* codes);

/* Training path (Alg. 2: hard masks in the forward, the
 * straight-through estimator hands dL/dM_i to the soft logits unchanged; reading R21).  Given the
 * layer's inputs and the upstream gradient dy = dL/dy:
 *   x [B][d], Wt [h][d]  handle dtype (bf16 / fp32), packed masks as for mglu_forward;
 *   dy [B][h] fp32;
 *   dx [B][d], dW [h][d], dlogits [n_m][h][d] fp32 outputs, each optional (NULL skips it).
 * Recomputes the forward streams s_i, v_i with the forward kernels (partials mode, the path the
 * handle would take), then a_i = dy g'(s_i) v_i, c_i = dy g(s_i) and
 *   dx = sum_i a_i (M_i (.) W) + c_i (Mbar_i (.) W),   dW = sum_i M_i (.) a_i^T x + Mbar_i (.) c_i^T x,
 *   dlogits_i = W (.) (a_i - c_i)^T x.
 * fp32 accumulation, deterministic.  n_m in {1, 2, 4, 8}.  Uses a handle workspace of
 * (3 n_m + 1) B h floats (grown on demand, the growing call synchronises `stream`).
 * Errors: INVALID_ARG, UNSUPPORTED, OOM, CUDA; plus those of the forward. */
mglu_status mglu_backward(mglu_handle hd, const void* x, int64_t B, const void* Wt, const void* packed,
                          const float* dy, float* dx, float* dW, float* dlogits, void* stream);

/* Pre-allocates the stream-K (MGLU_PATH_TCDEC) workspace for batches up to max_B on `stream`.
 * Without it the workspace is allocated on the first TCDEC call and grown when a larger batch
 * arrives (the growing call synchronises `stream`); call this before capturing forwards into a
 * CUDA graph.  The workspace is (n_m + 1) x {16, 32, 64} x 128 x 8 bytes per SM plus one word per
 * 128-row tile.  Errors: INVALID_ARG, OOM, CUDA. */
mglu_status mglu_reserve(mglu_handle hd, int64_t max_B, void* stream);

/* Test hook ("injected mask-corruption flag"): with MGLU_DEBUG_FLIP_MASK_BIT set, every
 * forward / partials call on the handle flips bit 0 of the caller's packed codes -- mask 1 of
 * element (row 0, column 0) -- for the duration of the call (one XOR kernel before the forward and
 * one after, stream-ordered; the buffer is restored when the call's work completes).  The parity
 * suite must then fail at exactly that element.  0 clears the hook.  Not for production use. */
#define MGLU_DEBUG_FLIP_MASK_BIT 1
mglu_status mglu_set_debug(mglu_handle hd, int flags);

/* Number of kernels the last mglu_forward on this handle enqueued (for launch accounting). */
int mglu_last_launch_count(mglu_handle hd);

/* Which mglu_path the last mglu_forward on this handle ran. */
int mglu_last_path(mglu_handle hd);

/* Static strings; never NULL. */
const char* mglu_status_string(mglu_status s);
const char* mglu_last_error(mglu_handle hd);

/* Library version, "major.minor.patch". */
const char* mglu_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MGLU_H_ */
