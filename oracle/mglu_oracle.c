/*
 * mglu_oracle.c -- CPU ORACLE for the FlashMGLU forward pass.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  The product path (paper_2506_23225_b200/) never links, imports or
 * calls it, and it shares no code, header, table or constant with the CUDA path.
 *
 * What it computes -- PAPER.md Eq. (3) ("MoEG Variant"), written out literally,
 * every accumulation in binary64, k ascending, i ascending:
 *
 *   t[b,j]       = sum_k x[b,k] * Wt[j,k]                               (the unmasked product)
 *   gate_i[b,j]  = sum_k x[b,k] * Wt[j,k] * M_i[j,k]                    (x(M_i (.) W))
 *   value_i[b,j] = sum_k x[b,k] * Wt[j,k] * (1 - M_i[j,k])              (x(Mbar_i (.) W),
 *                                                                         Mbar = 1 - M)
 *   y[b,j]       = sum_{i=1..n_m} g(gate_i[b,j]) * value_i[b,j]
 *
 * value_i is computed as its own dot product with the complementary mask -- NOT as t - gate_i
 * (that identity, is what the kernel exploits and what the tests check).
 *
 * Mask bits (reading R3): M_i[j,k] is bit (i-1) of the n_m-bit code c[j,k] (Alg. 1
 * bit test "mask[row,k] AND (1 << (i-1))"), stored densely (n_m bits per weight, Table 1
 * P:278) in the pair-split bit-plane layout: for row j, column group g = k / 32 and mask i, one
 * little-endian 32-bit word at byte offset ((j*(d/32) + g)*n_m + (i-1))*4 holds the 32 bits of
 * M_i[j, 32g .. 32g+31]; column 32g + e sits at bit (e / 2) + 16*(e mod 2) (even columns in the
 * low half-word, odd columns in the high half-word).  d % 32 == 0.  This file reads that layout
 * with its own bit-at-a-time loop, independent of the library's packer.
 *
 * g (reading R5): 0 identity, 1 swish z*sigmoid(z) (beta=1), 2 gelu 0.5 z (1+erf(z/sqrt2)),
 * 3 relu max(z,0), 4 sigmoid 1/(1+exp(-z)).
 *
 * Orientation (reading R2): Wt is [h][d] row-major -- row j is output feature j, the A matrix of
 * Alg. 1 and nn.Linear.weight.  x is [B][d], y is [B][h]; each token row of x
 * is an independent instance of Eq. 3 (reading R15).
 *
 * Parallelism: OpenMP over output columns only; each output's k loop is sequential, so the
 * result does not depend on the thread count.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* byte offset of the word holding M_i[j, 32g .. 32g+31] and the bit of column k in it */
static uint64_t word_offset(int n_m, int64_t d, int64_t j, int64_t k, int i) {
    uint64_t g = (uint64_t)k / 32u;
    return (((uint64_t)j * ((uint64_t)d / 32u) + g) * (uint64_t)n_m + (uint64_t)(i - 1)) * 4u;
}
static unsigned bit_in_word(int64_t k) {
    unsigned e = (unsigned)(k % 32);
    return e / 2u + 16u * (e % 2u);
}

/* M_i[j,k] for i = 1..n_m: byte (bit / 8) of the little-endian word, bit (bit mod 8) */
static int mask_bit(const uint8_t *packed, int n_m, int64_t d, int64_t j, int64_t k, int i) {
    unsigned b = bit_in_word(k);
    return (packed[word_offset(n_m, d, j, k, i) + b / 8u] >> (b % 8u)) & 1;
}

static double act_g(int act, double z) {
    switch (act) {
    case 0: return z;                                   /* identity */
    case 1: return z / (1.0 + exp(-z));                 /* swish = z * sigmoid(z) */
    case 2: return 0.5 * z * (1.0 + erf(z / sqrt(2.0)));/* gelu, exact erf form */
    case 3: return z > 0.0 ? z : 0.0;                   /* relu */
    case 4: return 1.0 / (1.0 + exp(-z));               /* sigmoid */
    default: return NAN;
    }
}

/* thread count of the column loop (the result does not depend on it: each output column is one
   sequential k loop) -- lets a benchmark that runs under torchrun (OMP_NUM_THREADS=1) use the host */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* bits[(i-1)][j][k] in {0,1}  ->  packed layout (h*d*n_m/8 bytes) */
int oracle_pack(const uint8_t *bits, int n_m, int64_t h, int64_t d, uint8_t *packed) {
    if (n_m < 1 || n_m > 16 || h < 0 || d < 0 || d % 32) return 1;
    memset(packed, 0, (size_t)((uint64_t)n_m * (uint64_t)h * (uint64_t)d / 8u));
    for (int64_t j = 0; j < h; ++j)
        for (int64_t k = 0; k < d; ++k)
            for (int i = 1; i <= n_m; ++i) {
                uint8_t b = bits[((uint64_t)(i - 1) * (uint64_t)h + (uint64_t)j) * (uint64_t)d + (uint64_t)k];
                if (b > 1) return 2;
                unsigned q = bit_in_word(k);
                if (b) packed[word_offset(n_m, d, j, k, i) + q / 8u] |= (uint8_t)(1u << (q % 8u));
            }
    return 0;
}

/* packed layout -> bits[(i-1)][j][k] */
int oracle_unpack(const uint8_t *packed, int n_m, int64_t h, int64_t d, uint8_t *bits) {
    if (n_m < 1 || n_m > 16 || h < 0 || d < 0 || d % 32) return 1;
    for (int i = 1; i <= n_m; ++i)
        for (int64_t j = 0; j < h; ++j)
            for (int64_t k = 0; k < d; ++k)
                bits[((uint64_t)(i - 1) * (uint64_t)h + (uint64_t)j) * (uint64_t)d + (uint64_t)k] =
                    (uint8_t)mask_bit(packed, n_m, d, j, k, i);
    return 0;
}

/*
 * Eq. 3 for the token rows x[0..B) and the output columns cols[0..ncols).
 *   x      [B][d]        binary64 (bf16/f32 inputs decoded exactly by the caller)
 *   Wt_sel [ncols][d]    binary64, row c is Wt[cols[c], :]
 *   packed full packed-mask buffer of the (h x d) layer (global row index cols[c] is used)
 *   y      [B][ncols]    output
 *   z      [B][2*n_m][ncols] or NULL: Alg. 1's accumulator order:
 *          row (i-1) = gate_i, row (n_m+i-1) = value_i
 *   t_out  [B][ncols] or NULL: the unmasked product t
 */
int oracle_mglu_forward(const double *x, int64_t B, int64_t d,
                        const double *Wt_sel, const int64_t *cols, int64_t ncols,
                        const uint8_t *packed, int n_m, int act,
                        double *y, double *z, double *t_out) {
    if (n_m < 1 || n_m > 16 || act < 0 || act > 4 || B < 0 || d < 0 || d % 32 || ncols < 0) return 1;
    int64_t c;
#pragma omp parallel for schedule(dynamic, 8)
    for (c = 0; c < ncols; ++c) {
        const int64_t j = cols[c];
        const double *w = Wt_sel + (uint64_t)c * (uint64_t)d;
        for (int64_t b = 0; b < B; ++b) {
            const double *xb = x + (uint64_t)b * (uint64_t)d;
            double t = 0.0;
            for (int64_t k = 0; k < d; ++k) t += xb[k] * w[k];
            double acc = 0.0;
            for (int i = 1; i <= n_m; ++i) {
                double gate = 0.0, value = 0.0;
                for (int64_t k = 0; k < d; ++k) {
                    double m = (double)mask_bit(packed, n_m, d, j, k, i);
                    gate += xb[k] * w[k] * m;
                }
                for (int64_t k = 0; k < d; ++k) {
                    double mbar = 1.0 - (double)mask_bit(packed, n_m, d, j, k, i);
                    value += xb[k] * w[k] * mbar;
                }
                acc += act_g(act, gate) * value;
                if (z) {
                    z[((uint64_t)b * (uint64_t)(2 * n_m) + (uint64_t)(i - 1)) * (uint64_t)ncols + (uint64_t)c] = gate;
                    z[((uint64_t)b * (uint64_t)(2 * n_m) + (uint64_t)(n_m + i - 1)) * (uint64_t)ncols + (uint64_t)c] = value;
                }
            }
            y[(uint64_t)b * (uint64_t)ncols + (uint64_t)c] = acc;
            if (t_out) t_out[(uint64_t)b * (uint64_t)ncols + (uint64_t)c] = t;
        }
    }
    return 0;
}
