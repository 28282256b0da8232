/*
 * q4_oracle.c -- CPU ORACLE for the q4f16 dequantize+matmul path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may link, import or
 * execute this file.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may call it.  It shares no code,
 * header, table or constant with the CUDA path (paper_2311_02103_b200/csrc,
 * include/).
 *
 * Citation key: P:n = /root/reference/PAPER.md line n (arXiv 2311.02103,
 * "Relax"); S:n = SPEC.md line n; SURVEY §8(c) = the readings adopted where
 * the paper is silent (restated in DESIGN.md §3).
 *
 * What is computed (the plain, unfused definition; fusion is semantics-
 * preserving, "FuseOps"/"FuseTensorIR", so the fused kernel must
 * reach this result):
 *
 *   q(k,j)  = (packed_w[j][k>>3] >> (4*(k&7))) & 0xF           reading 3
 *   s(k,j)  = scales[j][k>>5]                                     reading 2
 *   W(k,j)  = fp16_RNE( (q-7) * s )                               readings 1, 5
 *   r(i,j)  = sum_{k=0..K-1, ascending} x[i][k] * W(k,j)  in fp64 reading 6
 *   y(i,j)  = fp16_RNE( r(i,j) )                                  reading 7
 *
 * "int4 weight quantization and float16 activations" -- P:640.
 * Quantization is a tensor-program transform that can be lifted/fused
 * -- P:442-443; the naive triple loop as the reference semantics -- S:551.
 *
 * Everything is written out the slow, obvious way: one loop nest per
 * definition, fp64 sums in ascending k, no blocking, no reordering, no
 * vector intrinsics.  fp16 <-> fp64 conversion uses the C `_Float16` type
 * (ISO/IEC TS 18661-3, IEEE binary16, conversions round-to-nearest-even);
 * the build uses no -march flag, so GCC routes the conversions through its
 * portable soft-float routines, and -ffp-contract=off forbids fused
 * multiply-adds in the fp64 sums.
 *
 * Pinning (none of it re-types these formulas; see tests/test_oracle.py):
 *   - q4o_dequant: exhaustive 16 codes x 65536 scale bit patterns against
 *     numpy's IEEE float32 multiply + float16 cast; closed-form spot values;
 *     nibble-order words; golden fixture tests/golden/dequant_spot.txt.
 *   - q4o_matmul_f64 / q4o_matmul_cols_f64: brute force with exact rational
 *     arithmetic (fractions.Fraction) on tiny shapes; zero, identity-scale
 *     and one-hot invariants; row (prefix) independence.
 *   - q4o_round_f16: against numpy float64->float16 casts and closed forms.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define Q4O_OK 0
#define Q4O_ERR_ARG 1

/* fp16 bit pattern -> fp64 (exact: every binary16 value is a binary64 value). */
static double f16_bits_to_f64(uint16_t h)
{
    _Float16 v;
    memcpy(&v, &h, sizeof v);
    return (double)v;
}

/* fp64 -> fp16 bit pattern, one IEEE round-to-nearest-even rounding,
 * overflow to +-inf, subnormals kept, NaN stays NaN. */
static uint16_t f64_to_f16_bits(double d)
{
    _Float16 v = (_Float16)d;
    uint16_t h;
    memcpy(&h, &v, sizeof h);
    return h;
}

/* The 4-bit code of element k of output column j (reading 3: eight codes per
 * little-endian uint32, element k at bits 4*(k mod 8) .. 4*(k mod 8)+3). */
static unsigned code_at(const uint32_t* packed_w, int64_t K, int64_t j, int64_t k)
{
    uint32_t word = packed_w[j * (K / 8) + (k >> 3)];
    return (unsigned)((word >> (4 * (k & 7))) & 0xFu);
}

/* W(k,j) = fp16_RNE((q-7) * s), readings 1 (zero point 7), 2 (G=32 along K),
 * 5 (one RNE rounding of the exact product).  The product of an integer in
 * [-7,8] and a binary16 value is exact in binary64, so the only rounding is
 * the final conversion. */
static uint16_t dequant_one(const uint32_t* packed_w, const uint16_t* scales,
                            int64_t K, int64_t j, int64_t k)
{
    int q = (int)code_at(packed_w, K, j, k);
    double s = f16_bits_to_f64(scales[j * (K / 32) + (k >> 5)]);
    return f64_to_f16_bits((double)(q - 7) * s);
}

/* Dequantize the whole weight: w_out[j][k] = W(k,j) as fp16 bits, [N][K]. */
int q4o_dequant(const uint32_t* packed_w, const uint16_t* scales,
                int64_t K, int64_t N, uint16_t* w_out)
{
    if (K <= 0 || N < 0 || K % 32 != 0) return Q4O_ERR_ARG;
    for (int64_t j = 0; j < N; ++j)
        for (int64_t k = 0; k < K; ++k)
            w_out[j * K + k] = dequant_one(packed_w, scales, K, j, k);
    return Q4O_OK;
}

/* r[i][c] = sum_k x[i][k] * W(k, cols[c]) for the listed output columns,
 * fp64, k ascending.  "Dequantize, then matmul": each column's weights are
 * dequantized to fp16 first (into wrow), then used.  OpenMP splits the
 * independent columns only; every r entry is summed by one thread in the
 * fixed ascending order, so the result does not depend on the thread count. */
int q4o_matmul_cols_f64(const uint16_t* x, int64_t n, int64_t K,
                        const uint32_t* packed_w, const uint16_t* scales,
                        const int64_t* cols, int64_t ncols, double* r,
                        int nthreads)
{
    if (K <= 0 || n < 0 || ncols < 0 || K % 32 != 0) return Q4O_ERR_ARG;
    if (nthreads < 1) nthreads = 1;
    int64_t c;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (c = 0; c < ncols; ++c) {
        const int64_t j = cols[c];
        double* wrow = (double*)malloc((size_t)K * sizeof(double)); /* W(:,j) */
        for (int64_t k = 0; k < K; ++k)
            wrow[k] = f16_bits_to_f64(dequant_one(packed_w, scales, K, j, k));
        for (int64_t i = 0; i < n; ++i) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k)
                acc += f16_bits_to_f64(x[i * K + k]) * wrow[k];
            r[i * ncols + c] = acc;
        }
        free(wrow);
    }
    return Q4O_OK;
}

/* Full output: r[i][j], [n][N], fp64. */
int q4o_matmul_f64(const uint16_t* x, int64_t n, int64_t K, int64_t N,
                   const uint32_t* packed_w, const uint16_t* scales,
                   double* r, int nthreads)
{
    if (K <= 0 || n < 0 || N < 0 || K % 32 != 0) return Q4O_ERR_ARG;
    if (nthreads < 1) nthreads = 1;
    int64_t j;
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads)
    for (j = 0; j < N; ++j) {
        double* wrow = (double*)malloc((size_t)K * sizeof(double));
        for (int64_t k = 0; k < K; ++k)
            wrow[k] = f16_bits_to_f64(dequant_one(packed_w, scales, K, j, k));
        for (int64_t i = 0; i < n; ++i) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k)
                acc += f16_bits_to_f64(x[i * K + k]) * wrow[k];
            r[i * N + j] = acc;
        }
        free(wrow);
    }
    return Q4O_OK;
}

/* y = fp16_RNE(r) elementwise (reading 7: no saturation, overflow -> inf). */
void q4o_round_f16(const double* r, int64_t count, uint16_t* y)
{
    for (int64_t t = 0; t < count; ++t) y[t] = f64_to_f16_bits(r[t]);
}

/* fp16 bits -> fp64, exposed so tests can check the conversion itself. */
void q4o_f16_to_f64(const uint16_t* h, int64_t count, double* out)
{
    for (int64_t t = 0; t < count; ++t) out[t] = f16_bits_to_f64(h[t]);
}

int q4o_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
