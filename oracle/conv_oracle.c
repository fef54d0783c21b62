/*
 * oracle/conv_oracle.c -- TEST INFRASTRUCTURE ONLY. Never linked into, called by,
 * or measured as the product. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker.
 *
 * A plain-C restatement of the reference CPU convolution path
 * (/root/reference/proj/include/convgemm/), compiled with the reference's
 * forced -ffp-contract=off (proj/src/CMakeLists.txt:12-16) so its float
 * results are bit-identical to the reference operator:
 *
 *   orc_output_dims    conv_params.hpp:27-36   floor formula + InvalidGeometry
 *   orc_conv_direct    conv.hpp:24-55          seven-loop direct conv
 *   orc_im2col         im2col.hpp:77-120       explicit lowered matrix B (k x n, ld >= k)
 *   orc_conv_gemm      conv.hpp:60-91 + gemm.hpp:46-97 + microkernel.hpp:20-38
 *
 * Parity pinning: tests/test_oracle.py checks every function here bitwise
 * against oracle/_ref (the reference itself, compiled from its sources) and
 * against the committed golden fixtures in tests/golden/.
 *
 * Accumulation order of the blocked GEMM (why orc_conv_gemm is bit-exact):
 * the reference zeroes C (gemm.hpp:26-30), then for every p_c block of kc
 * rows (gemm.hpp:64-66) the micro-kernel accumulates acc = 0 + a0*b0 + a1*b1
 * ... in ascending p with separate multiply and add (microkernel.hpp:25-34,
 * no FMA because of -ffp-contract=off) and flushes C += acc once
 * (microkernel.hpp:35-37). Each C element is owned by exactly one micro-tile
 * per (j_c, p_c, i_c) step, so its value depends only on kc, not on
 * mc/nc/mr/nr or the thread count (gemm.hpp:40-45). This file reproduces that
 * per-element order directly.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_INVALID_GEOMETRY 1
#define ORC_INVALID_ARGUMENT 4

typedef struct {
    int64_t k_n, k_h, k_w, c_i, h_i, w_i, b, s, p; /* ConvParams, conv_params.hpp:8-16 */
} orc_params;

static orc_params unpack(const int64_t *a) {
    orc_params cp = {a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8]};
    return cp;
}

/* conv_params.hpp:27-36 */
int orc_output_dims(const int64_t *cpa, int64_t *h_o, int64_t *w_o) {
    const orc_params cp = unpack(cpa);
    if (cp.k_n < 1 || cp.k_h < 1 || cp.k_w < 1 || cp.c_i < 1 || cp.h_i < 1 || cp.w_i < 1 ||
        cp.b < 1 || cp.s < 1 || cp.p < 0)
        return ORC_INVALID_GEOMETRY;
    const int64_t dh = cp.h_i - cp.k_h + 2 * cp.p;
    const int64_t dw = cp.w_i - cp.k_w + 2 * cp.p;
    if (dh < 0 || dw < 0) return ORC_INVALID_GEOMETRY;
    *h_o = dh / cp.s + 1;
    *w_o = dw / cp.s + 1;
    return ORC_OK;
}

/* conv.hpp:24-55: O zero-filled, then b, c, w, h, kw, kh, k loop nest with
 * virtual padding (out-of-range reads are skipped). */
int orc_conv_direct_f32(const float *F, const float *I, const int64_t *cpa, float *O) {
    int64_t h_o, w_o;
    int rc = orc_output_dims(cpa, &h_o, &w_o);
    if (rc) return rc;
    const orc_params cp = unpack(cpa);
    const int64_t osize = cp.k_n * h_o * w_o * cp.b;
    memset(O, 0, (size_t)osize * sizeof(float));
    for (int64_t i_b = 0; i_b < cp.b; ++i_b)
        for (int64_t i_c = 0; i_c < cp.c_i; ++i_c) {
            const float *plane = I + (i_c + i_b * cp.c_i) * cp.h_i * cp.w_i;
            for (int64_t i_w = 0; i_w < w_o; ++i_w)
                for (int64_t i_h = 0; i_h < h_o; ++i_h) {
                    float *out_col = O + cp.k_n * (i_h + h_o * (i_w + w_o * i_b));
                    for (int64_t i_kw = 0; i_kw < cp.k_w; ++i_kw) {
                        const int64_t w_in = i_w * cp.s + i_kw - cp.p;
                        if (w_in < 0 || w_in >= cp.w_i) continue;
                        for (int64_t i_kh = 0; i_kh < cp.k_h; ++i_kh) {
                            const int64_t h_in = i_h * cp.s + i_kh - cp.p;
                            if (h_in < 0 || h_in >= cp.h_i) continue;
                            const float x = plane[w_in * cp.h_i + h_in];
                            const float *f_col = F + cp.k_n * (i_kh + cp.k_h * (i_kw + cp.k_w * i_c));
                            for (int64_t i_k = 0; i_k < cp.k_n; ++i_k) out_col[i_k] += f_col[i_k] * x;
                        }
                    }
                }
        }
    return ORC_OK;
}

/* One column of the lowered matrix: B(r, c) for r in [0, k), im2col.hpp:71-76.
 * r = i_kh + i_kw*k_h + i_c*k_h*k_w, c = i_h + i_w*h_o + i_b*h_o*w_o. */
static void lowered_column(const float *I, const orc_params *cp, int64_t h_o, int64_t w_o,
                           int64_t col, float *dst) {
    const int64_t hw = h_o * w_o;
    const int64_t i_b = col / hw, rem = col % hw;
    const int64_t i_w = rem / h_o, i_h = rem % h_o;
    int64_t r = 0;
    for (int64_t i_c = 0; i_c < cp->c_i; ++i_c) {
        const float *plane = I + (i_c + i_b * cp->c_i) * cp->h_i * cp->w_i;
        for (int64_t i_kw = 0; i_kw < cp->k_w; ++i_kw) {
            const int64_t w_in = i_w * cp->s + i_kw - cp->p;
            for (int64_t i_kh = 0; i_kh < cp->k_h; ++i_kh) {
                const int64_t h_in = i_h * cp->s + i_kh - cp->p;
                dst[r++] = (w_in >= 0 && w_in < cp->w_i && h_in >= 0 && h_in < cp->h_i)
                               ? plane[w_in * cp->h_i + h_in]
                               : 0.0f;
            }
        }
    }
}

/* im2col.hpp:77-120: B is k x n column-major with leading dimension ldb >= k. */
int orc_im2col_f32(const float *I, const int64_t *cpa, float *B, int64_t ldb) {
    int64_t h_o, w_o;
    int rc = orc_output_dims(cpa, &h_o, &w_o);
    if (rc) return rc;
    const orc_params cp = unpack(cpa);
    const int64_t k = cp.k_h * cp.k_w * cp.c_i;
    if (ldb < k) return ORC_INVALID_ARGUMENT;
    const int64_t n = h_o * w_o * cp.b;
#pragma omp parallel for schedule(static)
    for (int64_t col = 0; col < n; ++col) {
        lowered_column(I, &cp, h_o, w_o, col, B + col * ldb);
        for (int64_t r = k; r < ldb; ++r) B[col * ldb + r] = 0.0f;
    }
    return ORC_OK;
}

/* conv_gemm / conv_im2col_gemm result (they are bit-identical by construction,
 * test_convgemm.cpp:163-190): O(i_k, col) = sum over kc-blocks of
 * (0 + sum_{r in block} F(i_k, r) * B(r, col)), blocks and terms ascending. */
int orc_conv_gemm_f32(const float *F, const float *I, const int64_t *cpa, int64_t kc, float *O) {
    int64_t h_o, w_o;
    int rc = orc_output_dims(cpa, &h_o, &w_o);
    if (rc) return rc;
    if (kc < 1) return ORC_INVALID_ARGUMENT;
    const orc_params cp = unpack(cpa);
    const int64_t k = cp.k_h * cp.k_w * cp.c_i;
    const int64_t n = h_o * w_o * cp.b;
    const int64_t m = cp.k_n;
#pragma omp parallel
    {
        float *col = (float *)malloc((size_t)k * sizeof(float));
        float *acc = (float *)malloc((size_t)m * sizeof(float));
#pragma omp for schedule(static)
        for (int64_t j = 0; j < n; ++j) {
            lowered_column(I, &cp, h_o, w_o, j, col);
            float *out = O + j * m;
            for (int64_t i = 0; i < m; ++i) out[i] = 0.0f;
            for (int64_t p_c = 0; p_c < k; p_c += kc) {
                const int64_t p_end = p_c + kc < k ? p_c + kc : k;
                for (int64_t i = 0; i < m; ++i) acc[i] = 0.0f;
                for (int64_t p = p_c; p < p_end; ++p) {
                    const float bj = col[p];
                    const float *a = F + p * m;
                    for (int64_t i = 0; i < m; ++i) acc[i] += a[i] * bj;
                }
                for (int64_t i = 0; i < m; ++i) out[i] += acc[i];
            }
        }
        free(col);
        free(acc);
    }
    return ORC_OK;
}

/* f64 accumulation of the same lowered product, for diagnosing oracle error
 * versus GPU error. Not a reference function. */
int orc_conv_f64acc(const float *F, const float *I, const int64_t *cpa, double *O) {
    int64_t h_o, w_o;
    int rc = orc_output_dims(cpa, &h_o, &w_o);
    if (rc) return rc;
    const orc_params cp = unpack(cpa);
    const int64_t k = cp.k_h * cp.k_w * cp.c_i;
    const int64_t n = h_o * w_o * cp.b;
    const int64_t m = cp.k_n;
#pragma omp parallel
    {
        float *col = (float *)malloc((size_t)k * sizeof(float));
#pragma omp for schedule(static)
        for (int64_t j = 0; j < n; ++j) {
            lowered_column(I, &cp, h_o, w_o, j, col);
            double *out = O + j * m;
            for (int64_t i = 0; i < m; ++i) out[i] = 0.0;
            for (int64_t p = 0; p < k; ++p) {
                const double bj = col[p];
                const float *a = F + p * m;
                for (int64_t i = 0; i < m; ++i) out[i] += (double)a[i] * bj;
            }
        }
        free(col);
    }
    return ORC_OK;
}

/* Per-output Cauchy-Schwarz scale ||F[i_k,:]||_2 * ||B[:,col]||_2 used by the
 * north-star tolerance (BASELINE.json: "normalised by ||F||*||I|| per output"). */
int orc_output_scale(const float *F, const float *I, const int64_t *cpa, double *S) {
    int64_t h_o, w_o;
    int rc = orc_output_dims(cpa, &h_o, &w_o);
    if (rc) return rc;
    const orc_params cp = unpack(cpa);
    const int64_t k = cp.k_h * cp.k_w * cp.c_i;
    const int64_t n = h_o * w_o * cp.b;
    const int64_t m = cp.k_n;
    double *fn = (double *)calloc((size_t)m, sizeof(double));
    for (int64_t p = 0; p < k; ++p)
        for (int64_t i = 0; i < m; ++i) fn[i] += (double)F[p * m + i] * F[p * m + i];
#pragma omp parallel
    {
        float *col = (float *)malloc((size_t)k * sizeof(float));
#pragma omp for schedule(static)
        for (int64_t j = 0; j < n; ++j) {
            lowered_column(I, &cp, h_o, w_o, j, col);
            double bn = 0.0;
            for (int64_t p = 0; p < k; ++p) bn += (double)col[p] * col[p];
            for (int64_t i = 0; i < m; ++i) S[j * m + i] = __builtin_sqrt(fn[i] * bn);
        }
        free(col);
    }
    free(fn);
    return ORC_OK;
}
