/*
 * sale_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the SALE reference's CPU hot path (quantization,
 * Selection-Pass, Computation-Pass, dense oracle, block accounting). It is the
 * checker the GPU parity tests compare against; it is never linked into, or
 * called by, the product library (paper_2505_24179_b200/). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Pinning: tests/test_oracle.py checks every function here against (a) the
 * reference's own golden values (proj/tests/test_*.cpp, acceptance.cpp:320-323) and
 * (b) the real reference headers compiled into oracle/_ref/libsale_ref.so
 * (oracle/ref_capi.cpp) on seeded inputs, bit-for-bit.
 *
 * Build flags mirror the reference's (proj/CMakeLists.txt:8-10: -O3, no
 * -march) plus -ffp-contract=off so no FMA contraction changes the bits of the
 * double online update (SURVEY.md Appendix A / probe P4).
 *
 * Layout: one head at a time, row-major fp32 [tokens][dim] — the same layout as
 * sale::DenseMatrix (matrix.hpp:14-55). Masks are uint8 [nq][nk] like
 * sale::BlockMask (selection.hpp:48-85).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OK 0
#define E_INVALID 1
#define E_DOMAIN 2
#define E_RANGE 3

typedef struct {
    double tau;
    int64_t sink_tokens;
    int64_t local_tokens_min;
    int64_t segment_size;
    int64_t block_q;
    int64_t block_k;
} oracle_cfg;

static int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

/* matrix.hpp:78-83 — sequential fp32 dot, no contraction. */
static float dot_seq(const float *a, const float *b, int64_t n) {
    float acc = 0.0f;
    for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
    return acc;
}

/* SelectionConfig::validate, selection.hpp:26-37 */
int oracle_config_validate(const oracle_cfg *c) {
    if (!(c->tau > 0.0 && c->tau < 1.0)) return E_INVALID;
    if (c->sink_tokens < 1) return E_INVALID;
    if (c->block_q < 1 || c->block_k < 1) return E_INVALID;
    if (c->local_tokens_min < c->block_k) return E_INVALID;
    if (c->segment_size < 1) return E_INVALID;
    return OK;
}

/* ---------------------------------------------------------------- quant.hpp */

/* quant.hpp:68-74 (detail::max_abs) + quant.hpp:79-89 (detail::quantize_rows)
 * + quant.hpp:95-119: scale = peak>0 ? peak/7 : 1 in fp32; code =
 * clamp(lround((double)x / scale), -7, 7), lround being half-away-from-zero.
 * group_rows = 1 gives quantize_per_token, = block_k gives
 * quantize_per_key_block (last group may be ragged). */
int oracle_quantize(const float *x, int64_t rows, int64_t cols, int64_t group_rows,
                    int8_t *codes, float *scales) {
    if (group_rows < 1) return E_INVALID;
    for (int64_t g0 = 0, g = 0; g0 < rows; g0 += group_rows, ++g) {
        const int64_t g1 = imin(g0 + group_rows, rows);
        float peak = 0.0f;
        for (int64_t r = g0; r < g1; ++r)
            for (int64_t c = 0; c < cols; ++c) {
                const float a = fabsf(x[r * cols + c]);
                peak = peak < a ? a : peak; /* std::max(v, |x|) keeps v on ties */
            }
        const float scale = peak > 0.0f ? peak / 7.0f : 1.0f;
        scales[g] = scale;
        for (int64_t r = g0; r < g1; ++r)
            for (int64_t c = 0; c < cols; ++c) {
                long q = lround((double)x[r * cols + c] / (double)scale);
                if (q < -7) q = -7;
                if (q > 7) q = 7;
                codes[r * cols + c] = (int8_t)q;
            }
    }
    return OK;
}

/* quant.hpp:136-166 — int32 products of one (query rows x key rows) tile and
 * row_scales = q_scale * k_scale * inv_sqrt_d (left to right, fp32). */
int oracle_approx_weight_block(const int8_t *qcodes, const float *qscales, int64_t q_group_rows,
                               int64_t qb, int64_t qe, const int8_t *kcodes,
                               const float *kscales, int64_t k_group_rows, int64_t kb,
                               int64_t ke, int64_t d, int32_t *products, float *row_scales) {
    if (ke - kb == 0 || qe - qb == 0) return E_INVALID;
    if (kb / k_group_rows != (ke - 1) / k_group_rows) return E_INVALID;
    const float inv_sqrt_d = 1.0f / sqrtf((float)d);
    const float key_scale = kscales[kb / k_group_rows];
    for (int64_t r = 0; r < qe - qb; ++r) {
        row_scales[r] = qscales[(qb + r) / q_group_rows] * key_scale * inv_sqrt_d;
        const int8_t *qr = qcodes + (qb + r) * d;
        for (int64_t c = 0; c < ke - kb; ++c) {
            const int8_t *kr = kcodes + (kb + c) * d;
            int32_t acc = 0;
            for (int64_t t = 0; t < d; ++t) acc += (int32_t)qr[t] * (int32_t)kr[t];
            products[r * (ke - kb) + c] = acc;
        }
    }
    return OK;
}

/* quant.hpp:170-179 — first maximum wins ties; returns scale * (float)max. */
int oracle_max_then_dequantize(const int32_t *seg, int64_t n, float scale, float *value,
                               int64_t *col) {
    if (n == 0) return E_DOMAIN;
    int64_t best = 0;
    for (int64_t c = 1; c < n; ++c)
        if (seg[c] > seg[best]) best = c;
    *value = scale * (float)seg[best];
    *col = best;
    return OK;
}

/* ------------------------------------------------------------ block_grid.hpp */

typedef struct {
    int64_t tokens, bq, bk, nq, nk;
} grid_t;

static grid_t make_grid(int64_t tokens, int64_t bq, int64_t bk) {
    grid_t g = {tokens, bq, bk, (tokens + bq - 1) / bq, (tokens + bk - 1) / bk};
    return g;
}
static int64_t qbeg(const grid_t *g, int64_t i) { return i * g->bq; }
static int64_t qend(const grid_t *g, int64_t i) { return imin(i * g->bq + g->bq, g->tokens); }
static int64_t kbeg(const grid_t *g, int64_t j) { return j * g->bk; }
static int64_t kend(const grid_t *g, int64_t j) { return imin(j * g->bk + g->bk, g->tokens); }
/* block_grid.hpp:66-79 */
enum { FULLY_PAST = 0, OVERLAPPING = 1, FULLY_FUTURE = 2 };
static int causal_class(const grid_t *g, int64_t i, int64_t j) {
    if (kend(g, j) <= qbeg(g, i)) return FULLY_PAST;
    if (kbeg(g, j) >= qend(g, i)) return FULLY_FUTURE;
    return OVERLAPPING;
}

/* ------------------------------------------------------------- selection.hpp */

/* selection.hpp:92-123 — sorted, deduplicated I_SL. out must hold nk entries.
 * Returns the count, or -E_RANGE for a bad query block. */
int64_t oracle_sink_local_index_set(int64_t i, int64_t tokens, const oracle_cfg *cfg,
                                    int64_t *out) {
    const grid_t g = make_grid(tokens, cfg->block_q, cfg->block_k);
    if (i < 0 || i >= g.nq) return -E_RANGE;
    uint8_t *picked = (uint8_t *)calloc((size_t)g.nk, 1);
    for (int64_t j = 0; j < g.nk; ++j) {
        if (kbeg(&g, j) >= cfg->sink_tokens) break;
        if (kbeg(&g, j) >= qend(&g, i)) break;
        picked[j] = 1;
    }
    const int64_t frontier = imin((qend(&g, i) - 1) / g.bk, g.nk - 1);
    int64_t past = 0;
    for (int64_t j = frontier + 1; j-- > 0;) {
        if (causal_class(&g, i, j) == OVERLAPPING) {
            picked[j] = 1;
            continue;
        }
        if (past >= cfg->local_tokens_min) break;
        picked[j] = 1;
        past += kend(&g, j) - kbeg(&g, j);
    }
    int64_t n = 0;
    for (int64_t j = 0; j < g.nk; ++j)
        if (picked[j]) out[n++] = j;
    free(picked);
    return n;
}

/* selection.hpp:129-163 — exact statistics over the listed blocks, ascending,
 * no causal mask inside overlapping blocks. m/l have (qend-qbeg) entries. */
int oracle_sink_local_stats(const float *q, const float *k, int64_t tokens, int64_t d,
                            int64_t bq, int64_t bk, int64_t i, const int64_t *blocks,
                            int64_t nblocks, double *m, double *l) {
    if (nblocks == 0) return E_INVALID;
    const grid_t g = make_grid(tokens, bq, bk);
    const int64_t q0 = qbeg(&g, i), q1 = qend(&g, i);
    const float inv_sqrt_d = 1.0f / sqrtf((float)d);
    float logits[4096];
    if (bk > 4096) return E_INVALID;
    for (int64_t r = 0; r < q1 - q0; ++r) {
        m[r] = -INFINITY;
        l[r] = 0.0;
    }
    for (int64_t b = 0; b < nblocks; ++b) {
        const int64_t k0 = kbeg(&g, blocks[b]), k1 = kend(&g, blocks[b]);
        for (int64_t r = 0; r < q1 - q0; ++r) {
            const float *qr = q + (q0 + r) * d;
            double row_max = -INFINITY;
            for (int64_t t = 0; t < k1 - k0; ++t) {
                logits[t] = dot_seq(qr, k + (k0 + t) * d, d) * inv_sqrt_d;
                row_max = row_max < (double)logits[t] ? (double)logits[t] : row_max;
            }
            const double m_old = m[r];
            const double m_new = m_old < row_max ? row_max : m_old;
            double sum = 0.0;
            for (int64_t t = 0; t < k1 - k0; ++t) sum += exp((double)logits[t] - m_new);
            l[r] = l[r] * exp(m_old - m_new) + sum;
            m[r] = m_new;
        }
    }
    return OK;
}

/* selection.hpp:168-173 */
double oracle_threshold_bound(double tau, double running_max, double exp_sum) {
    double scaled = tau * exp_sum;
    if (scaled < DBL_MIN) scaled = DBL_MIN;
    return running_max + log(scaled);
}

/* selection.hpp:182-195 — OR within runs, trailing short run forced on. */
int oracle_segment_aggregate(uint8_t *middle, int64_t n, int64_t seg) {
    if (seg < 1) return E_INVALID;
    for (int64_t s = 0; s < n; s += seg) {
        const int64_t e = imin(s + seg, n);
        int keep = (e - s) < seg;
        for (int64_t i = s; i < e; ++i) keep = keep || middle[i] != 0;
        for (int64_t i = s; i < e; ++i) middle[i] = keep ? 1 : 0;
    }
    return OK;
}

/* selection.hpp:211-274 — the Selection-Pass for one head.
 * qcodes/qscales: per-token quantization of q (group 1); kcodes/kscales:
 * per-key-block quantization of k (group block_k). mask: uint8 [nq][nk].
 * Optional debug outputs (NULL to skip; when given, the early row exit of the
 * reference is disabled so every entry is filled — it cannot change the mask):
 *   m_out, l_out, bound_out: [tokens] doubles (rows of query blocks with an
 *     empty middle region are left NaN);
 *   block_max: int32 [tokens][nk], the per-row integer max of each estimated
 *     middle block (INT32_MIN elsewhere). */
int oracle_selection_pass(const float *q, const float *k, int64_t tokens, int64_t d,
                          const int8_t *qcodes, const float *qscales, const int8_t *kcodes,
                          const float *kscales, const oracle_cfg *cfg, uint8_t *mask,
                          double *m_out, double *l_out, double *bound_out,
                          int32_t *block_max) {
    if (oracle_config_validate(cfg)) return E_INVALID;
    if (tokens == 0 || d == 0) return E_INVALID;
    const grid_t g = make_grid(tokens, cfg->block_q, cfg->block_k);
    memset(mask, 0, (size_t)(g.nq * g.nk));
    const int64_t sink_blocks = (imin(cfg->sink_tokens, tokens) + g.bk - 1) / g.bk;
    int64_t *sl = (int64_t *)malloc(sizeof(int64_t) * (size_t)g.nk);
    double *m = (double *)malloc(sizeof(double) * (size_t)g.bq);
    double *l = (double *)malloc(sizeof(double) * (size_t)g.bq);
    double *bounds = (double *)malloc(sizeof(double) * (size_t)g.bq);
    uint8_t *raw = (uint8_t *)malloc((size_t)g.nk);
    const int full_debug = block_max != NULL;
    const float inv_sqrt_d = 1.0f / sqrtf((float)d);
    if (m_out)
        for (int64_t t = 0; t < tokens; ++t) m_out[t] = l_out[t] = bound_out[t] = NAN;
    if (block_max)
        for (int64_t t = 0; t < tokens * g.nk; ++t) block_max[t] = INT32_MIN;

    for (int64_t i = 0; i < g.nq; ++i) {
        const int64_t nsl = oracle_sink_local_index_set(i, tokens, cfg, sl);
        for (int64_t s = 0; s < nsl; ++s) mask[i * g.nk + sl[s]] = 1;
        const int64_t mb = imin(sink_blocks, g.nk);
        int64_t me = mb;
        for (int64_t s = 0; s < nsl; ++s)
            if (sl[s] >= sink_blocks) {
                me = imax(mb, sl[s]);
                break;
            }
        if (me == mb) continue;
        const int64_t q0 = qbeg(&g, i), q1 = qend(&g, i);
        oracle_sink_local_stats(q, k, tokens, d, g.bq, g.bk, i, sl, nsl, m, l);
        for (int64_t r = 0; r < q1 - q0; ++r) {
            bounds[r] = oracle_threshold_bound(cfg->tau, m[r], l[r]);
            if (m_out) {
                m_out[q0 + r] = m[r];
                l_out[q0 + r] = l[r];
                bound_out[q0 + r] = bounds[r];
            }
        }
        for (int64_t j = mb; j < me; ++j) {
            const int64_t k0 = kbeg(&g, j), k1 = kend(&g, j);
            const float key_scale = kscales[k0 / g.bk];
            int selected = 0;
            for (int64_t r = 0; r < q1 - q0 && (full_debug || !selected); ++r) {
                /* approx_weight_block row + max_then_dequantize (quant.hpp:152-178) */
                const float rs = qscales[q0 + r] * key_scale * inv_sqrt_d;
                const int8_t *qr = qcodes + (q0 + r) * d;
                int32_t best = 0;
                for (int64_t c = 0; c < k1 - k0; ++c) {
                    const int8_t *kr = kcodes + (k0 + c) * d;
                    int32_t acc = 0;
                    for (int64_t t = 0; t < d; ++t) acc += (int32_t)qr[t] * (int32_t)kr[t];
                    if (c == 0 || acc > best) best = acc;
                }
                if (block_max) block_max[(q0 + r) * g.nk + j] = best;
                const float est = rs * (float)best;
                if ((double)est >= bounds[r]) selected = 1;
            }
            raw[j - mb] = (uint8_t)selected;
        }
        oracle_segment_aggregate(raw, me - mb, cfg->segment_size);
        for (int64_t j = mb; j < me; ++j) mask[i * g.nk + j] = raw[j - mb];
    }
    free(sl);
    free(m);
    free(l);
    free(bounds);
    free(raw);
    return OK;
}

/* The statistics part of oracle_selection_pass alone (selection.hpp:224-251):
 * m, l and bound [tokens] for every query block with a non-empty middle
 * region (NaN elsewhere). Same loop, same calls; for parity runs at sizes
 * where the middle-block estimates are restated with exact BLAS products. */
int oracle_selection_stats(const float *q, const float *k, int64_t tokens, int64_t d,
                           const oracle_cfg *cfg, int64_t i_lo, int64_t i_hi, double *m_out,
                           double *l_out, double *bound_out) {
    if (oracle_config_validate(cfg)) return E_INVALID;
    if (tokens == 0 || d == 0) return E_INVALID;
    const grid_t g = make_grid(tokens, cfg->block_q, cfg->block_k);
    const int64_t sink_blocks = (imin(cfg->sink_tokens, tokens) + g.bk - 1) / g.bk;
    int64_t *sl = (int64_t *)malloc(sizeof(int64_t) * (size_t)g.nk);
    double *m = (double *)malloc(sizeof(double) * (size_t)g.bq);
    double *l = (double *)malloc(sizeof(double) * (size_t)g.bq);
    if (i_hi > g.nq || i_hi < 0) i_hi = g.nq;
    for (int64_t i = i_lo; i < i_hi; ++i) {
        const int64_t q0 = qbeg(&g, i), q1 = qend(&g, i);
        for (int64_t r = q0; r < q1; ++r) m_out[r] = l_out[r] = bound_out[r] = NAN;
        const int64_t nsl = oracle_sink_local_index_set(i, tokens, cfg, sl);
        const int64_t mb = imin(sink_blocks, g.nk);
        int64_t me = mb;
        for (int64_t s = 0; s < nsl; ++s)
            if (sl[s] >= sink_blocks) {
                me = imax(mb, sl[s]);
                break;
            }
        if (me == mb) continue;
        oracle_sink_local_stats(q, k, tokens, d, g.bq, g.bk, i, sl, nsl, m, l);
        for (int64_t r = 0; r < q1 - q0; ++r) {
            m_out[q0 + r] = m[r];
            l_out[q0 + r] = l[r];
            bound_out[q0 + r] = oracle_threshold_bound(cfg->tau, m[r], l[r]);
        }
    }
    free(sl);
    free(m);
    free(l);
    return OK;
}

/* ------------------------------------------------------ sparse_attention.hpp */

/* sparse_attention.hpp:37-97 — exact attention over the selected blocks,
 * ascending, causal clamp, fp32 logits, double online softmax. A row that
 * attends no token is a domain error (returned after all rows are written). */
int oracle_block_sparse_attention(const float *q, const float *k, const float *v,
                                  int64_t tokens, int64_t d, const uint8_t *mask, int64_t bq,
                                  int64_t bk, float *out, int64_t *coverage) {
    if (tokens == 0 || d == 0) return E_INVALID;
    const grid_t g = make_grid(tokens, bq, bk);
    const float inv_sqrt_d = 1.0f / sqrtf((float)d);
    double *acc = (double *)malloc(sizeof(double) * (size_t)d);
    int status = OK;
    for (int64_t i = 0; i < g.nq; ++i) {
        for (int64_t row = qbeg(&g, i); row < qend(&g, i); ++row) {
            const float *qr = q + row * d;
            double m = -INFINITY, l = 0.0;
            int64_t covered = 0;
            for (int64_t c = 0; c < d; ++c) acc[c] = 0.0;
            for (int64_t j = 0; j < g.nk; ++j) {
                if (causal_class(&g, i, j) == FULLY_FUTURE) break;
                if (!mask[i * g.nk + j]) continue;
                const int64_t end = imin(kend(&g, j), row + 1);
                for (int64_t t = kbeg(&g, j); t < end; ++t) {
                    const float s = dot_seq(qr, k + t * d, d) * inv_sqrt_d;
                    if (s > m) {
                        const double rescale = exp(m - (double)s);
                        l *= rescale;
                        for (int64_t c = 0; c < d; ++c) acc[c] *= rescale;
                        m = s;
                    }
                    const double w = exp((double)s - m);
                    l += w;
                    const float *vr = v + t * d;
                    for (int64_t c = 0; c < d; ++c) acc[c] += w * vr[c];
                    ++covered;
                }
            }
            if (covered == 0) {
                status = E_DOMAIN;
                for (int64_t c = 0; c < d; ++c) out[row * d + c] = NAN;
            } else {
                for (int64_t c = 0; c < d; ++c) out[row * d + c] = (float)(acc[c] / l);
            }
            if (coverage) coverage[row] = covered;
        }
    }
    free(acc);
    return status;
}

/* attention.hpp:18-50 — dense causal attention, same arithmetic. */
int oracle_full_attention(const float *q, const float *k, const float *v, int64_t tokens,
                          int64_t d, float *out) {
    if (tokens == 0 || d == 0) return E_INVALID;
    const float inv_sqrt_d = 1.0f / sqrtf((float)d);
    double *acc = (double *)malloc(sizeof(double) * (size_t)d);
    for (int64_t i = 0; i < tokens; ++i) {
        const float *qr = q + i * d;
        double m = -INFINITY, l = 0.0;
        for (int64_t c = 0; c < d; ++c) acc[c] = 0.0;
        for (int64_t j = 0; j <= i; ++j) {
            const float s = dot_seq(qr, k + j * d, d) * inv_sqrt_d;
            if (s > m) {
                const double rescale = exp(m - (double)s);
                l *= rescale;
                for (int64_t c = 0; c < d; ++c) acc[c] *= rescale;
                m = s;
            }
            const double w = exp((double)s - m);
            l += w;
            for (int64_t c = 0; c < d; ++c) acc[c] += w * v[j * d + c];
        }
        for (int64_t c = 0; c < d; ++c) out[i * d + c] = (float)(acc[c] / l);
    }
    free(acc);
    return OK;
}

/* sparse_attention.hpp:101-118 — counts[0..2] = computed, skipped, total. */
int oracle_flop_accounting(const uint8_t *mask, int64_t tokens, int64_t bq, int64_t bk,
                           int64_t *counts) {
    const grid_t g = make_grid(tokens, bq, bk);
    counts[0] = counts[1] = counts[2] = 0;
    for (int64_t i = 0; i < g.nq; ++i)
        for (int64_t j = 0; j < g.nk; ++j) {
            if (causal_class(&g, i, j) == FULLY_FUTURE) break;
            ++counts[2];
            if (mask[i * g.nk + j])
                ++counts[0];
            else
                ++counts[1];
        }
    return OK;
}

/* calibrate.hpp:20-29 — mean-per-token L1 distance. */
double oracle_l1_error(const float *a, const float *b, int64_t rows, int64_t cols) {
    double sum = 0.0;
    for (int64_t i = 0; i < rows * cols; ++i) sum += fabs((double)a[i] - (double)b[i]);
    return sum / (double)rows;
}
