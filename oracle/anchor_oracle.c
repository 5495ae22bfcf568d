/*
 * TEST INFRASTRUCTURE ONLY — see anchor_oracle.h.
 *
 * CPU restatement of the reference AnchorAttention pipeline.  Every function
 * names the reference lines it follows (R/ = /root/reference/proj/).  The
 * arithmetic mirrors the reference operation for operation (f64 dot products
 * over f32 operands in index order, 1/sqrt(d) applied after the dot, online
 * merge per kv block / per index chunk) so that its results agree with the
 * reference to the last few ulps; parity is pinned by
 * tests/test_oracle_golden.py against fixtures produced by oracle/_ref.
 *
 * Parallelism: rows / groups are independent (R/../SPEC.md "Query blocks are
 * independent"), so loops over query blocks and groups use OpenMP.  Per-row
 * arithmetic order is unchanged, so results do not depend on thread count.
 */
#include "anchor_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
static int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

/* R/src/matrix.cpp:31-42 */
int ao_validate(const ao_cfg* c) {
    if (c->b_q <= 0 || c->b_kv <= 0 || c->step <= 0) return 1;
    if (c->b_q % c->b_kv != 0 && c->b_kv % c->b_q != 0) return 1;
    if (!isfinite(c->theta)) return 1;
    return 0;
}

/* R/src/detail/geometry.hpp:36-38 */
int64_t ao_group_count(int64_t n, const ao_cfg* c) {
    return ceil_div(ceil_div(n, c->b_q), c->step);
}

/* R/src/detail/geometry.hpp:55-59 */
int64_t ao_window_start_block(int64_t g, const ao_cfg* c) {
    const int64_t row_begin = g * c->step * c->b_q;
    if (row_begin < c->b_kv * 2) return 1;
    return row_begin / c->b_kv - 1;
}

/* R/src/detail/geometry.hpp:61-64 */
int64_t ao_window_start_token(int64_t g, const ao_cfg* c, int64_t n) {
    return min64(ao_window_start_block(g, c) * c->b_kv, n);
}

/* R/src/detail/geometry.hpp:66-69 */
int64_t ao_middle_end_token(int64_t g, const ao_cfg* c, int64_t n) {
    return max64(ao_window_start_token(g, c, n), min64(c->b_kv, n));
}

/* R/src/detail/geometry.hpp:79-85 */
int64_t ao_covered_count_for_row(int64_t row, const ao_cfg* c, int64_t n) {
    const int64_t init = min64(c->b_kv, row + 1);
    const int64_t g = row / (c->step * c->b_q);
    const int64_t wstart = ao_window_start_token(g, c, n);
    const int64_t window = row + 1 > wstart ? row + 1 - wstart : 0;
    return init + window;
}

/* R/src/anchor_pass.cpp:113-118 */
int64_t ao_anchor_covered_count(int64_t n, const ao_cfg* c) {
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) total += ao_covered_count_for_row(i, c, n);
    return total;
}

static int64_t middle_len(int64_t g, const ao_cfg* c, int64_t n) {
    const int64_t e = ao_middle_end_token(g, c, n);
    return e > c->b_kv ? e - c->b_kv : 0;
}

int64_t ao_stripe_offset(int64_t g, const ao_cfg* c, int64_t n) {
    int64_t off = 0;
    for (int64_t h = 0; h < g; ++h) off += middle_len(h, c, n);
    return off;
}

int64_t ao_stripe_capacity(int64_t n, const ao_cfg* c) {
    return ao_stripe_offset(ao_group_count(n, c), c, n);
}

/* R/src/anchor_pass.cpp:12-30 */
int64_t ao_anchor_region(int64_t qb, const ao_cfg* c, int64_t n, int64_t* blocks, int64_t cap) {
    const int64_t t_n = ceil_div(n, c->b_kv);
    const int64_t g = qb / c->step;
    const int64_t last_row = min64((qb + 1) * c->b_q, n) - 1;
    const int64_t diag = last_row / c->b_kv;
    int64_t cnt = 0;
    if (cnt < cap) blocks[cnt] = 0;
    ++cnt;
    for (int64_t b = ao_window_start_block(g, c); b <= diag && b < t_n; ++b) {
        if (cnt < cap) blocks[cnt] = b;
        ++cnt;
    }
    return cnt;
}

/* R/src/anchor_pass.cpp:37-96 — per query block, per region block, per row:
 * dot (:66-74), block max, alpha = exp(m - m_new) (0 while m = -inf, :77-78),
 * rescale acc, accumulate p * v (:82-90), l = l * alpha + l_block (:91). */
void ao_compute_anchor(int64_t n, int64_t d, const float* q, const float* k, const float* v,
                       const ao_cfg* c, double* m, double* l, double* acc) {
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    const int64_t t_m = ceil_div(n, c->b_q);
    const int64_t t_n = ceil_div(n, c->b_kv);
    for (int64_t i = 0; i < n; ++i) {
        m[i] = -INFINITY;
        l[i] = 0.0;
    }
    memset(acc, 0, (size_t)(n * d) * sizeof(double));
#pragma omp parallel
    {
        double* qk = (double*)malloc((size_t)c->b_kv * sizeof(double));
        int64_t* blocks = (int64_t*)malloc((size_t)(t_n + 2) * sizeof(int64_t));
#pragma omp for schedule(dynamic, 1)
        for (int64_t qb = 0; qb < t_m; ++qb) {
            const int64_t row_begin = qb * c->b_q;
            const int64_t row_end = min64(row_begin + c->b_q, n);
            const int64_t nb = ao_anchor_region(qb, c, n, blocks, t_n + 2);
            for (int64_t bi = 0; bi < nb; ++bi) {
                const int64_t key_begin = blocks[bi] * c->b_kv;
                const int64_t key_end = min64(key_begin + c->b_kv, n);
                for (int64_t i = row_begin; i < row_end; ++i) {
                    const int64_t causal_end = min64(key_end, i + 1);
                    if (key_begin >= causal_end) continue;
                    const float* q_row = q + i * d;
                    double block_max = -INFINITY;
                    for (int64_t j = key_begin; j < causal_end; ++j) {
                        double sum = 0.0;
                        const float* k_row = k + j * d;
                        for (int64_t t = 0; t < d; ++t) sum += (double)q_row[t] * (double)k_row[t];
                        qk[j - key_begin] = sum * inv_sqrt_d;
                        if (qk[j - key_begin] > block_max) block_max = qk[j - key_begin];
                    }
                    const double m_new = m[i] > block_max ? m[i] : block_max;
                    const double alpha = isinf(m[i]) ? 0.0 : exp(m[i] - m_new);
                    double l_block = 0.0;
                    double* acc_row = acc + i * d;
                    for (int64_t t = 0; t < d; ++t) acc_row[t] *= alpha;
                    for (int64_t j = key_begin; j < causal_end; ++j) {
                        const double p = exp(qk[j - key_begin] - m_new);
                        l_block += p;
                        const float* v_row = v + j * d;
                        for (int64_t t = 0; t < d; ++t) acc_row[t] += p * (double)v_row[t];
                    }
                    l[i] = l[i] * alpha + l_block;
                    m[i] = m_new;
                }
            }
        }
        free(qk);
        free(blocks);
    }
}

/* R/src/matrix.cpp:44-65: f64 sums, multiplied by 1/len, rounded to f32. */
void ao_avgpool_rows(int64_t rows, int64_t cols, const float* x, int64_t block, float* out) {
    const int64_t out_rows = ceil_div(rows, block);
    double* sums = (double*)malloc((size_t)cols * sizeof(double));
    for (int64_t g = 0; g < out_rows; ++g) {
        const int64_t begin = g * block;
        const int64_t end = min64(begin + block, rows);
        for (int64_t j = 0; j < cols; ++j) sums[j] = 0.0;
        for (int64_t i = begin; i < end; ++i) {
            const float* row = x + i * cols;
            for (int64_t j = 0; j < cols; ++j) sums[j] += row[j];
        }
        const double inv = 1.0 / (double)(end - begin);
        for (int64_t j = 0; j < cols; ++j) out[g * cols + j] = (float)(sums[j] * inv);
    }
    free(sums);
}

/* R/src/matrix.cpp:67-81: f64 sum divided by len. */
void ao_avgpool_vector(int64_t len, const double* x, int64_t block, double* out) {
    const int64_t out_len = ceil_div(len, block);
    for (int64_t g = 0; g < out_len; ++g) {
        const int64_t begin = g * block;
        const int64_t end = min64(begin + block, len);
        double sum = 0.0;
        for (int64_t i = begin; i < end; ++i) sum += x[i];
        out[g] = sum / (double)(end - begin);
    }
}

/* R/src/stripe_identify.cpp:14-48: q_bar = avgpool_rows(Q, step*b_q); key j of
 * [b_kv, middle_end(g)) is kept iff anchor[g] - dot(q_bar_g, k_j)/sqrt(d) <= theta. */
void ao_identify(int64_t n, int64_t d, const float* q, const float* k, const double* anchor,
                 const ao_cfg* c, uint32_t* idx, int64_t* counts, double* margin_out) {
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    const int64_t groups = ao_group_count(n, c);
    float* pooled = (float*)malloc((size_t)(groups * d) * sizeof(float));
    ao_avgpool_rows(n, d, q, c->step * c->b_q, pooled);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t g = 0; g < groups; ++g) {
        const int64_t off = ao_stripe_offset(g, c, n);
        const int64_t middle_end = ao_middle_end_token(g, c, n);
        int64_t cnt = 0;
        if (middle_end > c->b_kv) {
            const float* q_row = pooled + g * d;
            for (int64_t j = c->b_kv; j < middle_end; ++j) {
                double sum = 0.0;
                const float* k_row = k + j * d;
                for (int64_t t = 0; t < d; ++t) sum += (double)q_row[t] * (double)k_row[t];
                const double diff = anchor[g] - sum * inv_sqrt_d;
                if (margin_out) margin_out[off + (j - c->b_kv)] = diff - c->theta;
                if (diff <= c->theta) idx[off + cnt++] = (uint32_t)j;
            }
        }
        counts[g] = cnt;
    }
    free(pooled);
}

/* R/src/sparse_exec.cpp:13-124 with FoldPlan{chunk, shuffle_seed = 0}:
 * resume (m, l, acc), per row fold each chunk of the group's list, skipping
 * j > i (:79) and anchor-covered j (:82), then O = acc / l (:114-120). */
int64_t ao_sparse_attention(int64_t n, int64_t d, const float* q, const float* k, const float* v,
                            const ao_cfg* c, const double* m_in, const double* l_in,
                            const double* acc_in, const uint32_t* idx, const int64_t* counts,
                            int64_t chunk, float* out) {
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    const int64_t groups = ao_group_count(n, c);
    for (int64_t g = 0; g < groups; ++g) {
        const int64_t off = ao_stripe_offset(g, c, n);
        for (int64_t s = 0; s < counts[g]; ++s)
            if ((int64_t)idx[off + s] >= n) return -1;
    }
    int64_t computed = ao_anchor_covered_count(n, c);
#pragma omp parallel reduction(+ : computed)
    {
        double* qk = (double*)malloc((size_t)chunk * sizeof(double));
        uint32_t* kept = (uint32_t*)malloc((size_t)chunk * sizeof(uint32_t));
        double* acc_row = (double*)malloc((size_t)d * sizeof(double));
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < n; ++i) {
            const int64_t g = i / (c->step * c->b_q);
            const int64_t off = ao_stripe_offset(g, c, n);
            const int64_t cnt = counts[g];
            const int64_t wstart = ao_window_start_token(g, c, n);
            double m = m_in[i], l = l_in[i];
            memcpy(acc_row, acc_in + i * d, (size_t)d * sizeof(double));
            const float* q_row = q + i * d;
            for (int64_t c0 = 0; c0 < cnt; c0 += chunk) {
                const int64_t c1 = min64(c0 + chunk, cnt);
                int64_t taken = 0;
                double chunk_max = -INFINITY;
                for (int64_t s = c0; s < c1; ++s) {
                    const int64_t j = idx[off + s];
                    if (j > i) continue;
                    if (j < c->b_kv || j >= wstart) continue;
                    double sum = 0.0;
                    const float* k_row = k + j * d;
                    for (int64_t t = 0; t < d; ++t) sum += (double)q_row[t] * (double)k_row[t];
                    qk[taken] = sum * inv_sqrt_d;
                    if (qk[taken] > chunk_max) chunk_max = qk[taken];
                    kept[taken] = (uint32_t)j;
                    ++taken;
                }
                if (taken == 0) continue;
                computed += taken;
                const double m_new = m > chunk_max ? m : chunk_max;
                const double alpha = exp(m - m_new);
                for (int64_t t = 0; t < d; ++t) acc_row[t] *= alpha;
                double l_chunk = 0.0;
                for (int64_t s = 0; s < taken; ++s) {
                    const double p = exp(qk[s] - m_new);
                    l_chunk += p;
                    const float* v_row = v + (int64_t)kept[s] * d;
                    for (int64_t t = 0; t < d; ++t) acc_row[t] += p * (double)v_row[t];
                }
                l = l * alpha + l_chunk;
                m = m_new;
            }
            const double inv_l = 1.0 / l;
            for (int64_t t = 0; t < d; ++t) out[i * d + t] = (float)(acc_row[t] * inv_l);
        }
        free(qk);
        free(kept);
        free(acc_row);
    }
    return computed;
}

/* R/src/sparse_exec.cpp:126-133 (+ pooled_anchor, stripe_identify.cpp:71-74). */
int64_t ao_anchor_attention(int64_t n, int64_t d, const float* q, const float* k,
                            const float* v, const ao_cfg* c, int zero_anchor, float* out,
                            double* m_out, double* l_out, uint32_t* idx_out,
                            int64_t* counts_out) {
    const int64_t groups = ao_group_count(n, c);
    const int64_t cap = ao_stripe_capacity(n, c);
    double* m = m_out ? m_out : (double*)malloc((size_t)n * sizeof(double));
    double* l = l_out ? l_out : (double*)malloc((size_t)n * sizeof(double));
    double* acc = (double*)malloc((size_t)(n * d) * sizeof(double));
    double* anchor = (double*)calloc((size_t)groups, sizeof(double));
    uint32_t* idx = idx_out ? idx_out : (uint32_t*)malloc((size_t)(cap > 0 ? cap : 1) * 4);
    int64_t* counts = counts_out ? counts_out : (int64_t*)malloc((size_t)groups * 8);
    ao_compute_anchor(n, d, q, k, v, c, m, l, acc);
    if (!zero_anchor) ao_avgpool_vector(n, m, c->step * c->b_q, anchor);
    ao_identify(n, d, q, k, anchor, c, idx, counts, NULL);
    const int64_t computed = ao_sparse_attention(n, d, q, k, v, c, m, l, acc, idx, counts, 64, out);
    if (!m_out) free(m);
    if (!l_out) free(l);
    if (!idx_out) free(idx);
    if (!counts_out) free(counts);
    free(acc);
    free(anchor);
    return computed;
}

/* R/src/anchor_pass.cpp:120-131 */
void ao_finalize(int64_t n, int64_t d, const double* l, const double* acc, float* out) {
    for (int64_t i = 0; i < n; ++i) {
        const double inv_l = 1.0 / l[i];
        for (int64_t t = 0; t < d; ++t) out[i * d + t] = (float)(acc[i * d + t] * inv_l);
    }
}

/* R/src/oracle.cpp:66-94 */
void ao_dense_attention(int64_t n, int64_t d, const float* q, const float* k, const float* v,
                        float* out) {
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
#pragma omp parallel
    {
        double* logits = (double*)malloc((size_t)n * sizeof(double));
        double* acc = (double*)malloc((size_t)d * sizeof(double));
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < n; ++i) {
            double row_max = -INFINITY;
            for (int64_t j = 0; j <= i; ++j) {
                double sum = 0.0;
                for (int64_t t = 0; t < d; ++t) sum += (double)q[i * d + t] * (double)k[j * d + t];
                logits[j] = sum * inv_sqrt_d;
                if (logits[j] > row_max) row_max = logits[j];
            }
            double denom = 0.0;
            for (int64_t t = 0; t < d; ++t) acc[t] = 0.0;
            for (int64_t j = 0; j <= i; ++j) {
                const double p = exp(logits[j] - row_max);
                denom += p;
                for (int64_t t = 0; t < d; ++t) acc[t] += p * v[j * d + t];
            }
            for (int64_t t = 0; t < d; ++t) out[i * d + t] = (float)(acc[t] / denom);
        }
        free(logits);
        free(acc);
    }
}

/* recall(union_mask(idx), dense_probs) — R/src/metrics.cpp:8-19 over the mask
 * of R/src/sparse_exec.cpp:135-153 and probabilities of R/src/oracle.cpp:38-64
 * (each probability rounded to f32 as dense_probs stores it). */
double ao_union_recall(int64_t n, int64_t d, const float* q, const float* k, const ao_cfg* c,
                       const uint32_t* idx, const int64_t* counts) {
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    double captured = 0.0;
#pragma omp parallel reduction(+ : captured)
    {
        double* logits = (double*)malloc((size_t)n * sizeof(double));
        unsigned char* sel = (unsigned char*)malloc((size_t)n);
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < n; ++i) {
            double row_max = -INFINITY;
            for (int64_t j = 0; j <= i; ++j) {
                double sum = 0.0;
                for (int64_t t = 0; t < d; ++t) sum += (double)q[i * d + t] * (double)k[j * d + t];
                logits[j] = sum * inv_sqrt_d;
                if (logits[j] > row_max) row_max = logits[j];
            }
            double denom = 0.0;
            for (int64_t j = 0; j <= i; ++j) {
                logits[j] = exp(logits[j] - row_max);
                denom += logits[j];
            }
            const int64_t g = i / (c->step * c->b_q);
            const int64_t wstart = ao_window_start_token(g, c, n);
            memset(sel, 0, (size_t)(i + 1));
            for (int64_t j = 0; j < min64(c->b_kv, i + 1); ++j) sel[j] = 1;
            for (int64_t j = wstart; j <= i; ++j) sel[j] = 1;
            const int64_t off = ao_stripe_offset(g, c, n);
            for (int64_t s = 0; s < counts[g]; ++s) {
                const int64_t j = idx[off + s];
                if (j <= i && j >= c->b_kv && j < wstart) sel[j] = 1;
            }
            for (int64_t j = 0; j <= i; ++j)
                if (sel[j]) captured += (double)(float)(logits[j] / denom);
        }
        free(logits);
        free(sel);
    }
    return captured / (double)n;
}
