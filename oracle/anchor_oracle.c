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

/* Dot products of one f32 query row against KT_W keys held transposed as
 * f64 kt[t * KT_W + u]: the loop over t is outermost, so the KT_W running
 * sums vectorise across keys while each key's sum still adds its d products
 * in index order t = 0 .. d-1 — the reference's order (anchor_pass.cpp:66-72,
 * stripe_identify.cpp:35-40, sparse_exec.cpp:85-92).  The product of two f32
 * values is exact in f64, so every sum equals the sequential scalar loop bit
 * for bit; only the evaluation order across DIFFERENT keys changes. */
#define KT_W 32

static void kt_load(const float* k, int64_t d, const int64_t* rows, int64_t cnt, double* kt) {
    for (int64_t t = 0; t < d; ++t)
        for (int64_t u = 0; u < KT_W; ++u)
            kt[t * KT_W + u] = u < cnt ? (double)k[rows[u] * d + t] : 0.0;
}

static void kt_load_range(const float* k, int64_t d, int64_t j0, int64_t cnt, double* kt) {
    for (int64_t t = 0; t < d; ++t)
        for (int64_t u = 0; u < KT_W; ++u)
            kt[t * KT_W + u] = u < cnt ? (double)k[(j0 + u) * d + t] : 0.0;
}

static void kt_dots(const float* q_row, int64_t d, const double* kt, double* out) {
    double s[KT_W];
    for (int u = 0; u < KT_W; ++u) s[u] = 0.0;
    for (int64_t t = 0; t < d; ++t) {
        const double qt = (double)q_row[t];
        const double* kr = kt + t * KT_W;
        for (int u = 0; u < KT_W; ++u) s[u] += qt * kr[u];
    }
    for (int u = 0; u < KT_W; ++u) out[u] = s[u];
}

/* R/src/anchor_pass.cpp:37-96 — per query block, per region block, per row:
 * dot (:66-74), block max, alpha = exp(m - m_new) (0 while m = -inf, :77-78),
 * rescale acc, accumulate p * v (:82-90), l = l * alpha + l_block (:91).
 * The region block's keys are transposed once (kt_load_range) and shared by
 * the block's rows. */
void ao_compute_anchor(int64_t n, int64_t d, const float* q, const float* k, const float* v,
                       const ao_cfg* c, double* m, double* l, double* acc) {
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    const int64_t t_m = ceil_div(n, c->b_q);
    const int64_t t_n = ceil_div(n, c->b_kv);
    const int64_t nsub = ceil_div(c->b_kv, KT_W);
    for (int64_t i = 0; i < n; ++i) {
        m[i] = -INFINITY;
        l[i] = 0.0;
    }
    memset(acc, 0, (size_t)(n * d) * sizeof(double));
#pragma omp parallel
    {
        double* qk = (double*)malloc((size_t)(nsub * KT_W) * sizeof(double));
        double* kt = (double*)malloc((size_t)(nsub * KT_W * d) * sizeof(double));
        int64_t* blocks = (int64_t*)malloc((size_t)(t_n + 2) * sizeof(int64_t));
#pragma omp for schedule(dynamic, 1)
        for (int64_t qb = 0; qb < t_m; ++qb) {
            const int64_t row_begin = qb * c->b_q;
            const int64_t row_end = min64(row_begin + c->b_q, n);
            const int64_t nb = ao_anchor_region(qb, c, n, blocks, t_n + 2);
            for (int64_t bi = 0; bi < nb; ++bi) {
                const int64_t key_begin = blocks[bi] * c->b_kv;
                const int64_t key_end = min64(key_begin + c->b_kv, n);
                for (int64_t sb = 0; sb < nsub; ++sb) {
                    const int64_t j0 = key_begin + sb * KT_W;
                    if (j0 < key_end) kt_load_range(k, d, j0, min64(KT_W, key_end - j0), kt + sb * KT_W * d);
                }
                for (int64_t i = row_begin; i < row_end; ++i) {
                    const int64_t causal_end = min64(key_end, i + 1);
                    if (key_begin >= causal_end) continue;
                    const int64_t cols = causal_end - key_begin;
                    for (int64_t sb = 0; sb * KT_W < cols; ++sb)
                        kt_dots(q + i * d, d, kt + sb * KT_W * d, qk + sb * KT_W);
                    double block_max = -INFINITY;
                    for (int64_t jj = 0; jj < cols; ++jj) {
                        qk[jj] = qk[jj] * inv_sqrt_d;
                        if (qk[jj] > block_max) block_max = qk[jj];
                    }
                    const double m_new = m[i] > block_max ? m[i] : block_max;
                    const double alpha = isinf(m[i]) ? 0.0 : exp(m[i] - m_new);
                    double l_block = 0.0;
                    double* acc_row = acc + i * d;
                    for (int64_t t = 0; t < d; ++t) acc_row[t] *= alpha;
                    for (int64_t jj = 0; jj < cols; ++jj) {
                        const double p = exp(qk[jj] - m_new);
                        l_block += p;
                        const float* v_row = v + (key_begin + jj) * d;
                        for (int64_t t = 0; t < d; ++t) acc_row[t] += p * (double)v_row[t];
                    }
                    l[i] = l[i] * alpha + l_block;
                    m[i] = m_new;
                }
            }
        }
        free(qk);
        free(kt);
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
 * j > i (:79) and anchor-covered j (:82), then O = acc / l (:114-120).
 *
 * The kept entries of a chunk do not depend on the row: a listed j is folded
 * iff b_kv <= j < window_start(g), and a non-empty [b_kv, window_start(g))
 * implies window_start(g) <= row_begin(g) - b_kv (geometry.hpp:55-64), so
 * j < i for every row of the group.  Each chunk is therefore filtered once
 * and its keys transposed once per block of ROWS rows. */
#define ROWS 16

/* Group g's list is idx[offs[g] .. offs[g] + counts[g]). */
static int64_t sparse_core(int64_t n, int64_t d, const float* q, const float* k, const float* v,
                           const ao_cfg* c, const double* m_in, const double* l_in,
                           const double* acc_in, const uint32_t* idx, const int64_t* offs,
                           const int64_t* counts, int64_t chunk, float* out) {
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    const int64_t groups = ao_group_count(n, c);
    const int64_t rows_per_group = c->step * c->b_q;
    int64_t* kept_n = (int64_t*)calloc((size_t)(groups > 0 ? groups : 1), sizeof(int64_t));
    for (int64_t g = 0; g < groups; ++g)
        for (int64_t s = 0; s < counts[g]; ++s)
            if ((int64_t)idx[offs[g] + s] >= n) {
                free(kept_n);
                return -1;
            }
    int64_t computed = ao_anchor_covered_count(n, c);
    for (int64_t g = 0; g < groups; ++g) {
        const int64_t wstart = ao_window_start_token(g, c, n);
        for (int64_t s = 0; s < counts[g]; ++s) {
            const int64_t j = idx[offs[g] + s];
            if (j >= c->b_kv && j < wstart) ++kept_n[g];
        }
        computed += kept_n[g] * (min64((g + 1) * rows_per_group, n) - g * rows_per_group);
    }
    const int64_t row_blocks = ceil_div(rows_per_group, ROWS);
    const int64_t nsub = ceil_div(chunk, KT_W);
#pragma omp parallel
    {
        double* qk = (double*)malloc((size_t)(ROWS * nsub * KT_W) * sizeof(double));
        double* kt = (double*)malloc((size_t)(KT_W * d) * sizeof(double));
        int64_t* kept = (int64_t*)malloc((size_t)(nsub * KT_W) * sizeof(int64_t));
        double* acc_rows = (double*)malloc((size_t)(ROWS * d) * sizeof(double));
        double ms[ROWS], ls[ROWS];
#pragma omp for schedule(dynamic, 1)
        for (int64_t w = 0; w < groups * row_blocks; ++w) {
            const int64_t g = w / row_blocks;
            const int64_t r0 = g * rows_per_group + (w % row_blocks) * ROWS;
            const int64_t r1 = min64(min64(r0 + ROWS, (g + 1) * rows_per_group), n);
            if (r0 >= r1) continue;
            const int64_t nr = r1 - r0;
            const int64_t off = offs[g];
            const int64_t cnt = counts[g];
            const int64_t wstart = ao_window_start_token(g, c, n);
            for (int64_t r = 0; r < nr; ++r) {
                ms[r] = m_in[r0 + r];
                ls[r] = l_in[r0 + r];
                memcpy(acc_rows + r * d, acc_in + (r0 + r) * d, (size_t)d * sizeof(double));
            }
            for (int64_t c0 = 0; c0 < cnt; c0 += chunk) {
                const int64_t c1 = min64(c0 + chunk, cnt);
                int64_t taken = 0;
                for (int64_t s = c0; s < c1; ++s) {
                    const int64_t j = idx[off + s];
                    if (j < c->b_kv || j >= wstart) continue;
                    kept[taken++] = j;
                }
                if (taken == 0) continue;
                for (int64_t sb = 0; sb * KT_W < taken; ++sb) {
                    kt_load(k, d, kept + sb * KT_W, min64(KT_W, taken - sb * KT_W), kt);
                    for (int64_t r = 0; r < nr; ++r)
                        kt_dots(q + (r0 + r) * d, d, kt, qk + r * nsub * KT_W + sb * KT_W);
                }
                for (int64_t r = 0; r < nr; ++r) {
                    double* qr = qk + r * nsub * KT_W;
                    double* acc_row = acc_rows + r * d;
                    double chunk_max = -INFINITY;
                    for (int64_t s = 0; s < taken; ++s) {
                        qr[s] = qr[s] * inv_sqrt_d;
                        if (qr[s] > chunk_max) chunk_max = qr[s];
                    }
                    const double m_new = ms[r] > chunk_max ? ms[r] : chunk_max;
                    const double alpha = exp(ms[r] - m_new);
                    for (int64_t t = 0; t < d; ++t) acc_row[t] *= alpha;
                    double l_chunk = 0.0;
                    for (int64_t s = 0; s < taken; ++s) {
                        const double p = exp(qr[s] - m_new);
                        l_chunk += p;
                        const float* v_row = v + kept[s] * d;
                        for (int64_t t = 0; t < d; ++t) acc_row[t] += p * (double)v_row[t];
                    }
                    ls[r] = ls[r] * alpha + l_chunk;
                    ms[r] = m_new;
                }
            }
            for (int64_t r = 0; r < nr; ++r) {
                const double inv_l = 1.0 / ls[r];
                for (int64_t t = 0; t < d; ++t)
                    out[(r0 + r) * d + t] = (float)(acc_rows[r * d + t] * inv_l);
            }
        }
        free(qk);
        free(kt);
        free(kept);
        free(acc_rows);
    }
    free(kept_n);
    return computed;
}

int64_t ao_sparse_attention(int64_t n, int64_t d, const float* q, const float* k, const float* v,
                            const ao_cfg* c, const double* m_in, const double* l_in,
                            const double* acc_in, const uint32_t* idx, const int64_t* counts,
                            int64_t chunk, float* out) {
    const int64_t groups = ao_group_count(n, c);
    int64_t* offs = (int64_t*)malloc((size_t)(groups + 1) * sizeof(int64_t));
    offs[0] = 0;
    for (int64_t g = 0; g < groups; ++g) offs[g + 1] = offs[g] + middle_len(g, c, n);
    const int64_t r = sparse_core(n, d, q, k, v, c, m_in, l_in, acc_in, idx, offs, counts, chunk, out);
    free(offs);
    return r;
}

int64_t ao_sparse_attention_lists(int64_t n, int64_t d, const float* q, const float* k,
                                  const float* v, const ao_cfg* c, const double* m_in,
                                  const double* l_in, const double* acc_in, const uint32_t* idx,
                                  const int64_t* starts, const int64_t* counts, int64_t chunk,
                                  float* out) {
    return sparse_core(n, d, q, k, v, c, m_in, l_in, acc_in, idx, starts, counts, chunk, out);
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

/* Causal logits of rows [r0, r1) against keys [0, r1 - 1], row r at
 * logits[(r - r0) * n + j]: key sub-blocks transposed once per row block. */
static void causal_logits(int64_t n, int64_t d, const float* q, const float* k, int64_t r0,
                          int64_t r1, double inv_sqrt_d, double* kt, double* logits) {
    double tmp[KT_W];
    for (int64_t j0 = 0; j0 < r1; j0 += KT_W) {
        const int64_t cnt = min64(KT_W, r1 - j0);
        kt_load_range(k, d, j0, cnt, kt);
        for (int64_t i = max64(r0, j0); i < r1; ++i) {
            kt_dots(q + i * d, d, kt, tmp);
            double* lr = logits + (i - r0) * n;
            for (int64_t u = 0; u < cnt && j0 + u <= i; ++u) lr[j0 + u] = tmp[u] * inv_sqrt_d;
        }
    }
}

/* R/src/oracle.cpp:66-94 */
void ao_dense_attention(int64_t n, int64_t d, const float* q, const float* k, const float* v,
                        float* out) {
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    const int64_t nblk = ceil_div(n, ROWS);
#pragma omp parallel
    {
        double* logits = (double*)malloc((size_t)(ROWS * n) * sizeof(double));
        double* kt = (double*)malloc((size_t)(KT_W * d) * sizeof(double));
        double* acc = (double*)malloc((size_t)d * sizeof(double));
#pragma omp for schedule(dynamic, 1)
        for (int64_t b = 0; b < nblk; ++b) {
            const int64_t r0 = (nblk - 1 - b) * ROWS, r1 = min64(r0 + ROWS, n);
            causal_logits(n, d, q, k, r0, r1, inv_sqrt_d, kt, logits);
            for (int64_t i = r0; i < r1; ++i) {
                const double* lr = logits + (i - r0) * n;
                double row_max = -INFINITY;
                for (int64_t j = 0; j <= i; ++j)
                    if (lr[j] > row_max) row_max = lr[j];
                double denom = 0.0;
                for (int64_t t = 0; t < d; ++t) acc[t] = 0.0;
                for (int64_t j = 0; j <= i; ++j) {
                    const double p = exp(lr[j] - row_max);
                    denom += p;
                    for (int64_t t = 0; t < d; ++t) acc[t] += p * v[j * d + t];
                }
                for (int64_t t = 0; t < d; ++t) out[i * d + t] = (float)(acc[t] / denom);
            }
        }
        free(logits);
        free(kt);
        free(acc);
    }
}

/* recall(union_mask(idx), dense_probs) — R/src/metrics.cpp:8-19 over the mask
 * of R/src/sparse_exec.cpp:135-153 and probabilities of R/src/oracle.cpp:38-64
 * (each probability rounded to f32 as dense_probs stores it).  The per-row
 * captured masses are summed in row order. */
double ao_union_recall(int64_t n, int64_t d, const float* q, const float* k, const ao_cfg* c,
                       const uint32_t* idx, const int64_t* counts) {
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    const int64_t nblk = ceil_div(n, ROWS);
    double* row_cap = (double*)malloc((size_t)n * sizeof(double));
#pragma omp parallel
    {
        double* logits = (double*)malloc((size_t)(ROWS * n) * sizeof(double));
        double* kt = (double*)malloc((size_t)(KT_W * d) * sizeof(double));
        unsigned char* sel = (unsigned char*)malloc((size_t)n);
#pragma omp for schedule(dynamic, 1)
        for (int64_t b = 0; b < nblk; ++b) {
            const int64_t r0 = (nblk - 1 - b) * ROWS, r1 = min64(r0 + ROWS, n);
            causal_logits(n, d, q, k, r0, r1, inv_sqrt_d, kt, logits);
            for (int64_t i = r0; i < r1; ++i) {
                double* lr = logits + (i - r0) * n;
                double row_max = -INFINITY;
                for (int64_t j = 0; j <= i; ++j)
                    if (lr[j] > row_max) row_max = lr[j];
                double denom = 0.0;
                for (int64_t j = 0; j <= i; ++j) {
                    lr[j] = exp(lr[j] - row_max);
                    denom += lr[j];
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
                double captured = 0.0;
                for (int64_t j = 0; j <= i; ++j)
                    if (sel[j]) captured += (double)(float)(lr[j] / denom);
                row_cap[i] = captured;
            }
        }
        free(logits);
        free(kt);
        free(sel);
    }
    double captured = 0.0;
    for (int64_t i = 0; i < n; ++i) captured += row_cap[i];
    free(row_cap);
    return captured / (double)n;
}
