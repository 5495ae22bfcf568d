/*
 * TEST INFRASTRUCTURE ONLY — CPU parity oracle for the AnchorAttention
 * prefill path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library; the product path never does.
 *
 * Plain-C restatement of the reference algorithm (f64 arithmetic over f32
 * storage, exactly as R/src (the reference sources)).  Parity of this
 * restatement is pinned against oracle/_ref (the reference compiled from its
 * own sources) through tests/golden/ fixtures and tests/test_oracle_golden.py.
 *
 * Stripe lists use the "capacity layout": group g of a head owns the slots
 * [stripe_offset(g), stripe_offset(g) + (middle_end(g) - b_kv)) and
 * counts[g] of them are valid, sorted ascending.
 */
#ifndef ANCHOR_ORACLE_H
#define ANCHOR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t b_q;
    int64_t b_kv;
    int64_t step;
    double theta;
} ao_cfg;

/* BlockConfig::validate (matrix.cpp:31-42). 0 on success, 1 on error. */
int ao_validate(const ao_cfg* cfg);

/* detail:: geometry (geometry.hpp:22-85). */
int64_t ao_group_count(int64_t n, const ao_cfg* cfg);
int64_t ao_window_start_block(int64_t g, const ao_cfg* cfg);
int64_t ao_window_start_token(int64_t g, const ao_cfg* cfg, int64_t n);
int64_t ao_middle_end_token(int64_t g, const ao_cfg* cfg, int64_t n);
int64_t ao_covered_count_for_row(int64_t row, const ao_cfg* cfg, int64_t n);
int64_t ao_anchor_covered_count(int64_t n, const ao_cfg* cfg);
int64_t ao_stripe_capacity(int64_t n, const ao_cfg* cfg);
int64_t ao_stripe_offset(int64_t g, const ao_cfg* cfg, int64_t n);
/* anchor_region (anchor_pass.cpp:12-30); returns count written to blocks. */
int64_t ao_anchor_region(int64_t q_block, const ao_cfg* cfg, int64_t n, int64_t* blocks,
                         int64_t cap);

/* compute_anchor (anchor_pass.cpp:37-96): m, l [n]; acc [n*d] unnormalised. */
void ao_compute_anchor(int64_t n, int64_t d, const float* q, const float* k, const float* v,
                       const ao_cfg* cfg, double* m, double* l, double* acc);

/* avgpool_rows (matrix.cpp:44-65) -> f32 [ceil(n/block) x d]. */
void ao_avgpool_rows(int64_t rows, int64_t cols, const float* x, int64_t block, float* out);
/* avgpool_vector (matrix.cpp:67-81). */
void ao_avgpool_vector(int64_t len, const double* x, int64_t block, double* out);

/* identify_with_reference (stripe_identify.cpp:14-48).  anchor: [G] (pass
 * zeros for identify_stripes_zero_anchor).  idx in capacity layout, counts
 * [G].  Optional score_out (may be NULL) receives anchor - s per candidate in
 * capacity layout (for the +-1e-3 band test). */
void ao_identify(int64_t n, int64_t d, const float* q, const float* k, const double* anchor,
                 const ao_cfg* cfg, uint32_t* idx, int64_t* counts, double* margin_out);

/* sparse_attention (sparse_exec.cpp:13-124) with FoldPlan{chunk, 0}.  idx in
 * capacity layout.  Returns computed_positions; -1 on out-of-range index. */
int64_t ao_sparse_attention(int64_t n, int64_t d, const float* q, const float* k, const float* v,
                            const ao_cfg* cfg, const double* m, const double* l,
                            const double* acc, const uint32_t* idx, const int64_t* counts,
                            int64_t chunk, float* out);

/* Same over arbitrary per-group lists (a StripeIndex of any lengths): group
 * g's list is idx[starts[g] .. starts[g] + counts[g]). */
int64_t ao_sparse_attention_lists(int64_t n, int64_t d, const float* q, const float* k,
                                  const float* v, const ao_cfg* cfg, const double* m,
                                  const double* l, const double* acc, const uint32_t* idx,
                                  const int64_t* starts, const int64_t* counts, int64_t chunk,
                                  float* out);

/* anchor_attention (sparse_exec.cpp:126-133): the whole chain. Returns
 * computed_positions.  If state/idx buffers are non-NULL they are filled. */
int64_t ao_anchor_attention(int64_t n, int64_t d, const float* q, const float* k,
                            const float* v, const ao_cfg* cfg, int zero_anchor, float* out,
                            double* m_out, double* l_out, uint32_t* idx_out,
                            int64_t* counts_out);

/* finalize_anchor (anchor_pass.cpp:120-131). */
void ao_finalize(int64_t n, int64_t d, const double* l, const double* acc, float* out);

/* Dense causal oracle (oracle.cpp:66-94) and recall of the union mask
 * (metrics.cpp:8-19 over sparse_exec.cpp:135-153), computed row by row
 * without materialising the n x n map. */
void ao_dense_attention(int64_t n, int64_t d, const float* q, const float* k, const float* v,
                        float* out);
double ao_union_recall(int64_t n, int64_t d, const float* q, const float* k, const ao_cfg* cfg,
                       const uint32_t* idx, const int64_t* counts);

#ifdef __cplusplus
}
#endif

#endif
