// Fast path (aa_problem.dtype == AA_BF16): tcgen05 / TMEM / TMA kernels for
// sm_100a with b_q == b_kv == 128 and d == 128.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace aa {

struct FastArgs {
    Geo geo;
    int64_t hq, hkv, rep;
    int64_t q_rs, q_hs, kv_rs, kv_hs;  // element strides (bf16 elements)
    double theta;
    // query groups computed: [g0, g1) (default all); rows of other groups
    // are neither read (q) nor written (state, lists, out)
    int64_t g0, g1;
};

// Records stage event i of aa_set_stage_events on `st` (no-op when unset).
void stage_mark(int i, cudaStream_t st);

// V (bf16, strided) -> packed f16 copy [hkv, n, d] consumed by the PV MMAs;
// values outside the f16 range are counted into *overflow (may be NULL).
cudaError_t fast_convert_v(const FastArgs& f, const void* v, void* v16, cudaStream_t s,
                           unsigned* overflow = nullptr);
// K1 — Alg. 1 anchor pass (tile list {0} ∪ [wsb(g), qb]); writes f32 m, l,
// acc and the per-q-block partial sums qsum [hq, T_m, d] / msum [hq, T_m].
// acc_f16: acc is written as f16 acc / l (the fused chain's hand-off to K3,
// half the bytes; fast_sparse must be given the same flag).
cudaError_t fast_anchor(const FastArgs& f, const void* q, const void* k, const void* v16, float* m,
                        float* l, float* acc, float* qsum, double* msum, cudaStream_t s,
                        bool acc_f16 = false);
// Per-group pooled query (f32) and anchor (f64) from K1 partials (or from
// q / m when the partials are NULL).
cudaError_t fast_pool(const FastArgs& f, const void* q, const float* m, const float* qsum,
                      const double* msum, double* anchor, float* qbar, cudaStream_t s);
// K2 — Alg. 2 scoring + threshold, one selection bit per candidate.
cudaError_t fast_identify(const FastArgs& f, const void* k, const float* qbar,
                          const double* anchor, uint32_t* bits, int64_t words_per_row,
                          cudaStream_t s,
                          void* scratch = nullptr, size_t scratch_bytes = 0);
// Bytes of K2's split A operand (pass as scratch to skip the stream-ordered allocation).
size_t fast_identify_scratch_bytes(const FastArgs& f);
// K3 — Alg. 3 gathered-stripe fold resumed from (m, l, acc).
cudaError_t fast_sparse(const FastArgs& f, const void* q, const void* k, const void* v16,
                        const float* m, const float* l, const float* acc,
                        const uint32_t* indices, const int32_t* counts, const int64_t* offsets,
                        int64_t cap, bool csr, void* out, aa_dtype out_dtype, cudaStream_t s,
                        bool acc_f16 = false);
cudaError_t fast_finalize(const FastArgs& f, const float* l, const float* acc, void* out,
                          aa_dtype out_dtype, cudaStream_t s);
// D — dense causal FlashAttention-style tcgen05 kernel (the speed baseline).
cudaError_t fast_dense(const FastArgs& f, const void* q, const void* k, const void* v16, void* out,
                       aa_dtype out_dtype, cudaStream_t s);
// Exact softmax mass of every (query block, key block) tile of the dense
// causal attention, [hq, T_m, T_n] f32 (two QK-only passes; for the
// block-granularity comparison).
cudaError_t fast_tile_mass(const FastArgs& f, const void* q, const void* k, float* tile_mass,
                           cudaStream_t s);
// Recall of the union mask from one dense pass.
cudaError_t fast_recall(const FastArgs& f, const void* q, const void* k, const uint32_t* indices,
                        const int32_t* counts, const int64_t* offsets, int64_t cap,
                        double* row_captured, double* recall, cudaStream_t s);

}  // namespace aa
