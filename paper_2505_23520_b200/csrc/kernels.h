// Internal launch interface between capi.cu and the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace aa {

struct ExactArgs {
    Geo geo;
    int64_t d, hq, hkv, rep;
    int64_t q_rs, q_hs, kv_rs, kv_hs;  // element strides
    double inv_sqrt_d, theta;
};

// ---- exact path (exact_kernels.cu) ----
cudaError_t launch_anchor_exact(const ExactArgs& a, const float* q, const float* k,
                                const float* v, double* m, double* l, double* acc, cudaStream_t s);
cudaError_t launch_pool_exact(const ExactArgs& a, const float* q, const double* m,
                              double* anchor, float* qbar, cudaStream_t s);
cudaError_t launch_identify_exact(const ExactArgs& a, const float* k, const float* qbar,
                                  const double* anchor, uint32_t* bits, int64_t words_per_row,
                                  cudaStream_t s);
cudaError_t launch_sparse_exact(const ExactArgs& a, const float* q, const float* k,
                                const float* v, const double* m, const double* l,
                                const double* acc, const uint32_t* indices, const int32_t* counts,
                                const int64_t* offsets, int64_t cap, bool csr, int64_t chunk,
                                void* out, aa_dtype out_dtype, unsigned long long* computed,
                                cudaStream_t s);
cudaError_t launch_finalize_exact(const ExactArgs& a, const double* l, const double* acc,
                                  void* out, aa_dtype out_dtype, cudaStream_t s);
cudaError_t launch_dense_exact(const ExactArgs& a, const float* q, const float* k,
                               const float* v, void* out, aa_dtype out_dtype, cudaStream_t s);
cudaError_t launch_recall_exact(const ExactArgs& a, const float* q, const float* k,
                                const uint32_t* indices, const int32_t* counts,
                                const int64_t* offsets, int64_t cap, double* row_captured,
                                double* recall, cudaStream_t s);

// ---- shared (common_kernels.cu) ----
// Ordered stream compaction of the per-(head, group) selection bitmask into
// the capacity-layout index lists (ballot/popc + block scan).
// Rows of groups [g0, g1) (g1 < 0: all groups).
cudaError_t launch_compact(const Geo& geo, int64_t hq, const uint32_t* bits,
                           int64_t words_per_row, const int64_t* offsets, int64_t cap,
                           uint32_t* indices, int32_t* counts, cudaStream_t s, int64_t g0 = 0,
                           int64_t g1 = -1);
// RunStats::computed_positions per head = covered + sum_g counts[h,g]*rows(g)
// (R/tests/test_sparse_exec.cpp:106-121 accounting identity).
// (over groups [g0, g1); covered = the anchor positions of those rows)
cudaError_t launch_computed(const Geo& geo, int64_t hq, int64_t covered, const int32_t* counts,
                            int64_t* computed, cudaStream_t s, int64_t g0 = 0, int64_t g1 = -1);
// offsets[g] = stripe_offset(g) for g in [0, groups] (capacity layout).
cudaError_t launch_offsets(const Geo& geo, int64_t* offsets, cudaStream_t s);
// Stage-API list check / filter (see k_filter_lists): folded entries of each
// caller list into out_idx at out_off (out_idx NULL = check only) and the
// first out-of-range entry's (row << 32 | position) into *first_bad.
cudaError_t launch_filter_lists(const Geo& geo, int64_t hq, const uint32_t* idx,
                                const int32_t* counts, const int64_t* offsets, int64_t cap,
                                bool csr, const int64_t* out_off, uint32_t* out_idx,
                                int32_t* out_counts, unsigned long long* first_bad,
                                cudaStream_t s);
cudaError_t launch_add_u64(int64_t hq, int64_t covered, const unsigned long long* taken,
                           int64_t* computed, cudaStream_t s);

}  // namespace aa
