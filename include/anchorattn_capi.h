/*
 * anchorattn_capi.h — C ABI of the B200-native AnchorAttention prefill stack.
 *
 * The drop-in boundary for the reference's operator API.
 * Plain pointers and sizes, status codes instead of exceptions, device
 * pointers plus a CUDA stream; multi-head and GQA-aware (Q head h reads KV
 * head h / (hq / hkv)).  Every entry point names the reference interface it
 * replaces (R/ = /root/reference/proj/).
 *
 * Two arithmetic paths, selected by aa_problem.dtype:
 *   AA_F32  — "exact" path: f32 inputs, f64 state/arithmetic in the
 *             reference's operation order (any b_q, b_kv, step, d).  Results
 *             agree with the reference to f64 round-off; stripe sets are
 *             identical.  SIMT CUDA kernels.
 *   AA_BF16 — "fast" path: bf16 inputs, tcgen05/TMEM/TMA kernels for sm_100a,
 *             f32 state.  Requires b_q == b_kv == 128 and d == 128.
 * There is no CPU fallback: without a CUDA device every call returns
 * AA_ERR_CUDA and aa_last_error() says why.
 *
 * Stripe indices (StripeIndex, R/include/anchorattn/stripe_identify.hpp:14-25)
 * use a CAPACITY layout instead of vector<vector<uint32>>: within a query head,
 * group g owns slots [aa_stripe_offset(p, g), aa_stripe_offset(p, g + 1)) —
 * exactly middle_end(g) - b_kv slots, the most it can select — and
 * counts[h * groups + g] of them are valid, sorted ascending.  No scan pass is
 * needed to place a group's list.
 *
 * Tensor layouts (element strides; 0 = packed head-major):
 *   q        [hq,  n, d]      q_row_stride (default d),  q_head_stride (default n*d)
 *   k, v     [hkv, n, d]      kv_row_stride, kv_head_stride
 *   m, l     [hq, n]          state dtype (aa_plan.state_dtype)
 *   acc      [hq, n, d]       state dtype, UNnormalised (AnchorState::acc)
 *   anchor   [hq, groups]     f64   (pooled_anchor)
 *   qbar     [hq, groups, d]  f32   (avgpool_rows(Q, step*b_q))
 *   indices  [hq, capacity]   u32
 *   counts   [hq, groups]     i32
 *   out      [hq, n, d]       out_dtype (AA_F32 or AA_BF16)
 *   computed [hq]             i64   (RunStats::computed_positions per head)
 */
#ifndef ANCHORATTN_CAPI_H
#define ANCHORATTN_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* aa_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum aa_status {
    AA_OK = 0,
    AA_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    AA_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range (stripe index >= n)   */
    AA_ERR_UNSUPPORTED = 3,      /* shape outside the selected path          */
    AA_ERR_CUDA = 4              /* CUDA runtime / launch failure            */
} aa_status;

typedef enum aa_dtype { AA_F32 = 0, AA_BF16 = 1, AA_F64 = 2 } aa_dtype;

/* BlockConfig (R/include/anchorattn/matrix.hpp:53-62). */
typedef struct aa_block_config {
    int64_t b_q;
    int64_t b_kv;
    int64_t step;
    double theta;
} aa_block_config;

typedef struct aa_problem {
    int64_t n, d;   /* sequence length, head dim (HeadWorkload n, d)          */
    int64_t hq;     /* query heads                                            */
    int64_t hkv;    /* key/value heads, hq % hkv == 0                          */
    aa_block_config cfg;
    aa_dtype dtype; /* AA_F32 (exact path) or AA_BF16 (tcgen05 path)           */
    int64_t q_row_stride, q_head_stride;   /* elements; 0 = packed            */
    int64_t kv_row_stride, kv_head_stride; /* elements; 0 = packed            */
} aa_problem;

typedef struct aa_plan {
    int64_t q_blocks;          /* ceil(n / b_q)                                 */
    int64_t groups;            /* group_count(n, cfg)                           */
    aa_dtype state_dtype;      /* AA_F64 (exact path) or AA_F32 (fast path)     */
    int64_t stripe_capacity;   /* slots per query head                          */
    int64_t covered_positions; /* anchor_covered_count(n, cfg), per head        */
    size_t workspace_bytes;    /* scratch for aa_anchor_attention / aa_identify */
} aa_plan;

/* Last error message of the calling thread (reference exception text). */
const char* aa_last_error(void);
const char* aa_version(void);

/* BlockConfig::validate (R/src/matrix.cpp:31-42). */
aa_status aa_config_validate(const aa_block_config* cfg);

/* Geometry helpers, host side, pure (R/src/detail/geometry.hpp:22-85;
 * anchor_region R/src/anchor_pass.cpp:12-30; group_count / middle_end_token
 * R/src/stripe_identify.cpp:56-67; anchor_covered_count
 * R/src/anchor_pass.cpp:113-118). */
int64_t aa_group_count(int64_t n, const aa_block_config* cfg);
int64_t aa_window_start_token(int64_t group, const aa_block_config* cfg, int64_t n);
int64_t aa_middle_end_token(int64_t group, const aa_block_config* cfg, int64_t n);
int64_t aa_anchor_covered_count(int64_t n, const aa_block_config* cfg);
/* Writes up to cap block ids, returns the full count (or -1: q_block out of range). */
int64_t aa_anchor_region(int64_t q_block, const aa_block_config* cfg, int64_t n,
                         int64_t* blocks, int64_t cap);
/* Slot base of `group` in a head's capacity-layout index list (group may be
 * == groups, giving the capacity). */
int64_t aa_stripe_offset(int64_t group, const aa_block_config* cfg, int64_t n);

/* Validates the problem for its path and fills the plan. */
aa_status aa_make_plan(const aa_problem* p, aa_plan* plan);

/* Alg. 1 — compute_anchor (R/src/anchor_pass.cpp:37-96).  Writes m, l, acc
 * (state dtype).  qsum/msum are optional (may be NULL) per-query-block
 * partial sums [hq, q_blocks, d] f32 / [hq, q_blocks] f64 that let aa_pool
 * skip re-reading Q (fast path only; ignored by the exact path). */
aa_status aa_compute_anchor(const aa_problem* p, const void* q, const void* k, const void* v,
                            void* m, void* l, void* acc, float* qsum, double* msum,
                            aa_stream_t stream);

/* pooled_anchor (R/src/stripe_identify.cpp:71-74) and avgpool_rows(Q,
 * step*b_q) (R/src/matrix.cpp:44-65, called at stripe_identify.cpp:25).
 * Uses qsum/msum when non-NULL, else reads q / m. */
aa_status aa_pool(const aa_problem* p, const void* q, const void* m, const float* qsum,
                  const double* msum, double* anchor, float* qbar, aa_stream_t stream);

/* Alg. 2 — identify_stripes / identify_stripes_zero_anchor
 * (R/src/stripe_identify.cpp:14-48,76-95).  anchor may be NULL when
 * zero_anchor != 0.  workspace: >= aa_plan.workspace_bytes. */
aa_status aa_identify(const aa_problem* p, const void* k, const float* qbar,
                      const double* anchor, int zero_anchor, uint32_t* indices,
                      int32_t* counts, void* workspace, size_t workspace_bytes,
                      aa_stream_t stream);

/* Alg. 3 — sparse_attention (R/src/sparse_exec.cpp:13-124).  Resumes (m, l,
 * acc), folds each group's listed stripes, writes O = acc / l.
 * offsets: NULL for the capacity layout, else a device CSR table
 * [hq * groups + 1] of list starts (counts gives the lengths).  Lists may hold
 * any indices, as the reference's StripeIndex may:
 *   - an index >= n fails with AA_ERR_OUT_OF_RANGE and the reference's text
 *     "sparse_attention: stripe index N out of range" (sparse_exec.cpp:51-56;
 *     the first such index in (head, group, position) order);
 *   - entries outside [b_kv, window_start(g)) (anchor-covered or non-causal)
 *     are skipped and duplicates fold twice, as sparse_exec.cpp:79-82 does —
 *     the exact path per row inside the reference's chunks; the fast path
 *     compacts each list on the device first (order kept) and folds 128-key
 *     tiles.
 * The lists are validated on the device before any output is written, so
 * this call synchronizes `stream` (the fused aa_anchor_attention does not).
 * fold_chunk is FoldPlan::index_chunk for the exact path (ignored by the fast
 * path).  computed may be NULL. */
aa_status aa_sparse_attention(const aa_problem* p, const void* q, const void* k, const void* v,
                              const void* m, const void* l, const void* acc,
                              const uint32_t* indices, const int32_t* counts,
                              const int64_t* offsets, int64_t fold_chunk, void* out,
                              aa_dtype out_dtype, int64_t* computed, aa_stream_t stream);

/* finalize_anchor (R/src/anchor_pass.cpp:120-131): out = acc / l. */
aa_status aa_finalize_anchor(const aa_problem* p, const void* l, const void* acc, void* out,
                             aa_dtype out_dtype, aa_stream_t stream);

/* anchor_attention (R/src/sparse_exec.cpp:126-133): the whole chain on device
 * buffers.  workspace >= aa_plan.workspace_bytes (holds state, pooled values
 * and stripe lists).  computed may be NULL. */
aa_status aa_anchor_attention(const aa_problem* p, const void* q, const void* k, const void* v,
                              int zero_anchor, void* out, aa_dtype out_dtype, int64_t* computed,
                              void* workspace, size_t workspace_bytes, aa_stream_t stream);

/* The same chain for the query groups [group_begin, group_end) of every head
 * only (groups of step * b_q rows, R/src/detail/geometry.hpp:36-47): reads
 * their q rows and K/V rows [0, row_end(group_end - 1)), writes their rows of
 * out, and computed[h] = the positions those rows compute.  Groups are
 * independent given the K/V prefix (R/../SPEC.md), so a layer split into
 * group ranges — e.g. balanced multi-GPU shards of a head
 * (paper_2505_23520_b200.sharding.shard_work) — reproduces the whole-layer
 * result bit for bit.  bf16 (tcgen05) path only. */
aa_status aa_anchor_attention_groups(const aa_problem* p, int64_t group_begin, int64_t group_end,
                                     const void* q, const void* k, const void* v, int zero_anchor,
                                     void* out, aa_dtype out_dtype, int64_t* computed,
                                     void* workspace, size_t workspace_bytes, aa_stream_t stream);

/* Same chain on HOST buffers (the reference's value-semantics calling
 * convention, bindings.cpp:21-32): copies q/k/v in, runs, copies out and the
 * per-head computed counts back; blocks until done.  Device buffers, streams
 * and events are cached per device across calls (calls on one device are
 * serialized; several devices may be driven from one process).  The bf16
 * path fails with AA_ERR_UNSUPPORTED when V holds values outside the f16
 * range (|v| > 65504, see below).  The copies are pipelined against the
 * chain over up to 32 chunks — blocks of KV heads, or runs of one KV head's
 * query heads when there are fewer KV heads than chunks — on copy-in, compute
 * and copy-out streams, so with page-locked host buffers the PCIe traffic
 * overlaps the kernels. */
aa_status aa_anchor_attention_host(const aa_problem* p, const void* q, const void* k,
                                   const void* v, int zero_anchor, void* out, aa_dtype out_dtype,
                                   int64_t* computed);

/* Numerical range of the bf16 (tcgen05) path: PV runs in f16 (V converted
 * bf16 -> f16 once, exact for 6.1e-5 <= |v| <= 65504; smaller magnitudes lose
 * relative, not absolute, precision) and the fused chain hands K1's state to
 * K3 as f16 acc / l (|.| <= max |v|).  V outside that range gives non-finite
 * outputs; aa_anchor_attention_host detects it, the device-buffer entries do
 * not check (use AA_F32 for such data). */

/* Dense causal attention (oracle.cpp:66-94 semantics) — the baseline the
 * sparse path is measured against (exact path: f64; fast path: tcgen05). */
aa_status aa_dense_attention(const aa_problem* p, const void* q, const void* k, const void* v,
                             void* out, aa_dtype out_dtype, aa_stream_t stream);

/* recall(union_mask(stripes), dense_probs) per head (metrics.cpp:8-19 over
 * sparse_exec.cpp:135-153) without materialising the n x n map: one dense
 * pass keeping (max, sum over all keys, sum over selected keys) per row.
 * recall [hq] f64. */
aa_status aa_union_recall(const aa_problem* p, const void* q, const void* k,
                          const uint32_t* indices, const int32_t* counts, double* recall,
                          aa_stream_t stream);

/* Softmax mass of every (query block, key block) tile of dense causal
 * attention: tile_mass [hq, ceil(n/b_q), ceil(n/b_kv)] f32, row-normalised
 * probabilities summed over the tile (the block-granularity score map of
 * R/src/baselines.cpp:62-83, pooled_score_map, computed without the n x n
 * map).  Fast path only (AA_BF16). */
aa_status aa_dense_tile_mass(const aa_problem* p, const void* q, const void* k,
                             float* tile_mass, aa_stream_t stream);

/* Stage timing for profilers/benchmarks: while set, the fast path of
 * aa_anchor_attention records events[i] (cudaEvent_t) on its stream at the
 * stage boundaries 0 start | 1 V->f16 | 2 K1 anchor | 3 pool + K2 identify +
 * compaction | 4 K3 sparse | 5 stats, and (count >= 8) 6 / 7 right before /
 * after the K2 identify kernel itself.  Per calling thread; NULL disables. */
aa_status aa_set_stage_events(void* const* events, int count);

/* Plumbing for host callers that do not link the CUDA runtime themselves. */
aa_status aa_stream_sync(aa_stream_t stream);
aa_status aa_device_alloc(size_t bytes, void** ptr);
aa_status aa_device_free(void* ptr);
aa_status aa_copy_to_device(void* dst, const void* src, size_t bytes);   /* blocking */
aa_status aa_copy_to_host(void* dst, const void* src, size_t bytes);     /* blocking */
aa_status aa_device_count(int* count);

#ifdef __cplusplus
}
#endif

#endif /* ANCHORATTN_CAPI_H */
