// C ABI implementation (include/anchorattn_capi.h): validation with the
// reference's exception texts, path dispatch, workspace carving and the
// host-buffer entry point.  No computation happens on the host: every entry
// that produces values launches CUDA kernels and fails with AA_ERR_CUDA when
// no device is present.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/anchorattn_capi.h"
#include "common.cuh"
#include "fast.h"
#include "kernels.h"

namespace {

thread_local std::string g_err;
// Optional per-stage timing events (aa_set_stage_events).
thread_local void* const* g_events = nullptr;
thread_local int g_nevents = 0;

void mark(int i, cudaStream_t st) {
    if (i < g_nevents && g_events[i]) cudaEventRecord(static_cast<cudaEvent_t>(g_events[i]), st);
}
}  // namespace

namespace aa {
void stage_mark(int i, cudaStream_t st) { mark(i, st); }
}  // namespace aa

namespace {

aa_status fail(aa_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

aa_status cuda_fail(cudaError_t e, const char* where) {
    return fail(AA_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define AA_CUDA(call)                                                  \
    do {                                                               \
        cudaError_t e_ = (call);                                       \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);            \
    } while (0)

aa::Geo geo_of(int64_t n, const aa_block_config& c) { return aa::Geo{n, c.b_q, c.b_kv, c.step}; }

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Selection-bitmask row pitch in 32-bit words (multiple of 4: 16-byte stores).
int64_t words_per_row(int64_t n) { return ((n + 31) / 32 + 3) / 4 * 4; }

aa::FastArgs fast_args(const aa_problem& p);

// Buffers of the fused chain, carved from one workspace.
struct Carve {
    size_t off = 0;
    char* base = nullptr;
    void* take(size_t bytes) {
        void* p = base ? base + off : nullptr;
        off += align256(bytes);
        return p;
    }
};

struct Layout {
    void *m, *l, *acc, *qsum, *msum, *anchor, *qbar, *offsets, *bits, *indices, *counts, *taken,
        *v16, *split, *flags;
    size_t split_bytes;
    int64_t words_per_row;
    size_t total;
};

Layout carve(const aa_problem& p, const aa_plan& plan, void* ws) {
    Carve c;
    c.base = static_cast<char*>(ws);
    Layout L{};
    const size_t se = plan.state_dtype == AA_F64 ? 8 : 4;
    const size_t hq = static_cast<size_t>(p.hq), n = static_cast<size_t>(p.n),
                 d = static_cast<size_t>(p.d), G = static_cast<size_t>(plan.groups),
                 T = static_cast<size_t>(plan.q_blocks);
    L.words_per_row = words_per_row(p.n);
    L.m = c.take(hq * n * se);
    L.l = c.take(hq * n * se);
    // the fused fast chain hands K1's state to K3 as f16 acc / l (half the
    // bytes of the f32 AnchorState::acc the stage API returns)
    L.acc = c.take(hq * n * d * (p.dtype == AA_BF16 ? 2 : se));
    L.qsum = c.take(hq * T * d * 4);
    L.msum = c.take(hq * T * 8);
    L.anchor = c.take(hq * G * 8);
    L.qbar = c.take(hq * G * d * 4);
    L.offsets = c.take((G + 1) * 8);
    L.bits = c.take(hq * G * static_cast<size_t>(L.words_per_row) * 4);
    L.indices = c.take(hq * static_cast<size_t>(plan.stripe_capacity > 0 ? plan.stripe_capacity : 1) * 4);
    L.counts = c.take(hq * G * 4);
    L.taken = c.take(hq * 8);
    L.v16 = p.dtype == AA_BF16 ? c.take(static_cast<size_t>(p.hkv) * n * d * 2) : nullptr;
    // K2's split A operand (q_bar = hi + lo, bf16) of the fast path
    L.split_bytes = p.dtype == AA_BF16 ? aa::fast_identify_scratch_bytes(fast_args(p)) : 0;
    L.split = L.split_bytes ? c.take(L.split_bytes) : nullptr;
    L.flags = c.take(8);  // fast path: count of V values outside the f16 range
    L.total = c.off;
    return L;
}

aa::ExactArgs exact_args(const aa_problem& p) {
    aa::ExactArgs a{};
    a.geo = geo_of(p.n, p.cfg);
    a.d = p.d;
    a.hq = p.hq;
    a.hkv = p.hkv;
    a.rep = p.hq / p.hkv;
    a.q_rs = p.q_row_stride ? p.q_row_stride : p.d;
    a.q_hs = p.q_head_stride ? p.q_head_stride : p.n * a.q_rs;
    a.kv_rs = p.kv_row_stride ? p.kv_row_stride : p.d;
    a.kv_hs = p.kv_head_stride ? p.kv_head_stride : p.n * a.kv_rs;
    a.inv_sqrt_d = 1.0 / std::sqrt(static_cast<double>(p.d));
    a.theta = p.cfg.theta;
    return a;
}

aa::FastArgs fast_args(const aa_problem& p) {
    aa::FastArgs f{};
    f.geo = geo_of(p.n, p.cfg);
    f.hq = p.hq;
    f.hkv = p.hkv;
    f.rep = p.hq / p.hkv;
    f.q_rs = p.q_row_stride ? p.q_row_stride : p.d;
    f.q_hs = p.q_head_stride ? p.q_head_stride : p.n * f.q_rs;
    f.kv_rs = p.kv_row_stride ? p.kv_row_stride : p.d;
    f.kv_hs = p.kv_head_stride ? p.kv_head_stride : p.n * f.kv_rs;
    f.theta = p.cfg.theta;
    f.g0 = 0;
    f.g1 = f.geo.groups();
    return f;
}

// Anchor-covered positions of the rows of groups [g0, g1) (per head).
int64_t covered_in_groups(const aa::Geo& G, int64_t g0, int64_t g1) {
    int64_t total = 0;
    for (int64_t i = G.row_begin(g0); i < G.row_end(g1 - 1); ++i) total += G.covered_count_for_row(i);
    return total;
}

// Stream-ordered temporary (cudaMallocAsync pool) freed on scope exit.
struct Temp {
    void* p = nullptr;
    cudaStream_t s;
    explicit Temp(cudaStream_t st) : s(st) {}
    cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes ? bytes : 1, s); }
    ~Temp() {
        if (p) cudaFreeAsync(p, s);
    }
};

aa_status require_device() {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(AA_ERR_CUDA, std::string("no CUDA device available (") +
                                     cudaGetErrorString(e) +
                                     "); anchorattn has no CPU fallback");
    // Stage-API temporaries come from the stream-ordered pool; keep its memory
    // mapped across synchronisations (the default threshold 0 unmaps it at
    // every sync and the next cudaMallocAsync remaps, a host stall).
    static thread_local int pooled_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev != pooled_dev) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        pooled_dev = dev;
    }
    return AA_OK;
}

}  // namespace

extern "C" {

const char* aa_last_error(void) { return g_err.c_str(); }
const char* aa_version(void) { return "anchorattn-b200 0.1 (sm_100a)"; }

aa_status aa_config_validate(const aa_block_config* c) {
    if (!c) return fail(AA_ERR_INVALID_ARGUMENT, "BlockConfig: null");
    // R/src/matrix.cpp:31-42
    if (c->b_q <= 0 || c->b_kv <= 0 || c->step <= 0)
        return fail(AA_ERR_INVALID_ARGUMENT, "BlockConfig: b_q, b_kv, step must be >= 1");
    if (c->b_q % c->b_kv != 0 && c->b_kv % c->b_q != 0)
        return fail(AA_ERR_INVALID_ARGUMENT,
                    "BlockConfig: one of b_q, b_kv must divide the other");
    if (!std::isfinite(c->theta))
        return fail(AA_ERR_INVALID_ARGUMENT, "BlockConfig: theta must be finite");
    return AA_OK;
}

int64_t aa_group_count(int64_t n, const aa_block_config* c) { return geo_of(n, *c).groups(); }
int64_t aa_window_start_token(int64_t g, const aa_block_config* c, int64_t n) {
    return geo_of(n, *c).window_start(g);
}
int64_t aa_middle_end_token(int64_t g, const aa_block_config* c, int64_t n) {
    return geo_of(n, *c).middle_end(g);
}
int64_t aa_anchor_covered_count(int64_t n, const aa_block_config* c) {
    const aa::Geo G = geo_of(n, *c);
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) total += G.covered_count_for_row(i);
    return total;
}
int64_t aa_anchor_region(int64_t qb, const aa_block_config* c, int64_t n, int64_t* blocks,
                         int64_t cap) {
    const aa::Geo G = geo_of(n, *c);
    if (qb < 0 || qb >= G.q_blocks()) {
        g_err = "anchor_region: query block out of range";
        return -1;
    }
    const int64_t last_row = ((qb + 1) * c->b_q < n ? (qb + 1) * c->b_q : n) - 1;
    const int64_t diag = last_row / c->b_kv;
    int64_t cnt = 0;
    if (cnt < cap) blocks[cnt] = 0;
    ++cnt;
    for (int64_t b = G.window_start_block(qb / c->step); b <= diag && b < G.kv_blocks(); ++b) {
        if (cnt < cap) blocks[cnt] = b;
        ++cnt;
    }
    return cnt;
}
int64_t aa_stripe_offset(int64_t g, const aa_block_config* c, int64_t n) {
    return geo_of(n, *c).stripe_offset(g);
}

aa_status aa_make_plan(const aa_problem* p, aa_plan* plan) {
    if (!p || !plan) return fail(AA_ERR_INVALID_ARGUMENT, "aa_make_plan: null argument");
    if (aa_status s = aa_config_validate(&p->cfg)) return s;
    if (p->n < 1 || p->d < 1)
        return fail(AA_ERR_INVALID_ARGUMENT, "HeadWorkload: n and d must be >= 1");
    if (p->n > (int64_t(1) << 31) - 1)
        return fail(AA_ERR_UNSUPPORTED, "n must fit 32-bit key indices (StripeIndex is uint32)");
    if (p->hq < 1 || p->hkv < 1 || p->hq % p->hkv != 0)
        return fail(AA_ERR_INVALID_ARGUMENT, "heads: hq must be a positive multiple of hkv");
    if (p->dtype == AA_BF16) {
        if (p->cfg.b_q != 128 || p->cfg.b_kv != 128 || p->d != 128)
            return fail(AA_ERR_UNSUPPORTED,
                        "bf16 tcgen05 path requires b_q == b_kv == 128 and d == 128");
        const int64_t qrs = p->q_row_stride ? p->q_row_stride : p->d;
        const int64_t krs = p->kv_row_stride ? p->kv_row_stride : p->d;
        const int64_t khs = p->kv_head_stride ? p->kv_head_stride : p->n * krs;
        if ((qrs * 2) % 16 || krs % p->d || khs % p->d)
            return fail(AA_ERR_UNSUPPORTED,
                        "bf16 path: q row stride must be a 16-byte multiple and k/v strides "
                        "multiples of d (TMA gather rows)");
    } else if (p->dtype != AA_F32) {
        return fail(AA_ERR_UNSUPPORTED, "dtype must be AA_F32 (exact) or AA_BF16 (fast)");
    }
    const aa::Geo G = geo_of(p->n, p->cfg);
    plan->q_blocks = G.q_blocks();
    plan->groups = G.groups();
    plan->state_dtype = p->dtype == AA_BF16 ? AA_F32 : AA_F64;
    plan->stripe_capacity = G.stripe_offset(G.groups());
    plan->covered_positions = aa_anchor_covered_count(p->n, &p->cfg);
    plan->workspace_bytes = 0;
    plan->workspace_bytes = carve(*p, *plan, nullptr).total;
    return AA_OK;
}

aa_status aa_stream_sync(aa_stream_t stream) {
    AA_CUDA(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)));
    return AA_OK;
}

aa_status aa_device_count(int* count) {
    *count = 0;
    const cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return cuda_fail(e, "cudaGetDeviceCount");
    }
    return AA_OK;
}

aa_status aa_device_alloc(size_t bytes, void** ptr) {
    if (aa_status s = require_device()) return s;
    AA_CUDA(cudaMalloc(ptr, bytes ? bytes : 1));
    return AA_OK;
}

aa_status aa_device_free(void* ptr) {
    if (ptr) AA_CUDA(cudaFree(ptr));
    return AA_OK;
}

aa_status aa_copy_to_device(void* dst, const void* src, size_t bytes) {
    if (bytes) AA_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    return AA_OK;
}

aa_status aa_copy_to_host(void* dst, const void* src, size_t bytes) {
    if (bytes) AA_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    return AA_OK;
}

// ------------------------------------------------------------------ stages

aa_status aa_compute_anchor(const aa_problem* p, const void* q, const void* k, const void* v,
                            void* m, void* l, void* acc, float* qsum, double* msum,
                            aa_stream_t stream) {
    aa_plan plan;
    if (aa_status s = aa_make_plan(p, &plan)) return s;
    if (aa_status s = require_device()) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (p->dtype == AA_F32) {
        AA_CUDA(aa::launch_anchor_exact(exact_args(*p), static_cast<const float*>(q),
                                        static_cast<const float*>(k), static_cast<const float*>(v),
                                        static_cast<double*>(m), static_cast<double*>(l),
                                        static_cast<double*>(acc), st));
    } else {
        const aa::FastArgs f = fast_args(*p);
        Temp v16(st);
        AA_CUDA(v16.alloc(static_cast<size_t>(p->hkv * p->n * p->d) * 2));
        AA_CUDA(aa::fast_convert_v(f, v, v16.p, st));
        AA_CUDA(aa::fast_anchor(f, q, k, v16.p, static_cast<float*>(m), static_cast<float*>(l),
                                static_cast<float*>(acc), qsum, msum, st));
    }
    return AA_OK;
}

aa_status aa_pool(const aa_problem* p, const void* q, const void* m, const float* qsum,
                  const double* msum, double* anchor, float* qbar, aa_stream_t stream) {
    aa_plan plan;
    if (aa_status s = aa_make_plan(p, &plan)) return s;
    if (aa_status s = require_device()) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (p->dtype == AA_F32) {
        AA_CUDA(aa::launch_pool_exact(exact_args(*p), static_cast<const float*>(q),
                                      static_cast<const double*>(m), anchor, qbar, st));
    } else {
        AA_CUDA(aa::fast_pool(fast_args(*p), q, static_cast<const float*>(m), qsum, msum, anchor,
                              qbar, st));
    }
    return AA_OK;
}

static aa_status identify_impl(const aa_problem* p, const aa_plan& plan, const void* k,
                               const float* qbar, const double* anchor, int zero_anchor,
                               uint32_t* indices, int32_t* counts, int64_t* offsets_dev,
                               uint32_t* bits, int64_t words_per_row, cudaStream_t st,
                               void* scratch = nullptr, size_t scratch_bytes = 0,
                               int64_t g0 = 0, int64_t g1 = -1) {
    const aa::Geo G = geo_of(p->n, p->cfg);
    if (g1 < 0) g1 = G.groups();
    const double* ref = zero_anchor ? nullptr : anchor;
    if (p->dtype == AA_F32) {
        AA_CUDA(aa::launch_identify_exact(exact_args(*p), static_cast<const float*>(k), qbar, ref,
                                          bits, words_per_row, st));
    } else {
        aa::FastArgs f = fast_args(*p);
        f.g0 = g0;
        f.g1 = g1;
        AA_CUDA(aa::fast_identify(f, k, qbar, ref, bits, words_per_row, st, scratch, scratch_bytes));
    }
    AA_CUDA(aa::launch_offsets(G, offsets_dev, st));
    AA_CUDA(aa::launch_compact(G, p->hq, bits, words_per_row, offsets_dev,
                               plan.stripe_capacity > 0 ? plan.stripe_capacity : 1, indices,
                               counts, st, g0, g1));
    return AA_OK;
}

aa_status aa_identify(const aa_problem* p, const void* k, const float* qbar,
                      const double* anchor, int zero_anchor, uint32_t* indices, int32_t* counts,
                      void* workspace, size_t workspace_bytes, aa_stream_t stream) {
    aa_plan plan;
    if (aa_status s = aa_make_plan(p, &plan)) return s;
    if (!zero_anchor && !anchor)
        return fail(AA_ERR_INVALID_ARGUMENT, "aa_identify: anchor required unless zero_anchor");
    if (aa_status s = require_device()) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t wpr = words_per_row(p->n);
    const size_t need = align256(static_cast<size_t>(plan.groups + 1) * 8) +
                        static_cast<size_t>(p->hq * plan.groups * wpr) * 4;
    Temp tmp(st);
    char* base = static_cast<char*>(workspace);
    if (!workspace || workspace_bytes < need) {
        AA_CUDA(tmp.alloc(need));
        base = static_cast<char*>(tmp.p);
    }
    int64_t* offs = reinterpret_cast<int64_t*>(base);
    uint32_t* bits = reinterpret_cast<uint32_t*>(base + align256(static_cast<size_t>(plan.groups + 1) * 8));
    return identify_impl(p, plan, k, qbar, anchor, zero_anchor, indices, counts, offs, bits, wpr,
                         st);
}

aa_status aa_sparse_attention(const aa_problem* p, const void* q, const void* k, const void* v,
                              const void* m, const void* l, const void* acc,
                              const uint32_t* indices, const int32_t* counts,
                              const int64_t* offsets, int64_t fold_chunk, void* out,
                              aa_dtype out_dtype, int64_t* computed, aa_stream_t stream) {
    aa_plan plan;
    if (aa_status s = aa_make_plan(p, &plan)) return s;
    if (fold_chunk < 1)
        return fail(AA_ERR_INVALID_ARGUMENT, "sparse_attention: index_chunk must be >= 1");
    if (out_dtype != AA_F32 && out_dtype != AA_BF16)
        return fail(AA_ERR_INVALID_ARGUMENT, "out_dtype must be AA_F32 or AA_BF16");
    if (aa_status s = require_device()) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const aa::Geo G = geo_of(p->n, p->cfg);
    const int64_t groups = plan.groups, rows = p->hq * groups;
    const int64_t cap = plan.stripe_capacity > 0 ? plan.stripe_capacity : 1;
    const bool fast = p->dtype == AA_BF16;
    // The caller's lists are checked on the device first (R/src/sparse_exec.cpp:51-56:
    // an index >= n is std::out_of_range, reported for the first one in
    // (head, group, position) order); the fast path then folds 128-key tiles
    // of the entries the reference folds (:79-82), compacted per list.
    std::vector<int32_t> hcounts(static_cast<size_t>(rows));
    if (rows > 0)
        AA_CUDA(cudaMemcpyAsync(hcounts.data(), counts, hcounts.size() * 4, cudaMemcpyDeviceToHost, st));
    AA_CUDA(cudaStreamSynchronize(st));
    std::vector<int64_t> hoff(static_cast<size_t>(rows) + 1, 0);
    int64_t max_count = 1;
    for (int64_t r = 0; r < rows; ++r) {
        max_count = std::max<int64_t>(max_count, hcounts[r]);
        if (hcounts[r] < 0)
            return fail(AA_ERR_INVALID_ARGUMENT, "sparse_attention: negative stripe count");
        hoff[r + 1] = hoff[r] + hcounts[r];
    }
    const size_t off_b = align256(static_cast<size_t>(groups + 1) * 8);
    const size_t coff_b = align256(hoff.size() * 8);
    const size_t cnt_b = align256(static_cast<size_t>(rows) * 4 + 4);
    const size_t idx_b = fast ? align256(static_cast<size_t>(hoff[rows]) * 4 + 4) : 0;
    Temp tmp(st);
    AA_CUDA(tmp.alloc(off_b + coff_b + cnt_b + idx_b + align256(static_cast<size_t>(p->hq) * 8) + 256));
    char* base = static_cast<char*>(tmp.p);
    int64_t* offs = reinterpret_cast<int64_t*>(base);
    int64_t* coff = reinterpret_cast<int64_t*>(base + off_b);
    int32_t* fcounts = reinterpret_cast<int32_t*>(base + off_b + coff_b);
    uint32_t* fidx = fast ? reinterpret_cast<uint32_t*>(base + off_b + coff_b + cnt_b) : nullptr;
    unsigned long long* taken =
        reinterpret_cast<unsigned long long*>(base + off_b + coff_b + cnt_b + idx_b);
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(
        base + off_b + coff_b + cnt_b + idx_b + align256(static_cast<size_t>(p->hq) * 8));
    if (!offsets) AA_CUDA(aa::launch_offsets(G, offs, st));
    const int64_t* offs_used = offsets ? offsets : offs;
    AA_CUDA(cudaMemcpyAsync(coff, hoff.data(), hoff.size() * 8, cudaMemcpyHostToDevice, st));
    AA_CUDA(cudaMemsetAsync(bad, 0xff, 8, st));
    AA_CUDA(aa::launch_filter_lists(G, p->hq, indices, counts, offs_used, cap, offsets != nullptr,
                                    coff, fidx, fast ? fcounts : nullptr, bad, st));
    unsigned long long hbad = 0;
    AA_CUDA(cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, st));
    AA_CUDA(cudaStreamSynchronize(st));
    if (hbad != ~0ull) {
        const int64_t row = static_cast<int64_t>(hbad >> 32), pos = static_cast<int64_t>(hbad & 0xffffffffull);
        const int64_t h = row / groups, g = row % groups;
        int64_t start = 0;
        if (offsets) {
            AA_CUDA(cudaMemcpy(&start, offsets + row, 8, cudaMemcpyDeviceToHost));
        } else {
            start = h * cap + G.stripe_offset(g);
        }
        uint32_t j = 0;
        AA_CUDA(cudaMemcpy(&j, indices + start + pos, 4, cudaMemcpyDeviceToHost));
        return fail(AA_ERR_OUT_OF_RANGE,
                    "sparse_attention: stripe index " + std::to_string(j) + " out of range");
    }
    if (!fast) {
        AA_CUDA(cudaMemsetAsync(taken, 0, static_cast<size_t>(p->hq) * 8, st));
        AA_CUDA(aa::launch_sparse_exact(
            exact_args(*p), static_cast<const float*>(q), static_cast<const float*>(k),
            static_cast<const float*>(v), static_cast<const double*>(m),
            static_cast<const double*>(l), static_cast<const double*>(acc), indices, counts,
            offs_used, offsets ? 0 : cap, offsets != nullptr,
            // a chunk longer than every list folds each list in one chunk,
            // exactly as the requested chunk does (it bounds shared memory)
            std::min(fold_chunk, max_count), out, out_dtype, taken, st));
        if (computed)
            AA_CUDA(aa::launch_add_u64(p->hq, plan.covered_positions, taken, computed, st));
    } else {
        const aa::FastArgs f = fast_args(*p);
        Temp v16(st);
        AA_CUDA(v16.alloc(static_cast<size_t>(p->hkv * p->n * p->d) * 2));
        AA_CUDA(aa::fast_convert_v(f, v, v16.p, st));
        AA_CUDA(aa::fast_sparse(f, q, k, v16.p, static_cast<const float*>(m),
                                static_cast<const float*>(l), static_cast<const float*>(acc), fidx,
                                fcounts, coff, 0, true, out, out_dtype, st));
        if (computed)
            AA_CUDA(aa::launch_computed(G, p->hq, plan.covered_positions, fcounts, computed, st));
    }
    return AA_OK;
}

aa_status aa_finalize_anchor(const aa_problem* p, const void* l, const void* acc, void* out,
                             aa_dtype out_dtype, aa_stream_t stream) {
    aa_plan plan;
    if (aa_status s = aa_make_plan(p, &plan)) return s;
    if (aa_status s = require_device()) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (p->dtype == AA_F32) {
        AA_CUDA(aa::launch_finalize_exact(exact_args(*p), static_cast<const double*>(l),
                                          static_cast<const double*>(acc), out, out_dtype, st));
    } else {
        AA_CUDA(aa::fast_finalize(fast_args(*p), static_cast<const float*>(l),
                                  static_cast<const float*>(acc), out, out_dtype, st));
    }
    return AA_OK;
}

// The fast path's fused chain (V->f16, K1, pool, K2 + compaction, K3,
// stats) over the query groups [g0, g1) of every head.
static aa_status fused_fast(const aa_problem* p, const aa_plan& plan, const Layout& L,
                            const void* q, const void* k, const void* v, int zero_anchor,
                            void* out, aa_dtype out_dtype, int64_t* computed, cudaStream_t st,
                            int64_t g0, int64_t g1) {
    const aa::Geo G = geo_of(p->n, p->cfg);
    const int64_t cap = plan.stripe_capacity > 0 ? plan.stripe_capacity : 1;
    aa::FastArgs f = fast_args(*p);
    f.g0 = g0;
    f.g1 = g1;
    mark(0, st);
    AA_CUDA(cudaMemsetAsync(L.flags, 0, 8, st));
    AA_CUDA(aa::fast_convert_v(f, v, L.v16, st, static_cast<unsigned*>(L.flags)));
    mark(1, st);
    AA_CUDA(aa::fast_anchor(f, q, k, L.v16, static_cast<float*>(L.m), static_cast<float*>(L.l),
                            static_cast<float*>(L.acc), static_cast<float*>(L.qsum),
                            static_cast<double*>(L.msum), st, /*acc_f16=*/true));
    mark(2, st);
    AA_CUDA(aa::fast_pool(f, q, static_cast<float*>(L.m), static_cast<float*>(L.qsum),
                          static_cast<double*>(L.msum), static_cast<double*>(L.anchor),
                          static_cast<float*>(L.qbar), st));
    if (aa_status s = identify_impl(p, plan, k, static_cast<float*>(L.qbar),
                                    static_cast<double*>(L.anchor), zero_anchor,
                                    static_cast<uint32_t*>(L.indices),
                                    static_cast<int32_t*>(L.counts),
                                    static_cast<int64_t*>(L.offsets),
                                    static_cast<uint32_t*>(L.bits), L.words_per_row, st, L.split,
                                    L.split_bytes, g0, g1))
        return s;
    mark(3, st);
    AA_CUDA(aa::fast_sparse(f, q, k, L.v16, static_cast<float*>(L.m), static_cast<float*>(L.l),
                            static_cast<float*>(L.acc), static_cast<uint32_t*>(L.indices),
                            static_cast<int32_t*>(L.counts), static_cast<int64_t*>(L.offsets), cap,
                            false, out, out_dtype, st, /*acc_f16=*/true));
    mark(4, st);
    if (computed) {
        const int64_t covered = (g0 == 0 && g1 == plan.groups) ? plan.covered_positions
                                                               : covered_in_groups(G, g0, g1);
        AA_CUDA(aa::launch_computed(G, p->hq, covered, static_cast<int32_t*>(L.counts), computed, st,
                                    g0, g1));
    }
    mark(5, st);
    return AA_OK;
}

aa_status aa_anchor_attention(const aa_problem* p, const void* q, const void* k, const void* v,
                              int zero_anchor, void* out, aa_dtype out_dtype, int64_t* computed,
                              void* workspace, size_t workspace_bytes, aa_stream_t stream) {
    aa_plan plan;
    if (aa_status s = aa_make_plan(p, &plan)) return s;
    if (out_dtype != AA_F32 && out_dtype != AA_BF16)
        return fail(AA_ERR_INVALID_ARGUMENT, "out_dtype must be AA_F32 or AA_BF16");
    if (aa_status s = require_device()) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Temp tmp(st);
    if (!workspace || workspace_bytes < plan.workspace_bytes) {
        if (workspace)
            return fail(AA_ERR_INVALID_ARGUMENT, "aa_anchor_attention: workspace too small");
        AA_CUDA(tmp.alloc(plan.workspace_bytes));
        workspace = tmp.p;
    }
    const Layout L = carve(*p, plan, workspace);
    const aa::Geo G = geo_of(p->n, p->cfg);
    const int64_t cap = plan.stripe_capacity > 0 ? plan.stripe_capacity : 1;
    if (p->dtype == AA_F32) {
        const aa::ExactArgs a = exact_args(*p);
        AA_CUDA(aa::launch_anchor_exact(a, static_cast<const float*>(q),
                                        static_cast<const float*>(k), static_cast<const float*>(v),
                                        static_cast<double*>(L.m), static_cast<double*>(L.l),
                                        static_cast<double*>(L.acc), st));
        AA_CUDA(aa::launch_pool_exact(a, static_cast<const float*>(q),
                                      static_cast<const double*>(L.m),
                                      static_cast<double*>(L.anchor), static_cast<float*>(L.qbar),
                                      st));
        if (aa_status s = identify_impl(p, plan, k, static_cast<float*>(L.qbar),
                                        static_cast<double*>(L.anchor), zero_anchor,
                                        static_cast<uint32_t*>(L.indices),
                                        static_cast<int32_t*>(L.counts),
                                        static_cast<int64_t*>(L.offsets),
                                        static_cast<uint32_t*>(L.bits), L.words_per_row, st))
            return s;
        AA_CUDA(cudaMemsetAsync(L.taken, 0, static_cast<size_t>(p->hq) * 8, st));
        AA_CUDA(aa::launch_sparse_exact(
            a, static_cast<const float*>(q), static_cast<const float*>(k),
            static_cast<const float*>(v), static_cast<double*>(L.m), static_cast<double*>(L.l),
            static_cast<double*>(L.acc), static_cast<uint32_t*>(L.indices),
            static_cast<int32_t*>(L.counts), static_cast<int64_t*>(L.offsets), cap, false, 64,
            out, out_dtype, static_cast<unsigned long long*>(L.taken), st));
        if (computed)
            AA_CUDA(aa::launch_add_u64(p->hq, plan.covered_positions,
                                       static_cast<unsigned long long*>(L.taken), computed, st));
        return AA_OK;
    }
    return fused_fast(p, plan, L, q, k, v, zero_anchor, out, out_dtype, computed, st, 0,
                      plan.groups);
}

aa_status aa_anchor_attention_groups(const aa_problem* p, int64_t group_begin, int64_t group_end,
                                     const void* q, const void* k, const void* v, int zero_anchor,
                                     void* out, aa_dtype out_dtype, int64_t* computed,
                                     void* workspace, size_t workspace_bytes, aa_stream_t stream) {
    aa_plan plan;
    if (aa_status s = aa_make_plan(p, &plan)) return s;
    if (p->dtype != AA_BF16)
        return fail(AA_ERR_UNSUPPORTED, "aa_anchor_attention_groups: bf16 (tcgen05) path only");
    if (group_begin < 0 || group_end > plan.groups || group_begin >= group_end)
        return fail(AA_ERR_INVALID_ARGUMENT, "aa_anchor_attention_groups: empty or out-of-range group range");
    if (out_dtype != AA_F32 && out_dtype != AA_BF16)
        return fail(AA_ERR_INVALID_ARGUMENT, "out_dtype must be AA_F32 or AA_BF16");
    if (aa_status s = require_device()) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Temp tmp(st);
    if (!workspace || workspace_bytes < plan.workspace_bytes) {
        if (workspace)
            return fail(AA_ERR_INVALID_ARGUMENT, "aa_anchor_attention_groups: workspace too small");
        AA_CUDA(tmp.alloc(plan.workspace_bytes));
        workspace = tmp.p;
    }
    const Layout L = carve(*p, plan, workspace);
    return fused_fast(p, plan, L, q, k, v, zero_anchor, out, out_dtype, computed, st, group_begin,
                      group_end);
}

aa_status aa_set_stage_events(void* const* events, int count) {
    g_events = events;
    g_nevents = events ? count : 0;
    return AA_OK;
}

aa_status aa_dense_tile_mass(const aa_problem* p, const void* q, const void* k,
                             float* tile_mass, aa_stream_t stream) {
    aa_plan plan;
    if (aa_status s = aa_make_plan(p, &plan)) return s;
    if (p->dtype != AA_BF16)
        return fail(AA_ERR_UNSUPPORTED, "aa_dense_tile_mass: bf16 (tcgen05) path only");
    if (aa_status s = require_device()) return s;
    AA_CUDA(aa::fast_tile_mass(fast_args(*p), q, k, tile_mass,
                               reinterpret_cast<cudaStream_t>(stream)));
    return AA_OK;
}

aa_status aa_anchor_attention_host(const aa_problem* p, const void* q, const void* k,
                                   const void* v, int zero_anchor, void* out, aa_dtype out_dtype,
                                   int64_t* computed) {
    // Pipelined over KV-head chunks (heads are independent, R/../SPEC.md:269):
    // chunk c's inputs go up on the copy-in stream while chunk c-1 computes and
    // chunk c-2's output comes back on the copy-out stream, so the PCIe
    // transfers (both directions at once) hide the chain instead of adding to it.
    // Cached per device (streams, events and buffers belong to one device
    // context; a process may drive several GPUs one after another).
    constexpr int kMaxChunks = 32;
    constexpr int kMaxDevices = 64;
    struct DeviceState {
        std::mutex mu;
        void* dbuf = nullptr;
        size_t dbytes = 0;
        cudaStream_t st_in = nullptr, st_c = nullptr, st_out = nullptr;
        cudaEvent_t ev_in[kMaxChunks], ev_done[kMaxChunks];
        unsigned* v_flags = nullptr;  // pinned: per-chunk V-range counts
    };
    static DeviceState states[kMaxDevices];
    int dev_id = 0;
    if (aa_status s = require_device()) return s;
    AA_CUDA(cudaGetDevice(&dev_id));
    if (dev_id < 0 || dev_id >= kMaxDevices)
        return fail(AA_ERR_UNSUPPORTED, "aa_anchor_attention_host: device ordinal >= 64");
    DeviceState& ds = states[dev_id];
    std::lock_guard<std::mutex> lock(ds.mu);
    void*& dbuf = ds.dbuf;
    size_t& dbytes = ds.dbytes;
    cudaStream_t &st_in = ds.st_in, &st_c = ds.st_c, &st_out = ds.st_out;
    cudaEvent_t* ev_in = ds.ev_in;
    cudaEvent_t* ev_done = ds.ev_done;
    aa_plan plan;
    if (aa_status s = aa_make_plan(p, &plan)) return s;
    if (out_dtype != AA_F32 && out_dtype != AA_BF16)
        return fail(AA_ERR_INVALID_ARGUMENT, "out_dtype must be AA_F32 or AA_BF16");
    const auto packed = [&](int64_t s, int64_t want) { return s == 0 || s == want; };
    if (!packed(p->q_row_stride, p->d) || !packed(p->q_head_stride, p->n * p->d) ||
        !packed(p->kv_row_stride, p->d) || !packed(p->kv_head_stride, p->n * p->d))
        return fail(AA_ERR_UNSUPPORTED, "aa_anchor_attention_host: packed layouts only");
    if (!st_c) {
        AA_CUDA(cudaStreamCreateWithFlags(&st_in, cudaStreamNonBlocking));
        AA_CUDA(cudaStreamCreateWithFlags(&st_c, cudaStreamNonBlocking));
        AA_CUDA(cudaStreamCreateWithFlags(&st_out, cudaStreamNonBlocking));
        for (int c = 0; c < kMaxChunks; ++c) {
            AA_CUDA(cudaEventCreateWithFlags(&ev_in[c], cudaEventDisableTiming));
            AA_CUDA(cudaEventCreateWithFlags(&ev_done[c], cudaEventDisableTiming));
        }
        AA_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ds.v_flags), kMaxChunks * sizeof(unsigned),
                              cudaHostAllocDefault));
    }
    const int64_t rep = p->hkv > 0 ? p->hq / p->hkv : 1;
    // Chunks: blocks of whole KV heads, or — with fewer KV heads than chunks
    // (e.g. one KV head per rank under sharding) — runs of one KV head's
    // query heads, the first run of each KV head carrying its K / V copy.
    struct Chunk {
        int64_t kv0, nkv, h0, nh;
        bool copy_kv;
    };
    std::vector<Chunk> chunks;
    int64_t max_nkv = 0, max_nh = 0;
    if (p->hkv >= kMaxChunks || rep == 1) {
        const int64_t per = p->hkv > 0 ? (p->hkv + kMaxChunks - 1) / kMaxChunks : 1;  // KV heads per chunk
        for (int64_t kv0 = 0; kv0 < p->hkv; kv0 += per) {
            const int64_t nkv = std::min(per, p->hkv - kv0);
            chunks.push_back({kv0, nkv, kv0 * rep, nkv * rep, true});
        }
    } else {
        const int64_t parts = std::min<int64_t>(rep, std::max<int64_t>(1, kMaxChunks / p->hkv));
        for (int64_t kvh = 0; kvh < p->hkv; ++kvh)
            for (int64_t part = 0; part < parts; ++part) {
                const int64_t a0 = part * rep / parts, a1 = (part + 1) * rep / parts;
                if (a1 > a0) chunks.push_back({kvh, 1, kvh * rep + a0, a1 - a0, part == 0});
            }
    }
    for (const Chunk& ch : chunks) {
        max_nkv = std::max(max_nkv, ch.nkv);
        max_nh = std::max(max_nh, ch.nh);
    }
    const int nchunks = static_cast<int>(chunks.size());
    if (nchunks > kMaxChunks) return fail(AA_ERR_INVALID_ARGUMENT, "aa_anchor_attention_host: chunking");
    aa_problem sub = *p;
    sub.q_row_stride = sub.kv_row_stride = p->d;
    sub.q_head_stride = sub.kv_head_stride = p->n * p->d;
    aa_plan sub_plan;
    if (nchunks > 0) {
        // workspace for the largest chunk (a run's query heads share one KV head)
        sub.hkv = max_nkv;
        sub.hq = max_nkv == 1 ? max_nh : max_nkv * rep;
        if (aa_status s = aa_make_plan(&sub, &sub_plan)) return s;
    }
    const size_t es = p->dtype == AA_BF16 ? 2 : 4;
    const size_t os = out_dtype == AA_BF16 ? 2 : 4;
    const size_t head_in = static_cast<size_t>(p->n * p->d) * es;
    const size_t head_out = static_cast<size_t>(p->n * p->d) * os;
    const size_t qb = static_cast<size_t>(p->hq) * head_in;
    const size_t kvb = static_cast<size_t>(p->hkv) * head_in;
    const size_t ob = static_cast<size_t>(p->hq) * head_out;
    const size_t cb = static_cast<size_t>(p->hq) * 8;
    const size_t ws_bytes = nchunks > 0 ? sub_plan.workspace_bytes : 0;
    const size_t need = align256(qb) + 2 * align256(kvb) + align256(ob) + align256(cb) + ws_bytes;
    if (need > dbytes) {
        if (dbuf) AA_CUDA(cudaFree(dbuf));
        dbuf = nullptr;
        dbytes = 0;
        AA_CUDA(cudaMalloc(&dbuf, need));
        dbytes = need;
    }
    char* b = static_cast<char*>(dbuf);
    char* dq = b;
    char* dk = dq + align256(qb);
    char* dv = dk + align256(kvb);
    char* dout = dv + align256(kvb);
    int64_t* dc = reinterpret_cast<int64_t*>(dout + align256(ob));
    void* ws = reinterpret_cast<char*>(dc) + align256(cb);
    const char* hq_ = static_cast<const char*>(q);
    const char* hk_ = static_cast<const char*>(k);
    const char* hv_ = static_cast<const char*>(v);
    char* ho_ = static_cast<char*>(out);
    unsigned* v_flags = ds.v_flags;
    for (int c = 0; c < nchunks; ++c) v_flags[c] = 0;
    for (int c = 0; c < nchunks; ++c) {
        const int64_t kv0 = chunks[c].kv0, nkv = chunks[c].nkv, h0 = chunks[c].h0, nh = chunks[c].nh;
        const size_t qo = static_cast<size_t>(h0) * head_in, qn = static_cast<size_t>(nh) * head_in;
        const size_t ko = static_cast<size_t>(kv0) * head_in, kn = static_cast<size_t>(nkv) * head_in;
        AA_CUDA(cudaMemcpyAsync(dq + qo, hq_ + qo, qn, cudaMemcpyHostToDevice, st_in));
        if (chunks[c].copy_kv) {
            AA_CUDA(cudaMemcpyAsync(dk + ko, hk_ + ko, kn, cudaMemcpyHostToDevice, st_in));
            AA_CUDA(cudaMemcpyAsync(dv + ko, hv_ + ko, kn, cudaMemcpyHostToDevice, st_in));
        }
        AA_CUDA(cudaEventRecord(ev_in[c], st_in));
        AA_CUDA(cudaStreamWaitEvent(st_c, ev_in[c], 0));
        sub.hkv = nkv;
        sub.hq = nh;
        if (aa_status s = aa_anchor_attention(&sub, dq + qo, dk + ko, dv + ko, zero_anchor,
                                              dout + static_cast<size_t>(h0) * head_out,
                                              out_dtype, dc + h0, ws, ws_bytes,
                                              reinterpret_cast<aa_stream_t>(st_c))) {
            cudaStreamSynchronize(st_in);
            cudaStreamSynchronize(st_c);
            cudaStreamSynchronize(st_out);
            return s;
        }
        if (p->dtype == AA_BF16) {
            // the chunk's V-range count (workspace flags), summed on the host
            const Layout WL = carve(sub, sub_plan, ws);
            AA_CUDA(cudaMemcpyAsync(&v_flags[c], WL.flags, 4, cudaMemcpyDeviceToHost, st_c));
        }
        AA_CUDA(cudaEventRecord(ev_done[c], st_c));
        AA_CUDA(cudaStreamWaitEvent(st_out, ev_done[c], 0));
        const size_t oo = static_cast<size_t>(h0) * head_out, on = static_cast<size_t>(nh) * head_out;
        AA_CUDA(cudaMemcpyAsync(ho_ + oo, dout + oo, on, cudaMemcpyDeviceToHost, st_out));
    }
    if (computed && nchunks > 0)
        AA_CUDA(cudaMemcpyAsync(computed, dc, cb, cudaMemcpyDeviceToHost, st_out));
    AA_CUDA(cudaStreamSynchronize(st_in));
    AA_CUDA(cudaStreamSynchronize(st_c));
    AA_CUDA(cudaStreamSynchronize(st_out));
    unsigned v_overflow = 0;
    for (int c = 0; c < nchunks; ++c) v_overflow += v_flags[c];
    if (p->dtype == AA_BF16 && v_overflow != 0)
        return fail(AA_ERR_UNSUPPORTED,
                    "aa_anchor_attention_host: |v| > 65504 does not fit the f16 PV operand of "
                    "the bf16 path (output is not finite); use the exact path (AA_F32)");
    return AA_OK;
}

aa_status aa_dense_attention(const aa_problem* p, const void* q, const void* k, const void* v,
                             void* out, aa_dtype out_dtype, aa_stream_t stream) {
    aa_plan plan;
    if (aa_status s = aa_make_plan(p, &plan)) return s;
    if (aa_status s = require_device()) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (p->dtype == AA_F32) {
        AA_CUDA(aa::launch_dense_exact(exact_args(*p), static_cast<const float*>(q),
                                       static_cast<const float*>(k), static_cast<const float*>(v),
                                       out, out_dtype, st));
    } else {
        const aa::FastArgs f = fast_args(*p);
        Temp v16(st);
        AA_CUDA(v16.alloc(static_cast<size_t>(p->hkv * p->n * p->d) * 2));
        AA_CUDA(aa::fast_convert_v(f, v, v16.p, st));
        AA_CUDA(aa::fast_dense(f, q, k, v16.p, out, out_dtype, st));
    }
    return AA_OK;
}

aa_status aa_union_recall(const aa_problem* p, const void* q, const void* k,
                          const uint32_t* indices, const int32_t* counts, double* recall,
                          aa_stream_t stream) {
    aa_plan plan;
    if (aa_status s = aa_make_plan(p, &plan)) return s;
    if (aa_status s = require_device()) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const aa::Geo G = geo_of(p->n, p->cfg);
    const int64_t cap = plan.stripe_capacity > 0 ? plan.stripe_capacity : 1;
    Temp tmp(st);
    const size_t ob = align256(static_cast<size_t>(plan.groups + 1) * 8);
    AA_CUDA(tmp.alloc(ob + static_cast<size_t>(p->hq * p->n) * 8));
    int64_t* offs = static_cast<int64_t*>(tmp.p);
    double* rows = reinterpret_cast<double*>(static_cast<char*>(tmp.p) + ob);
    AA_CUDA(aa::launch_offsets(G, offs, st));
    if (p->dtype == AA_F32) {
        AA_CUDA(aa::launch_recall_exact(exact_args(*p), static_cast<const float*>(q),
                                        static_cast<const float*>(k), indices, counts, offs, cap,
                                        rows, recall, st));
    } else {
        AA_CUDA(aa::fast_recall(fast_args(*p), q, k, indices, counts, offs, cap, rows, recall,
                                st));
    }
    return AA_OK;
}

}  // extern "C"
