// TEST INFRASTRUCTURE ONLY — C entry points over the UNMODIFIED reference
// library (/root/reference/proj/src, compiled in place by oracle/Makefile into
// oracle/_ref/libanchorref.so).  Used to (1) generate the golden fixtures that
// pin the plain-C restatement (oracle/anchor_oracle.c) and (2) time the
// reference CPU path in bench.py's reference arm / cpu_baseline.
//
// Every call goes through the reference's own public API:
//   compute_anchor          R/include/anchorattn/anchor_pass.hpp:37
//   identify_stripes[_zero] R/include/anchorattn/stripe_identify.hpp:44-49
//   sparse_attention        R/include/anchorattn/sparse_exec.hpp:35-37
//   anchor_attention        R/include/anchorattn/sparse_exec.hpp:42-43
//   parallel_for            R/include/anchorattn/parallel.hpp:12-16
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "anchorattn/anchor_pass.hpp"
#include "anchorattn/metrics.hpp"
#include "anchorattn/oracle.hpp"
#include "anchorattn/parallel.hpp"
#include "anchorattn/sparse_exec.hpp"
#include "anchorattn/stripe_identify.hpp"
#include "anchorattn/workload_io.hpp"
#include "anchorattn/workloads.hpp"

using namespace anchorattn;

namespace {

thread_local std::string g_err;

Matrix mat(const float* p, std::int64_t rows, std::int64_t cols) {
    Matrix m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
    std::memcpy(m.data.data(), p, m.data.size() * sizeof(float));
    return m;
}

BlockConfig cfg_of(std::int64_t b_q, std::int64_t b_kv, std::int64_t step, double theta) {
    BlockConfig c;
    c.b_q = static_cast<std::size_t>(b_q);
    c.b_kv = static_cast<std::size_t>(b_kv);
    c.step = static_cast<std::size_t>(step);
    c.theta = theta;
    return c;
}

// Group g's slot base in the capacity layout used by the oracle and the GPU ABI.
std::size_t stripe_offset(std::size_t g, const BlockConfig& c, std::size_t n) {
    std::size_t off = 0;
    for (std::size_t h = 0; h < g; ++h) {
        const std::size_t e = middle_end_token(h, c, n);
        off += e > c.b_kv ? e - c.b_kv : 0;
    }
    return off;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// One head through compute_anchor -> identify_stripes -> sparse_attention,
// exposing every intermediate.  Returns 0 on success, 1 on exception.
int ref_pipeline(std::int64_t n, std::int64_t d, const float* q, const float* k, const float* v,
                 std::int64_t b_q, std::int64_t b_kv, std::int64_t step, double theta,
                 int zero_anchor, float* out, double* m, double* l, double* acc,
                 float* anchor_out_f /*finalize_anchor*/, double* pooled_anchor_out,
                 std::uint32_t* idx, std::int64_t* counts, std::int64_t* computed) {
    try {
        const HeadWorkload w = HeadWorkload::create(mat(q, n, d), mat(k, n, d), mat(v, n, d));
        const BlockConfig cfg = cfg_of(b_q, b_kv, step, theta);
        const AnchorState st = compute_anchor(w, cfg);
        const StripeIndex si =
            zero_anchor ? identify_stripes_zero_anchor(w, cfg) : identify_stripes(w, st, cfg);
        const SparseResult res = sparse_attention(w, st, si, cfg);
        std::memcpy(out, res.out.o.data.data(), static_cast<std::size_t>(n * d) * sizeof(float));
        if (m) std::memcpy(m, st.m.data(), st.m.size() * sizeof(double));
        if (l) std::memcpy(l, st.l.data(), st.l.size() * sizeof(double));
        if (acc) std::memcpy(acc, st.acc.data(), st.acc.size() * sizeof(double));
        if (anchor_out_f) {
            const AttentionOutput fa = finalize_anchor(st);
            std::memcpy(anchor_out_f, fa.o.data.data(), fa.o.data.size() * sizeof(float));
        }
        if (pooled_anchor_out) {
            const auto pa = pooled_anchor(st, cfg);
            std::memcpy(pooled_anchor_out, pa.data(), pa.size() * sizeof(double));
        }
        for (std::size_t g = 0; g < si.groups.size(); ++g) {
            const std::size_t off = stripe_offset(g, cfg, static_cast<std::size_t>(n));
            if (idx)
                std::memcpy(idx + off, si.groups[g].data(), si.groups[g].size() * 4);
            if (counts) counts[g] = static_cast<std::int64_t>(si.groups[g].size());
        }
        if (computed) *computed = static_cast<std::int64_t>(res.stats.computed_positions);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// A layer of `heads` independent heads (GQA: Q head h reads KV head
// h / (heads / kv_heads)), each through anchor_attention, spread over the
// reference's own parallel_for.  Layouts: q [heads, n, d], k/v [kv_heads, n, d].
int ref_layer(std::int64_t heads, std::int64_t kv_heads, std::int64_t n, std::int64_t d,
              const float* q, const float* k, const float* v, std::int64_t b_q,
              std::int64_t b_kv, std::int64_t step, double theta, int zero_anchor, float* out,
              std::int64_t* computed) {
    try {
        const BlockConfig cfg = cfg_of(b_q, b_kv, step, theta);
        const std::int64_t per = heads / kv_heads;
        const std::size_t hd = static_cast<std::size_t>(n * d);
        parallel_for(static_cast<std::size_t>(heads), [&](std::size_t h) {
            const std::size_t kvh = h / static_cast<std::size_t>(per);
            const HeadWorkload w = HeadWorkload::create(
                mat(q + h * hd, n, d), mat(k + kvh * hd, n, d), mat(v + kvh * hd, n, d));
            const SparseResult res = anchor_attention(w, cfg, zero_anchor != 0);
            std::memcpy(out + h * hd, res.out.o.data.data(), hd * sizeof(float));
            computed[h] = static_cast<std::int64_t>(res.stats.computed_positions);
        });
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_dense_attention(std::int64_t n, std::int64_t d, const float* q, const float* k,
                        const float* v, float* out) {
    try {
        const HeadWorkload w = HeadWorkload::create(mat(q, n, d), mat(k, n, d), mat(v, n, d));
        const AttentionOutput o = dense_attention(w);
        std::memcpy(out, o.o.data.data(), o.o.data.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// recall(union_mask(identify_stripes(...)), dense_probs(q, k)) — the
// reference's own recall measurement (R/src/metrics.cpp:8-19).
int ref_recall(std::int64_t n, std::int64_t d, const float* q, const float* k, const float* v,
               std::int64_t b_q, std::int64_t b_kv, std::int64_t step, double theta,
               int zero_anchor, double* recall_out, double* sparsity_out) {
    try {
        const HeadWorkload w = HeadWorkload::create(mat(q, n, d), mat(k, n, d), mat(v, n, d));
        const BlockConfig cfg = cfg_of(b_q, b_kv, step, theta);
        const AnchorState st = compute_anchor(w, cfg);
        const StripeIndex si =
            zero_anchor ? identify_stripes_zero_anchor(w, cfg) : identify_stripes(w, st, cfg);
        const SelectionMask mask = union_mask(si, cfg, static_cast<std::size_t>(n));
        *recall_out = recall(mask, dense_probs(w.q, w.k));
        *sparsity_out = sparsity(mask);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Reference generators, for building fixtures (workloads.hpp:12-38).
int ref_gen_random(std::int64_t n, std::int64_t d, std::uint64_t seed, float* q, float* k,
                   float* v) {
    try {
        const auto heads = gen_random(static_cast<std::size_t>(n), static_cast<std::size_t>(d), 1,
                                      seed);
        std::memcpy(q, heads[0].q.data.data(), static_cast<std::size_t>(n * d) * 4);
        std::memcpy(k, heads[0].k.data.data(), static_cast<std::size_t>(n * d) * 4);
        std::memcpy(v, heads[0].v.data.data(), static_cast<std::size_t>(n * d) * 4);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_gen_sink_local(std::int64_t n, std::int64_t d, double sink_strength,
                       std::int64_t window, std::uint64_t seed, float* q, float* k, float* v) {
    try {
        const HeadWorkload w = gen_sink_local(static_cast<std::size_t>(n),
                                              static_cast<std::size_t>(d), sink_strength,
                                              static_cast<std::size_t>(window), seed);
        std::memcpy(q, w.q.data.data(), static_cast<std::size_t>(n * d) * 4);
        std::memcpy(k, w.k.data.data(), static_cast<std::size_t>(n * d) * 4);
        std::memcpy(v, w.v.data.data(), static_cast<std::size_t>(n * d) * 4);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}


// ---------------------------------------------------------------------------
// A layer held across calls, for stage-sampled timing of the reference in
// bench.py (reference arm and cpu_baseline).  Every stage runs the reference's
// own public functions over its own parallel_for (one head per task):
//   ref_layer_anchor_identify  compute_anchor + identify_stripes, all heads
//   ref_layer_sparse_groups    sparse_attention, each head's StripeIndex cut
//                              down to one group (the rest emptied; the
//                              reference then only copies / finalizes their
//                              rows), or the whole index (group -1), or
//                              nothing (group -2: the fixed per-head cost);
//                              group -3 leaves the head out of the pass
struct RefLayer {
    BlockConfig cfg;
    std::vector<HeadWorkload> w;
    std::vector<AnchorState> st;
    std::vector<StripeIndex> si;
};

void* ref_layer_open(std::int64_t heads, std::int64_t kv_heads, std::int64_t n, std::int64_t d,
                     const float* q, const float* k, const float* v, std::int64_t b_q,
                     std::int64_t b_kv, std::int64_t step, double theta) {
    try {
        auto* L = new RefLayer;
        L->cfg = cfg_of(b_q, b_kv, step, theta);
        const std::int64_t per = heads / kv_heads;
        const std::size_t hd = static_cast<std::size_t>(n * d);
        L->w.resize(static_cast<std::size_t>(heads));
        L->st.resize(static_cast<std::size_t>(heads));
        L->si.resize(static_cast<std::size_t>(heads));
        parallel_for(static_cast<std::size_t>(heads), [&](std::size_t h) {
            const std::size_t kvh = h / static_cast<std::size_t>(per);
            L->w[h] = HeadWorkload::create(mat(q + h * hd, n, d), mat(k + kvh * hd, n, d),
                                           mat(v + kvh * hd, n, d));
        });
        return L;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_layer_close(void* handle) { delete static_cast<RefLayer*>(handle); }

int ref_layer_anchor_identify(void* handle, int zero_anchor) {
    try {
        auto* L = static_cast<RefLayer*>(handle);
        parallel_for(L->w.size(), [&](std::size_t h) {
            L->st[h] = compute_anchor(L->w[h], L->cfg);
            L->si[h] = zero_anchor ? identify_stripes_zero_anchor(L->w[h], L->cfg)
                                   : identify_stripes(L->w[h], L->st[h], L->cfg);
        });
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// f_c per (head, group): counts [heads * groups].
int ref_layer_counts(void* handle, std::int64_t* counts) {
    auto* L = static_cast<RefLayer*>(handle);
    std::size_t o = 0;
    for (const StripeIndex& s : L->si)
        for (const auto& g : s.groups) counts[o++] = static_cast<std::int64_t>(g.size());
    return 0;
}

int ref_layer_sparse_groups(void* handle, const std::int64_t* group_of_head,
                            std::int64_t* computed) {
    try {
        auto* L = static_cast<RefLayer*>(handle);
        parallel_for(L->w.size(), [&](std::size_t h) {
            const std::int64_t keep = group_of_head[h];
            if (keep == -3) {  // head not in this pass
                computed[h] = 0;
                return;
            }
            StripeIndex sub = L->si[h];
            if (keep != -1)
                for (std::size_t g = 0; g < sub.groups.size(); ++g)
                    if (static_cast<std::int64_t>(g) != keep) sub.groups[g].clear();
            const SparseResult res = sparse_attention(L->w[h], L->st[h], sub, L->cfg);
            computed[h] = static_cast<std::int64_t>(res.stats.computed_positions);
        });
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

std::int64_t ref_max_threads() { return static_cast<std::int64_t>(max_threads()); }

// write_workload / read_workload (R/include/anchorattn/workload_io.hpp) for
// byte-level checks of paper_2505_23520_b200.aqkv.  q/k/v: [heads, n, d].
int ref_write_workload(const char* path, std::int64_t heads, std::int64_t n, std::int64_t d,
                       const float* q, const float* k, const float* v) {
    try {
        std::vector<HeadWorkload> hs;
        const std::size_t hd = static_cast<std::size_t>(n * d);
        for (std::int64_t h = 0; h < heads; ++h)
            hs.push_back(HeadWorkload::create(mat(q + h * hd, n, d), mat(k + h * hd, n, d),
                                              mat(v + h * hd, n, d)));
        write_workload(path, hs);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Returns the number of heads read, or -1 with ref_last_error() set.
std::int64_t ref_read_workload(const char* path) {
    try {
        return static_cast<std::int64_t>(read_workload(path).size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
