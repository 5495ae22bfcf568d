// anchorattn:: operator API over the B200 C ABI.  See anchorattn.hpp.
//
// Validation order and exception texts follow the reference
// (R/src/{matrix,anchor_pass,stripe_identify,sparse_exec}.cpp); the numerical
// work is delegated to the GPU through include/anchorattn_capi.h.  Host code
// here only moves data, builds index tables and does index arithmetic.
#include "anchorattn.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>

#include "anchorattn_capi.h"

namespace anchorattn {

namespace {

// Default: the tcgen05 path wherever the shape allows it (the product); the
// f64 exact path on request (ANCHORATTN_PRECISION=exact or set_precision).
Precision g_precision = [] {
    const char* e = std::getenv("ANCHORATTN_PRECISION");
    return (e && std::string(e) == "exact") ? Precision::Exact : Precision::Bf16;
}();

void check(aa_status s) {
    if (s == AA_OK) return;
    const std::string msg = aa_last_error();
    switch (s) {
        case AA_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case AA_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

// Device allocation owned by the shim for the duration of one call.
struct DevBuf {
    void* p = nullptr;
    DevBuf() = default;
    explicit DevBuf(std::size_t bytes) { check(aa_device_alloc(bytes, &p)); }
    DevBuf(const void* host, std::size_t bytes) : DevBuf(bytes) {
        check(aa_copy_to_device(p, host, bytes));
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { aa_device_free(p); }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

template <class T>
void download(std::vector<T>& dst, const void* src, std::size_t count) {
    dst.resize(count);
    check(aa_copy_to_host(dst.data(), src, count * sizeof(T)));
}

aa_block_config cfg_c(const BlockConfig& c) {
    return aa_block_config{static_cast<int64_t>(c.b_q), static_cast<int64_t>(c.b_kv),
                           static_cast<int64_t>(c.step), c.theta};
}

bool use_fast(std::size_t d, const BlockConfig& c) {
    return g_precision == Precision::Bf16 && d == 128 && c.b_q == 128 && c.b_kv == 128;
}

aa_problem problem(std::size_t n, std::size_t d, const BlockConfig& c, bool fast) {
    aa_problem p{};
    p.n = static_cast<int64_t>(n);
    p.d = static_cast<int64_t>(d);
    p.hq = 1;
    p.hkv = 1;
    p.cfg = cfg_c(c);
    p.dtype = fast ? AA_BF16 : AA_F32;
    return p;
}

// Round-to-nearest-even f32 -> bf16 bits.
std::vector<std::uint16_t> to_bf16(const std::vector<float>& x) {
    std::vector<std::uint16_t> out(x.size());
    for (std::size_t i = 0; i < x.size(); ++i) {
        std::uint32_t u;
        std::memcpy(&u, &x[i], 4);
        if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) {
            out[i] = static_cast<std::uint16_t>((u >> 16) | 0x40u);
        } else {
            u += 0x7fffu + ((u >> 16) & 1u);
            out[i] = static_cast<std::uint16_t>(u >> 16);
        }
    }
    return out;
}

// Q/K/V (or a subset) resident on the device in the path's input dtype.
struct DevMatrix {
    DevBuf buf;
    DevMatrix(const Matrix& m, bool fast)
        : buf(fast ? DevBuf(to_bf16(m.data).data(), m.data.size() * 2)
                   : DevBuf(m.data.data(), m.data.size() * 4)) {}
};

// splitmix64, as R/src/detail/rng.hpp:11-26 (FoldPlan shuffles).
struct SplitMix {
    std::uint64_t s;
    std::uint64_t next() {
        std::uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
};

void check_blocking(const BlockConfig& a, const BlockConfig& b, const char* msg) {
    if (a.b_q != b.b_q || a.b_kv != b.b_kv || a.step != b.step) throw std::invalid_argument(msg);
}

StripeIndex stripes_from_capacity(std::size_t n, const BlockConfig& cfg,
                                  const std::vector<std::uint32_t>& idx,
                                  const std::vector<std::int32_t>& counts) {
    const aa_block_config c = cfg_c(cfg);
    StripeIndex out;
    out.n = n;
    out.cfg = cfg;
    out.groups.resize(counts.size());
    for (std::size_t g = 0; g < counts.size(); ++g) {
        const std::size_t off = static_cast<std::size_t>(aa_stripe_offset(g, &c, n));
        out.groups[g].assign(idx.begin() + off, idx.begin() + off + counts[g]);
    }
    return out;
}

StripeIndex identify_impl(const HeadWorkload& w, const BlockConfig& cfg, const AnchorState* st) {
    const bool fast = use_fast(w.d, cfg);
    aa_problem p = problem(w.n, w.d, cfg, fast);
    aa_plan plan;
    check(aa_make_plan(&p, &plan));
    DevMatrix dq(w.q, fast), dk(w.k, fast);
    DevBuf anchor(static_cast<std::size_t>(plan.groups) * 8);
    DevBuf qbar(static_cast<std::size_t>(plan.groups) * w.d * 4);
    if (st) {
        if (fast) {
            std::vector<float> m32(st->m.begin(), st->m.end());
            DevBuf dm(m32.data(), m32.size() * 4);
            check(aa_pool(&p, dq.buf.p, dm.p, nullptr, nullptr, anchor.as<double>(),
                          qbar.as<float>(), nullptr));
        } else {
            DevBuf dm(st->m.data(), st->m.size() * 8);
            check(aa_pool(&p, dq.buf.p, dm.p, nullptr, nullptr, anchor.as<double>(),
                          qbar.as<float>(), nullptr));
        }
    } else {
        check(aa_pool(&p, dq.buf.p, nullptr, nullptr, nullptr, nullptr, qbar.as<float>(), nullptr));
    }
    const std::size_t cap = static_cast<std::size_t>(std::max<int64_t>(plan.stripe_capacity, 1));
    DevBuf idx(cap * 4), counts(static_cast<std::size_t>(plan.groups) * 4);
    check(aa_identify(&p, dk.buf.p, qbar.as<float>(), st ? anchor.as<double>() : nullptr,
                      st ? 0 : 1, idx.as<std::uint32_t>(), counts.as<std::int32_t>(), nullptr, 0,
                      nullptr));
    check(aa_stream_sync(nullptr));
    std::vector<std::uint32_t> hidx;
    std::vector<std::int32_t> hcounts;
    download(hidx, idx.p, cap);
    download(hcounts, counts.p, static_cast<std::size_t>(plan.groups));
    return stripes_from_capacity(w.n, cfg, hidx, hcounts);
}

}  // namespace

void set_precision(Precision p) { g_precision = p; }
Precision precision() { return g_precision; }

// ---- matrix.cpp ------------------------------------------------------------
bool Matrix::all_finite() const {
    return std::all_of(data.begin(), data.end(), [](float x) { return std::isfinite(x); });
}

HeadWorkload HeadWorkload::create(Matrix q, Matrix k, Matrix v) {
    if (q.rows == 0 || q.cols == 0)
        throw std::invalid_argument("HeadWorkload: n and d must be >= 1");
    if (!q.same_shape(k) || !q.same_shape(v))
        throw std::invalid_argument("HeadWorkload: q, k, v must share shape (n, d)");
    HeadWorkload w;
    w.n = q.rows;
    w.d = q.cols;
    w.q = std::move(q);
    w.k = std::move(k);
    w.v = std::move(v);
    return w;
}

void BlockConfig::validate() const {
    const aa_block_config c = cfg_c(*this);
    check(aa_config_validate(&c));
}

// Host utilities (plain pooling arithmetic, not on the GPU pipeline, which
// pools inside its own kernels): R/src/matrix.cpp:44-81.
Matrix avgpool_rows(const Matrix& m, std::size_t block) {
    if (block == 0) throw std::invalid_argument("avgpool_rows: block must be >= 1");
    if (m.rows == 0) throw std::invalid_argument("avgpool_rows: empty matrix");
    const std::size_t out_rows = (m.rows + block - 1) / block;
    Matrix out(out_rows, m.cols);
    std::vector<double> sums(m.cols);
    for (std::size_t g = 0; g < out_rows; ++g) {
        const std::size_t b = g * block, e = std::min(b + block, m.rows);
        std::fill(sums.begin(), sums.end(), 0.0);
        for (std::size_t i = b; i < e; ++i)
            for (std::size_t j = 0; j < m.cols; ++j) sums[j] += m.data[i * m.cols + j];
        const double inv = 1.0 / static_cast<double>(e - b);
        for (std::size_t j = 0; j < m.cols; ++j) out.at(g, j) = static_cast<float>(sums[j] * inv);
    }
    return out;
}

std::vector<double> avgpool_vector(std::span<const double> v, std::size_t block) {
    if (block == 0) throw std::invalid_argument("avgpool_vector: block must be >= 1");
    if (v.empty()) throw std::invalid_argument("avgpool_vector: empty vector");
    std::vector<double> out((v.size() + block - 1) / block);
    for (std::size_t g = 0; g < out.size(); ++g) {
        const std::size_t b = g * block, e = std::min(b + block, v.size());
        double s = 0.0;
        for (std::size_t i = b; i < e; ++i) s += v[i];
        out[g] = s / static_cast<double>(e - b);
    }
    return out;
}

// ---- selection_mask.cpp ----------------------------------------------------
SelectionMask SelectionMask::full_causal(std::size_t n) {
    SelectionMask m(n);
    for (std::size_t i = 0; i < n; ++i) {
        m.rows[i].resize(i + 1);
        std::iota(m.rows[i].begin(), m.rows[i].end(), 0u);
    }
    return m;
}

std::size_t SelectionMask::total_selected() const {
    std::size_t t = 0;
    for (const auto& r : rows) t += r.size();
    return t;
}

bool SelectionMask::contains(std::size_t i, std::uint32_t j) const {
    return std::binary_search(rows[i].begin(), rows[i].end(), j);
}

void SelectionMask::normalize() {
    for (std::size_t i = 0; i < rows.size(); ++i) {
        auto& r = rows[i];
        std::sort(r.begin(), r.end());
        r.erase(std::unique(r.begin(), r.end()), r.end());
        while (!r.empty() && r.back() > i) r.pop_back();
    }
}

bool SelectionMask::valid() const {
    if (rows.size() != n) return false;
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t k = 0; k < rows[i].size(); ++k) {
            if (rows[i][k] > i) return false;
            if (k > 0 && rows[i][k] <= rows[i][k - 1]) return false;
        }
    return true;
}

// ---- anchor_pass -------------------------------------------------------------
std::vector<std::size_t> anchor_region(std::size_t q_block, const BlockConfig& cfg,
                                       std::size_t n) {
    cfg.validate();
    const aa_block_config c = cfg_c(cfg);
    const int64_t cnt = aa_anchor_region(static_cast<int64_t>(q_block), &c, n, nullptr, 0);
    if (cnt < 0) throw std::invalid_argument(aa_last_error());
    std::vector<int64_t> b(static_cast<std::size_t>(cnt));
    aa_anchor_region(static_cast<int64_t>(q_block), &c, n, b.data(), cnt);
    return std::vector<std::size_t>(b.begin(), b.end());
}

std::size_t window_start_token(std::size_t group, const BlockConfig& cfg, std::size_t n) {
    const aa_block_config c = cfg_c(cfg);
    return static_cast<std::size_t>(aa_window_start_token(group, &c, n));
}

AnchorState compute_anchor(const HeadWorkload& w, const BlockConfig& cfg) {
    cfg.validate();
    const bool fast = use_fast(w.d, cfg);
    aa_problem p = problem(w.n, w.d, cfg, fast);
    aa_plan plan;
    check(aa_make_plan(&p, &plan));
    const std::size_t es = fast ? 4 : 8;
    DevMatrix dq(w.q, fast), dk(w.k, fast), dv(w.v, fast);
    DevBuf m(w.n * es), l(w.n * es), acc(w.n * w.d * es);
    check(aa_compute_anchor(&p, dq.buf.p, dk.buf.p, dv.buf.p, m.p, l.p, acc.p, nullptr, nullptr,
                            nullptr));
    check(aa_stream_sync(nullptr));
    AnchorState st;
    st.n = w.n;
    st.d = w.d;
    st.cfg = cfg;
    if (fast) {
        std::vector<float> hm, hl, hacc;
        download(hm, m.p, w.n);
        download(hl, l.p, w.n);
        download(hacc, acc.p, w.n * w.d);
        st.m.assign(hm.begin(), hm.end());
        st.l.assign(hl.begin(), hl.end());
        st.acc.assign(hacc.begin(), hacc.end());
    } else {
        download(st.m, m.p, w.n);
        download(st.l, l.p, w.n);
        download(st.acc, acc.p, w.n * w.d);
    }
    return st;
}

SelectionMask anchor_mask(std::size_t n, const BlockConfig& cfg) {
    cfg.validate();
    SelectionMask mask(n);
    const std::size_t gr = cfg.step * cfg.b_q;
    for (std::size_t i = 0; i < n; ++i) {
        const std::size_t init_end = std::min(cfg.b_kv, i + 1);
        const std::size_t ws = window_start_token(i / gr, cfg, n);
        auto& r = mask.rows[i];
        for (std::size_t j = 0; j < init_end; ++j) r.push_back(static_cast<std::uint32_t>(j));
        for (std::size_t j = ws; j <= i; ++j) r.push_back(static_cast<std::uint32_t>(j));
    }
    return mask;
}

std::size_t anchor_covered_count(std::size_t n, const BlockConfig& cfg) {
    cfg.validate();
    const aa_block_config c = cfg_c(cfg);
    return static_cast<std::size_t>(aa_anchor_covered_count(n, &c));
}

AttentionOutput finalize_anchor(const AnchorState& state) {
    aa_problem p = problem(state.n, state.d, state.cfg, false);
    DevBuf l(state.l.data(), state.l.size() * 8), acc(state.acc.data(), state.acc.size() * 8);
    DevBuf out(state.n * state.d * 4);
    check(aa_finalize_anchor(&p, l.p, acc.p, out.p, AA_F32, nullptr));
    check(aa_stream_sync(nullptr));
    AttentionOutput o;
    o.o = Matrix(state.n, state.d);
    check(aa_copy_to_host(o.o.data.data(), out.p, o.o.data.size() * 4));
    return o;
}

// ---- stripe_identify ---------------------------------------------------------
std::size_t StripeIndex::total_selected() const {
    std::size_t t = 0;
    for (const auto& g : groups) t += g.size();
    return t;
}

bool StripeIndex::empty() const { return total_selected() == 0; }

std::size_t group_count(std::size_t n, const BlockConfig& cfg) {
    cfg.validate();
    const aa_block_config c = cfg_c(cfg);
    return static_cast<std::size_t>(aa_group_count(n, &c));
}

std::size_t middle_end_token(std::size_t group, const BlockConfig& cfg, std::size_t n) {
    cfg.validate();
    const aa_block_config c = cfg_c(cfg);
    return static_cast<std::size_t>(aa_middle_end_token(group, &c, n));
}

std::vector<double> pooled_anchor(const AnchorState& state, const BlockConfig& cfg) {
    cfg.validate();
    return avgpool_vector(state.m, cfg.step * cfg.b_q);
}

StripeIndex identify_stripes(const HeadWorkload& w, const AnchorState& state,
                             const BlockConfig& cfg) {
    cfg.validate();
    if (state.n != w.n) throw std::invalid_argument("identify_stripes: state/workload mismatch");
    check_blocking(state.cfg, cfg, "identify_stripes: anchor state uses another blocking");
    return identify_impl(w, cfg, &state);
}

StripeIndex identify_stripes_zero_anchor(const HeadWorkload& w, const BlockConfig& cfg) {
    cfg.validate();
    return identify_impl(w, cfg, nullptr);
}

// ---- sparse_exec ---------------------------------------------------------------
SparseResult sparse_attention(const HeadWorkload& w, const AnchorState& state,
                              const StripeIndex& idx, const BlockConfig& cfg,
                              const FoldPlan& plan) {
    cfg.validate();
    if (state.n != w.n || idx.n != w.n)
        throw std::invalid_argument("sparse_attention: inputs built for another workload");
    check_blocking(state.cfg, cfg, "sparse_attention: anchor state uses another blocking");
    const std::size_t groups = group_count(w.n, cfg);
    if (idx.groups.size() != groups)
        throw std::invalid_argument("sparse_attention: stripe index group count mismatch");
    if (plan.index_chunk == 0)
        throw std::invalid_argument("sparse_attention: index_chunk must be >= 1");
    for (const auto& g : idx.groups)
        for (std::uint32_t j : g)
            if (j >= w.n)
                throw std::out_of_range("sparse_attention: stripe index " + std::to_string(j) +
                                        " out of range");

    const bool fast = use_fast(w.d, cfg);
    // CSR of the lists in fold order (FoldPlan shuffle, sparse_exec.cpp:58-64).
    // The ABI skips covered / non-causal entries itself (sparse_exec.cpp:79-82:
    // per row inside the chunks on the exact path, by a device compaction of
    // each list on the fast path).
    std::vector<std::uint32_t> flat;
    std::vector<int64_t> offsets(groups + 1, 0);
    std::vector<std::int32_t> counts(groups, 0);
    for (std::size_t g = 0; g < groups; ++g) {
        std::vector<std::uint32_t> order(idx.groups[g]);
        if (plan.shuffle_seed != 0) {
            SplitMix rng{plan.shuffle_seed + g};
            for (std::size_t i = order.size(); i > 1; --i)
                std::swap(order[i - 1], order[rng.next() % i]);
        }
        offsets[g] = static_cast<int64_t>(flat.size());
        counts[g] = static_cast<std::int32_t>(order.size());
        flat.insert(flat.end(), order.begin(), order.end());
    }
    offsets[groups] = static_cast<int64_t>(flat.size());

    aa_problem p = problem(w.n, w.d, cfg, fast);
    DevMatrix dq(w.q, fast), dk(w.k, fast), dv(w.v, fast);
    const std::size_t es = fast ? 4 : 8;
    DevBuf dm(w.n * es), dl(w.n * es), dacc(w.n * w.d * es);
    if (fast) {
        std::vector<float> m(state.m.begin(), state.m.end()), l(state.l.begin(), state.l.end()),
            acc(state.acc.begin(), state.acc.end());
        check(aa_copy_to_device(dm.p, m.data(), m.size() * 4));
        check(aa_copy_to_device(dl.p, l.data(), l.size() * 4));
        check(aa_copy_to_device(dacc.p, acc.data(), acc.size() * 4));
    } else {
        check(aa_copy_to_device(dm.p, state.m.data(), state.m.size() * 8));
        check(aa_copy_to_device(dl.p, state.l.data(), state.l.size() * 8));
        check(aa_copy_to_device(dacc.p, state.acc.data(), state.acc.size() * 8));
    }
    DevBuf dflat(std::max<std::size_t>(flat.size(), 1) * 4);
    if (!flat.empty()) check(aa_copy_to_device(dflat.p, flat.data(), flat.size() * 4));
    DevBuf doff(offsets.data(), offsets.size() * 8), dcnt(counts.data(), counts.size() * 4);
    DevBuf out(w.n * w.d * 4), computed(8);
    check(aa_sparse_attention(&p, dq.buf.p, dk.buf.p, dv.buf.p, dm.p, dl.p, dacc.p,
                              dflat.as<std::uint32_t>(), dcnt.as<std::int32_t>(),
                              doff.as<int64_t>(), static_cast<int64_t>(plan.index_chunk), out.p,
                              AA_F32, computed.as<int64_t>(), nullptr));
    check(aa_stream_sync(nullptr));
    SparseResult res;
    res.out.o = Matrix(w.n, w.d);
    check(aa_copy_to_host(res.out.o.data.data(), out.p, w.n * w.d * 4));
    int64_t c = 0;
    check(aa_copy_to_host(&c, computed.p, 8));
    res.stats.causal_positions = w.n * (w.n + 1) / 2;
    res.stats.computed_positions = static_cast<std::size_t>(c);
    res.stats.sparsity = 1.0 - static_cast<double>(res.stats.computed_positions) /
                                   static_cast<double>(res.stats.causal_positions);
    return res;
}

SparseResult anchor_attention(const HeadWorkload& w, const BlockConfig& cfg, bool zero_anchor) {
    cfg.validate();
    const bool fast = use_fast(w.d, cfg);
    aa_problem p = problem(w.n, w.d, cfg, fast);
    aa_plan plan;
    check(aa_make_plan(&p, &plan));
    SparseResult res;
    res.out.o = Matrix(w.n, w.d);
    int64_t computed = 0;
    if (fast) {
        const auto q = to_bf16(w.q.data), k = to_bf16(w.k.data), v = to_bf16(w.v.data);
        check(aa_anchor_attention_host(&p, q.data(), k.data(), v.data(), zero_anchor ? 1 : 0,
                                       res.out.o.data.data(), AA_F32, &computed));
    } else {
        check(aa_anchor_attention_host(&p, w.q.data.data(), w.k.data.data(), w.v.data.data(),
                                       zero_anchor ? 1 : 0, res.out.o.data.data(), AA_F32,
                                       &computed));
    }
    res.stats.causal_positions = w.n * (w.n + 1) / 2;
    res.stats.computed_positions = static_cast<std::size_t>(computed);
    res.stats.sparsity = 1.0 - static_cast<double>(res.stats.computed_positions) /
                                   static_cast<double>(res.stats.causal_positions);
    return res;
}

SelectionMask union_mask(const StripeIndex& idx, const BlockConfig& cfg, std::size_t n) {
    cfg.validate();
    SelectionMask mask = anchor_mask(n, cfg);
    const std::size_t gr = cfg.step * cfg.b_q;
    for (std::size_t g = 0; g < idx.groups.size(); ++g) {
        const std::size_t ws = window_start_token(g, cfg, n);
        const std::size_t rb = g * gr, re = std::min(rb + gr, n);
        for (std::size_t i = rb; i < re; ++i)
            for (std::uint32_t j : idx.groups[g]) {
                if (j > i) break;
                if (j < cfg.b_kv || j >= ws) continue;
                mask.rows[i].push_back(j);
            }
    }
    mask.normalize();
    return mask;
}

AttentionOutput dense_attention(const HeadWorkload& w) {
    const BlockConfig cfg{128, 128, 16, 12.0};
    const bool fast = use_fast(w.d, cfg);
    aa_problem p = problem(w.n, w.d, cfg, fast);
    DevMatrix dq(w.q, fast), dk(w.k, fast), dv(w.v, fast);
    DevBuf out(w.n * w.d * 4);
    check(aa_dense_attention(&p, dq.buf.p, dk.buf.p, dv.buf.p, out.p, AA_F32, nullptr));
    check(aa_stream_sync(nullptr));
    AttentionOutput o;
    o.o = Matrix(w.n, w.d);
    check(aa_copy_to_host(o.o.data.data(), out.p, w.n * w.d * 4));
    return o;
}

double union_recall(const HeadWorkload& w, const StripeIndex& idx, const BlockConfig& cfg) {
    cfg.validate();
    const bool fast = use_fast(w.d, cfg);
    aa_problem p = problem(w.n, w.d, cfg, fast);
    aa_plan plan;
    check(aa_make_plan(&p, &plan));
    const std::size_t cap = static_cast<std::size_t>(std::max<int64_t>(plan.stripe_capacity, 1));
    std::vector<std::uint32_t> flat(cap, 0);
    std::vector<std::int32_t> counts(idx.groups.size());
    const aa_block_config c = cfg_c(cfg);
    for (std::size_t g = 0; g < idx.groups.size(); ++g) {
        const std::size_t off = static_cast<std::size_t>(aa_stripe_offset(g, &c, w.n));
        const std::size_t len = static_cast<std::size_t>(aa_stripe_offset(g + 1, &c, w.n)) - off;
        std::vector<std::uint32_t> sel;
        const std::size_t ws = window_start_token(g, cfg, w.n);
        for (std::uint32_t j : idx.groups[g])
            if (j >= cfg.b_kv && j < ws) sel.push_back(j);
        std::sort(sel.begin(), sel.end());
        sel.erase(std::unique(sel.begin(), sel.end()), sel.end());
        if (sel.size() > len) sel.resize(len);
        std::copy(sel.begin(), sel.end(), flat.begin() + off);
        counts[g] = static_cast<std::int32_t>(sel.size());
    }
    DevMatrix dq(w.q, fast), dk(w.k, fast);
    DevBuf dflat(flat.data(), flat.size() * 4), dcnt(counts.data(), counts.size() * 4), r(8);
    check(aa_union_recall(&p, dq.buf.p, dk.buf.p, dflat.as<std::uint32_t>(),
                          dcnt.as<std::int32_t>(), r.as<double>(), nullptr));
    check(aa_stream_sync(nullptr));
    double out = 0.0;
    check(aa_copy_to_host(&out, r.p, 8));
    return out;
}

}  // namespace anchorattn
