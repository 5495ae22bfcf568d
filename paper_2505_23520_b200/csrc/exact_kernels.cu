// Exact path (aa_problem.dtype == AA_F32): f32 inputs, f64 state.
//
// These SIMT kernels restate the reference's arithmetic operation for
// operation — f64 dot products in index order, 1/sqrt(d) applied after the
// dot, the online merge per kv block (Alg. 1) and per index chunk (Alg. 3),
// sequential l / acc accumulation in key order — so their results agree with
// R/src/{anchor_pass,stripe_identify,sparse_exec}.cpp to f64 round-off and the
// selected stripe sets are identical.  They serve every BlockConfig and head
// dim the reference accepts; speed comes from the AA_BF16 tcgen05 path.
//
// One warp owns one query row: lanes split keys for the dot products (each
// dot is still sequential over d) and split head-dim columns for the
// accumulator, while the merge scalars are replicated bit-identically in all
// lanes.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace aa {
namespace {

__device__ __forceinline__ double warp_max(double x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

__device__ __forceinline__ double dot_f64(const float* __restrict__ a, const float* __restrict__ b,
                                          int64_t d) {
    double s = 0.0;
    for (int64_t t = 0; t < d; ++t) s += static_cast<double>(a[t]) * static_cast<double>(b[t]);
    return s;
}

__device__ __forceinline__ void store_out(void* out, aa_dtype dt, int64_t idx, double x) {
    if (dt == AA_BF16)
        static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16(static_cast<float>(x));
    else
        static_cast<float*>(out)[idx] = static_cast<float>(x);
}

// ---------------------------------------------------------------- Alg. 1 --
// R/src/anchor_pass.cpp:37-96.  grid (n, hq), block 32, smem (b_kv + d) f64.
__global__ void k_anchor_exact(ExactArgs a, const float* __restrict__ q,
                               const float* __restrict__ k, const float* __restrict__ v,
                               double* __restrict__ m_out, double* __restrict__ l_out,
                               double* __restrict__ acc_out) {
    extern __shared__ double smem[];
    double* qk = smem;
    double* acc = smem + a.geo.b_kv;
    const int lane = threadIdx.x;
    const int64_t i = blockIdx.x;
    const int64_t h = blockIdx.y;
    const int64_t d = a.d;
    const float* qr = q + h * a.q_hs + i * a.q_rs;
    const float* kb = k + (h / a.rep) * a.kv_hs;
    const float* vb = v + (h / a.rep) * a.kv_hs;
    for (int64_t t = lane; t < d; t += 32) acc[t] = 0.0;
    double mi = -INFINITY, li = 0.0;

    const Geo& G = a.geo;
    const int64_t qb = i / G.b_q;
    const int64_t g = qb / G.step;
    const int64_t last_row = ((qb + 1) * G.b_q < G.n ? (qb + 1) * G.b_q : G.n) - 1;
    const int64_t diag = last_row / G.b_kv;
    const int64_t t_n = G.kv_blocks();
    const int64_t wsb = G.window_start_block(g);
    // anchor_region: {0} then [wsb, diag] (anchor_pass.cpp:24-28)
    for (int64_t bi = 0;; ++bi) {
        int64_t blk = 0;
        if (bi > 0) {
            blk = wsb + bi - 1;
            if (blk > diag || blk >= t_n) break;
        }
        const int64_t key_begin = blk * G.b_kv;
        int64_t key_end = key_begin + G.b_kv;
        if (key_end > G.n) key_end = G.n;
        const int64_t causal_end = key_end < i + 1 ? key_end : i + 1;
        if (key_begin >= causal_end) continue;
        double bmax = -INFINITY;
        for (int64_t j = key_begin + lane; j < causal_end; j += 32) {
            const double s = dot_f64(qr, kb + j * a.kv_rs, d) * a.inv_sqrt_d;
            qk[j - key_begin] = s;
            bmax = fmax(bmax, s);
        }
        bmax = warp_max(bmax);
        __syncwarp();
        const double m_new = fmax(mi, bmax);
        const double alpha = isinf(mi) ? 0.0 : exp(mi - m_new);
        for (int64_t t = lane; t < d; t += 32) acc[t] *= alpha;
        double lb = 0.0;
        for (int64_t j = key_begin; j < causal_end; ++j) {
            const double p = exp(qk[j - key_begin] - m_new);
            lb += p;
            const float* vr = vb + j * a.kv_rs;
            for (int64_t t = lane; t < d; t += 32) acc[t] += p * static_cast<double>(vr[t]);
        }
        li = li * alpha + lb;
        mi = m_new;
        __syncwarp();
    }
    if (lane == 0) {
        m_out[h * G.n + i] = mi;
        l_out[h * G.n + i] = li;
    }
    for (int64_t t = lane; t < d; t += 32) acc_out[(h * G.n + i) * d + t] = acc[t];
}

// ------------------------------------------------- pooling (Alg. 2 input) --
// avgpool_rows(Q, step*b_q) (R/src/matrix.cpp:44-65) and pooled_anchor
// (R/src/stripe_identify.cpp:71-74 -> matrix.cpp:67-81).  grid (groups, hq).
__global__ void k_pool_exact(ExactArgs a, const float* __restrict__ q,
                             const double* __restrict__ m, double* __restrict__ anchor,
                             float* __restrict__ qbar) {
    const int64_t g = blockIdx.x, h = blockIdx.y;
    const Geo& G = a.geo;
    const int64_t rb = G.row_begin(g), re = G.row_end(g);
    const double inv = 1.0 / static_cast<double>(re - rb);
    const int64_t groups = G.groups();
    for (int64_t t = threadIdx.x; t < a.d; t += blockDim.x) {
        double s = 0.0;
        for (int64_t i = rb; i < re; ++i) s += q[h * a.q_hs + i * a.q_rs + t];
        qbar[(h * groups + g) * a.d + t] = static_cast<float>(s * inv);
    }
    if (threadIdx.x == 0 && anchor != nullptr) {
        double s = 0.0;
        for (int64_t i = rb; i < re; ++i) s += m[h * G.n + i];
        anchor[h * groups + g] = s / static_cast<double>(re - rb);
    }
}

// --------------------------------------------------------------- Alg. 2 --
// R/src/stripe_identify.cpp:31-46: key j of [b_kv, middle_end(g)) is kept iff
// anchor[g] - dot(qbar_g, k_j)/sqrt(d) <= theta.  One bit per candidate,
// written a 32-key word at a time (ballot).  grid (groups, hq), block 256.
__global__ void k_identify_exact(ExactArgs a, const float* __restrict__ k,
                                 const float* __restrict__ qbar, const double* __restrict__ anchor,
                                 uint32_t* __restrict__ bits, int64_t words_per_row) {
    const int64_t g = blockIdx.x, h = blockIdx.y;
    const Geo& G = a.geo;
    const int64_t groups = G.groups();
    const int64_t len = G.middle_len(g);
    const float* qr = qbar + (h * groups + g) * a.d;
    const float* kb = k + (h / a.rep) * a.kv_hs;
    const double ref = anchor ? anchor[h * groups + g] : 0.0;
    uint32_t* row = bits + (h * groups + g) * words_per_row;
    for (int64_t base = 0; base < len; base += blockDim.x) {
        const int64_t c = base + threadIdx.x;
        bool keep = false;
        if (c < len) {
            const int64_t j = G.b_kv + c;
            const double s = dot_f64(qr, kb + j * a.kv_rs, a.d);
            keep = (ref - s * a.inv_sqrt_d <= a.theta);
        }
        const uint32_t w = __ballot_sync(0xffffffffu, keep);
        if ((threadIdx.x & 31) == 0 && c < len) row[c >> 5] = w;
    }
}

// --------------------------------------------------------------- Alg. 3 --
// R/src/sparse_exec.cpp:13-124.  grid (n, hq), block 32,
// smem chunk*(f64 + u32) + d*f64.
// Scores staged in shared memory per fold chunk up to this many entries;
// longer FoldPlan chunks fold in two passes (same values, same order).
constexpr int64_t kSparseStage = 4096;

__global__ void k_sparse_exact(ExactArgs a, const float* __restrict__ q,
                               const float* __restrict__ k, const float* __restrict__ v,
                               const double* __restrict__ m_in, const double* __restrict__ l_in,
                               const double* __restrict__ acc_in,
                               const uint32_t* __restrict__ indices,
                               const int32_t* __restrict__ counts,
                               const int64_t* __restrict__ offsets, int64_t cap, bool csr,
                               int64_t chunk, void* out, aa_dtype out_dtype,
                               unsigned long long* __restrict__ computed) {
    extern __shared__ double smem[];
    double* acc = smem;
    double* qk = smem + a.d;
    uint32_t* kept = reinterpret_cast<uint32_t*>(qk + (chunk > kSparseStage ? 0 : chunk));
    const int lane = threadIdx.x;
    const int64_t i = blockIdx.x, h = blockIdx.y;
    const Geo& G = a.geo;
    const int64_t d = a.d;
    const int64_t groups = G.groups();
    const int64_t g = i / G.group_rows();
    const int64_t cnt = counts[h * groups + g];
    const uint32_t* list = csr ? indices + offsets[h * groups + g] : indices + h * cap + offsets[g];
    const int64_t wstart = G.window_start(g);
    const float* qr = q + h * a.q_hs + i * a.q_rs;
    const float* kb = k + (h / a.rep) * a.kv_hs;
    const float* vb = v + (h / a.rep) * a.kv_hs;
    double mi = m_in[h * G.n + i], li = l_in[h * G.n + i];
    for (int64_t t = lane; t < d; t += 32) acc[t] = acc_in[(h * G.n + i) * d + t];
    unsigned long long taken_total = 0;
    for (int64_t c0 = 0; c0 < cnt; c0 += chunk) {
        const int64_t c1 = c0 + chunk < cnt ? c0 + chunk : cnt;
        int64_t taken = 0;
        double cmax = -INFINITY;
        if (chunk > kSparseStage) {
            // chunks longer than the staging buffer: pass 1 takes the chunk max
            // and count, pass 2 recomputes each kept score (the same f64 dot in
            // the same order, so the same value) and folds it in list order —
            // bit-identical to the staged fold below, for any FoldPlan chunk
            for (int64_t s0 = c0; s0 < c1; s0 += 32) {
                const int64_t s = s0 + lane;
                bool keep = false;
                uint32_t j = 0;
                if (s < c1) {
                    j = list[s];
                    keep = !(static_cast<int64_t>(j) > i) &&
                           !(static_cast<int64_t>(j) < G.b_kv || static_cast<int64_t>(j) >= wstart);
                }
                if (keep)
                    cmax = fmax(cmax, dot_f64(qr, kb + static_cast<int64_t>(j) * a.kv_rs, d) * a.inv_sqrt_d);
                taken += __popc(__ballot_sync(0xffffffffu, keep));
            }
            cmax = warp_max(cmax);
            if (taken == 0) continue;
            taken_total += static_cast<unsigned long long>(taken);
            const double m_new = fmax(mi, cmax);
            const double alpha = exp(mi - m_new);
            for (int64_t t = lane; t < d; t += 32) acc[t] *= alpha;
            double lc = 0.0;
            for (int64_t s0 = c0; s0 < c1; s0 += 32) {
                const int64_t s = s0 + lane;
                bool keep = false;
                uint32_t j = 0;
                double sc = 0.0;
                if (s < c1) {
                    j = list[s];
                    keep = !(static_cast<int64_t>(j) > i) &&
                           !(static_cast<int64_t>(j) < G.b_kv || static_cast<int64_t>(j) >= wstart);
                }
                if (keep) sc = dot_f64(qr, kb + static_cast<int64_t>(j) * a.kv_rs, d) * a.inv_sqrt_d;
                for (uint32_t bal = __ballot_sync(0xffffffffu, keep); bal; bal &= bal - 1) {
                    const int src = __ffs(bal) - 1;
                    const double p = exp(__shfl_sync(0xffffffffu, sc, src) - m_new);
                    const uint32_t jj = __shfl_sync(0xffffffffu, j, src);
                    lc += p;
                    const float* vr = vb + static_cast<int64_t>(jj) * a.kv_rs;
                    for (int64_t t = lane; t < d; t += 32) acc[t] += p * static_cast<double>(vr[t]);
                }
            }
            li = li * alpha + lc;
            mi = m_new;
            __syncwarp();
            continue;
        }
        for (int64_t s0 = c0; s0 < c1; s0 += 32) {
            const int64_t s = s0 + lane;
            bool keep = false;
            uint32_t j = 0;
            if (s < c1) {
                j = list[s];
                keep = !(static_cast<int64_t>(j) > i) &&
                       !(static_cast<int64_t>(j) < G.b_kv || static_cast<int64_t>(j) >= wstart);
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int pos = __popc(bal & ((1u << lane) - 1u));
                const double sc = dot_f64(qr, kb + static_cast<int64_t>(j) * a.kv_rs, d) *
                                  a.inv_sqrt_d;
                qk[taken + pos] = sc;
                kept[taken + pos] = j;
                cmax = fmax(cmax, sc);
            }
            taken += __popc(bal);
        }
        cmax = warp_max(cmax);
        __syncwarp();
        if (taken == 0) continue;
        taken_total += static_cast<unsigned long long>(taken);
        const double m_new = fmax(mi, cmax);
        const double alpha = exp(mi - m_new);
        for (int64_t t = lane; t < d; t += 32) acc[t] *= alpha;
        double lc = 0.0;
        for (int64_t s = 0; s < taken; ++s) {
            const double p = exp(qk[s] - m_new);
            lc += p;
            const float* vr = vb + static_cast<int64_t>(kept[s]) * a.kv_rs;
            for (int64_t t = lane; t < d; t += 32) acc[t] += p * static_cast<double>(vr[t]);
        }
        li = li * alpha + lc;
        mi = m_new;
        __syncwarp();
    }
    const double inv_l = 1.0 / li;
    for (int64_t t = lane; t < d; t += 32) store_out(out, out_dtype, (h * G.n + i) * d + t, acc[t] * inv_l);
    if (lane == 0 && computed != nullptr && taken_total)
        atomicAdd(computed + h, taken_total);
}

// finalize_anchor (R/src/anchor_pass.cpp:120-131).  grid (n, hq), block 32.
__global__ void k_finalize_exact(ExactArgs a, const double* __restrict__ l,
                                 const double* __restrict__ acc, void* out, aa_dtype out_dtype) {
    const int64_t i = blockIdx.x, h = blockIdx.y;
    const double inv_l = 1.0 / l[h * a.geo.n + i];
    for (int64_t t = threadIdx.x; t < a.d; t += 32) {
        const int64_t o = (h * a.geo.n + i) * a.d + t;
        store_out(out, out_dtype, o, acc[o] * inv_l);
    }
}

// Dense causal attention (R/src/oracle.cpp:66-94).  grid (n, hq), block 32,
// smem (32 + d) f64.  Two passes: row max, then p / denom / acc in key order.
__global__ void k_dense_exact(ExactArgs a, const float* __restrict__ q,
                              const float* __restrict__ k, const float* __restrict__ v, void* out,
                              aa_dtype out_dtype) {
    extern __shared__ double smem[];
    double* acc = smem;
    double* lg = smem + a.d;
    const int lane = threadIdx.x;
    const int64_t i = blockIdx.x, h = blockIdx.y, d = a.d;
    const float* qr = q + h * a.q_hs + i * a.q_rs;
    const float* kb = k + (h / a.rep) * a.kv_hs;
    const float* vb = v + (h / a.rep) * a.kv_hs;
    double mx = -INFINITY;
    for (int64_t j = lane; j <= i; j += 32) mx = fmax(mx, dot_f64(qr, kb + j * a.kv_rs, d) * a.inv_sqrt_d);
    mx = warp_max(mx);
    for (int64_t t = lane; t < d; t += 32) acc[t] = 0.0;
    double denom = 0.0;
    for (int64_t j0 = 0; j0 <= i; j0 += 32) {
        const int64_t j = j0 + lane;
        if (j <= i) lg[lane] = dot_f64(qr, kb + j * a.kv_rs, d) * a.inv_sqrt_d;
        __syncwarp();
        const int64_t e = (i - j0 + 1) < 32 ? (i - j0 + 1) : 32;
        for (int64_t s = 0; s < e; ++s) {
            const double p = exp(lg[s] - mx);
            denom += p;
            const float* vr = vb + (j0 + s) * a.kv_rs;
            for (int64_t t = lane; t < d; t += 32) acc[t] += p * static_cast<double>(vr[t]);
        }
        __syncwarp();
    }
    for (int64_t t = lane; t < d; t += 32) store_out(out, out_dtype, (h * a.geo.n + i) * d + t, acc[t] / denom);
}

// recall(union_mask, dense_probs) row terms (R/src/metrics.cpp:8-19,
// oracle.cpp:38-64, sparse_exec.cpp:135-153).  grid (n, hq), block 32, smem
// 32 f64.  row_captured[h, i] = sum over selected j of (float)(p_ij).
__global__ void k_recall_exact(ExactArgs a, const float* __restrict__ q,
                               const float* __restrict__ k, const uint32_t* __restrict__ indices,
                               const int32_t* __restrict__ counts,
                               const int64_t* __restrict__ offsets, int64_t cap,
                               double* __restrict__ row_captured) {
    __shared__ double lg[32];
    const int lane = threadIdx.x;
    const int64_t i = blockIdx.x, h = blockIdx.y, d = a.d;
    const Geo& G = a.geo;
    const float* qr = q + h * a.q_hs + i * a.q_rs;
    const float* kb = k + (h / a.rep) * a.kv_hs;
    const int64_t g = i / G.group_rows();
    const int64_t wstart = G.window_start(g);
    const int64_t cnt = counts[h * G.groups() + g];
    const uint32_t* list = indices + h * cap + offsets[g];
    double mx = -INFINITY;
    for (int64_t j = lane; j <= i; j += 32) mx = fmax(mx, dot_f64(qr, kb + j * a.kv_rs, d) * a.inv_sqrt_d);
    mx = warp_max(mx);
    double denom = 0.0;  // replicated, sequential in key order (oracle.cpp:56-59)
    for (int64_t j0 = 0; j0 <= i; j0 += 32) {
        const int64_t j = j0 + lane;
        if (j <= i) lg[lane] = exp(dot_f64(qr, kb + j * a.kv_rs, d) * a.inv_sqrt_d - mx);
        __syncwarp();
        const int64_t e = (i - j0 + 1) < 32 ? (i - j0 + 1) : 32;
        for (int64_t s = 0; s < e; ++s) denom += lg[s];
        __syncwarp();
    }
    double cap_sum = 0.0;
    for (int64_t j0 = 0; j0 <= i; j0 += 32) {
        const int64_t j = j0 + lane;
        bool sel = false;
        if (j <= i) {
            if (j < G.b_kv || j >= wstart) {
                sel = true;
            } else {  // binary search in the group's sorted stripe list
                int64_t lo = 0, hi = cnt;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (static_cast<int64_t>(list[mid]) < j) lo = mid + 1; else hi = mid;
                }
                sel = lo < cnt && static_cast<int64_t>(list[lo]) == j;
            }
            lg[lane] = sel ? static_cast<double>(static_cast<float>(
                                 exp(dot_f64(qr, kb + j * a.kv_rs, d) * a.inv_sqrt_d - mx) / denom))
                           : 0.0;
        }
        __syncwarp();
        const int64_t e = (i - j0 + 1) < 32 ? (i - j0 + 1) : 32;
        for (int64_t s = 0; s < e; ++s) cap_sum += lg[s];
        __syncwarp();
    }
    if (lane == 0) row_captured[h * G.n + i] = cap_sum;
}

__global__ void k_recall_reduce(int64_t n, const double* __restrict__ row_captured,
                                double* __restrict__ recall) {
    const int64_t h = blockIdx.x;
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += row_captured[h * n + i];
        recall[h] = s / static_cast<double>(n);
    }
}

}  // namespace

cudaError_t launch_anchor_exact(const ExactArgs& a, const float* q, const float* k,
                                const float* v, double* m, double* l, double* acc,
                                cudaStream_t s) {
    const size_t smem = static_cast<size_t>(a.geo.b_kv + a.d) * sizeof(double);
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(
            k_anchor_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    k_anchor_exact<<<dim3(static_cast<unsigned>(a.geo.n), static_cast<unsigned>(a.hq)), 32, smem,
                     s>>>(a, q, k, v, m, l, acc);
    return cudaGetLastError();
}

cudaError_t launch_pool_exact(const ExactArgs& a, const float* q, const double* m,
                              double* anchor, float* qbar, cudaStream_t s) {
    k_pool_exact<<<dim3(static_cast<unsigned>(a.geo.groups()), static_cast<unsigned>(a.hq)), 128,
                   0, s>>>(a, q, m, anchor, qbar);
    return cudaGetLastError();
}

cudaError_t launch_identify_exact(const ExactArgs& a, const float* k, const float* qbar,
                                  const double* anchor, uint32_t* bits, int64_t words_per_row,
                                  cudaStream_t s) {
    k_identify_exact<<<dim3(static_cast<unsigned>(a.geo.groups()), static_cast<unsigned>(a.hq)),
                       256, 0, s>>>(a, k, qbar, anchor, bits, words_per_row);
    return cudaGetLastError();
}

cudaError_t launch_sparse_exact(const ExactArgs& a, const float* q, const float* k,
                                const float* v, const double* m, const double* l,
                                const double* acc, const uint32_t* indices, const int32_t* counts,
                                const int64_t* offsets, int64_t cap, bool csr, int64_t chunk,
                                void* out, aa_dtype out_dtype, unsigned long long* computed,
                                cudaStream_t s) {
    const int64_t staged = chunk > kSparseStage ? 0 : chunk;
    const size_t smem = static_cast<size_t>(a.d) * 8 + static_cast<size_t>(staged) * 12;
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(
            k_sparse_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    k_sparse_exact<<<dim3(static_cast<unsigned>(a.geo.n), static_cast<unsigned>(a.hq)), 32, smem,
                     s>>>(a, q, k, v, m, l, acc, indices, counts, offsets, cap, csr, chunk, out,
                          out_dtype, computed);
    return cudaGetLastError();
}

cudaError_t launch_finalize_exact(const ExactArgs& a, const double* l, const double* acc,
                                  void* out, aa_dtype out_dtype, cudaStream_t s) {
    k_finalize_exact<<<dim3(static_cast<unsigned>(a.geo.n), static_cast<unsigned>(a.hq)), 32, 0,
                       s>>>(a, l, acc, out, out_dtype);
    return cudaGetLastError();
}

cudaError_t launch_dense_exact(const ExactArgs& a, const float* q, const float* k,
                               const float* v, void* out, aa_dtype out_dtype, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(a.d + 32) * sizeof(double);
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(
            k_dense_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    k_dense_exact<<<dim3(static_cast<unsigned>(a.geo.n), static_cast<unsigned>(a.hq)), 32, smem,
                    s>>>(a, q, k, v, out, out_dtype);
    return cudaGetLastError();
}

cudaError_t launch_recall_exact(const ExactArgs& a, const float* q, const float* k,
                                const uint32_t* indices, const int32_t* counts,
                                const int64_t* offsets, int64_t cap, double* row_captured,
                                double* recall, cudaStream_t s) {
    k_recall_exact<<<dim3(static_cast<unsigned>(a.geo.n), static_cast<unsigned>(a.hq)), 32, 0,
                     s>>>(a, q, k, indices, counts, offsets, cap, row_captured);
    k_recall_reduce<<<static_cast<unsigned>(a.hq), 32, 0, s>>>(a.geo.n, row_captured, recall);
    return cudaGetLastError();
}

}  // namespace aa
