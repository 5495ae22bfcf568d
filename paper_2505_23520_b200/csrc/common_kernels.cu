// Kernels shared by both arithmetic paths.
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.h"

namespace aa {
namespace {

// Ordered compaction of the (head, group) selection rows into the sorted,
// unique lists of StripeIndex (R/include/anchorattn/stripe_identify.hpp:17-19),
// without atomics.  One block per row (heaviest groups first), kCompactWarps
// warps, each owning a contiguous run of bit-words: pass 1 counts the run's
// selected keys, a block scan gives each run its output offset, pass 2 walks
// the run 32 words (1024 candidates) at a time, staging the step's keys in
// shared memory in ascending order and writing them out contiguously.
// Global traffic: the bits (twice, the second time from L2) plus 4 B per
// selected key.
#ifndef AA_COMPACT_WARPS
#define AA_COMPACT_WARPS 8
#endif
constexpr int kCompactWarps = AA_COMPACT_WARPS;

__global__ void __launch_bounds__(kCompactWarps * 32)
    k_compact(Geo geo, int64_t hq, int64_t g_end, const uint32_t* __restrict__ bits,
              int64_t words_per_row, const int64_t* __restrict__ offsets, int64_t cap,
              uint32_t* __restrict__ indices, int32_t* __restrict__ counts) {
    __shared__ uint32_t stage[kCompactWarps][1024];
    __shared__ int run_excl[kCompactWarps + 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t groups = geo.groups();
    const int64_t g = g_end - 1 - blockIdx.x / hq, h = blockIdx.x % hq;
    const int64_t len = geo.middle_len(g);
    const int64_t words = (len + 31) >> 5;
    const uint32_t* row = bits + (h * groups + g) * words_per_row;
    uint32_t* dst = indices + h * cap + offsets[g];
    const int64_t per = (words + kCompactWarps * 32 - 1) / (kCompactWarps * 32) * 32;
    const int64_t s0 = min(words, wid * per), s1 = min(words, s0 + per);
    auto word_at = [&](int64_t w) -> uint32_t {
        if (w >= s1) return 0u;
        uint32_t x = row[w];
        if (w == words - 1 && (len & 31)) x &= (1u << (len & 31)) - 1u;
        return x;
    };
    // pass 1: keys selected in this warp's run
    int cnt = 0;
#pragma unroll 8
    for (int64_t w = s0 + lane; w < s1; w += 32) cnt += __popc(word_at(w));
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) run_excl[wid + 1] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        run_excl[0] = 0;
        for (int i = 1; i <= kCompactWarps; ++i) run_excl[i] += run_excl[i - 1];
        counts[h * groups + g] = run_excl[kCompactWarps];
    }
    __syncthreads();
    // pass 2: ordered, coalesced writes (next word loaded one step ahead):
    // a warp scan of the word popcounts places each lane's keys in shared
    // memory in ascending order, then the warp writes the step's keys out
    // contiguously
    uint32_t* stg = stage[wid];
    int64_t base = run_excl[wid];
    uint32_t nxt = word_at(s0 + lane);
    for (int64_t w0 = s0; w0 < s1; w0 += 32) {
        uint32_t word = nxt;
        nxt = word_at(w0 + 32 + lane);
        const int c = __popc(word);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        // highest set bit first, written from the end of this lane's slots
        int pos = incl;
        const uint32_t key0 = static_cast<uint32_t>(geo.b_kv + ((w0 + lane) << 5));
        while (word) {  // (a fixed 32-step predicated loop measured 53 vs 43 us)
            const int b = 31 - __clz(word);
            stg[--pos] = key0 + static_cast<uint32_t>(b);
            word ^= 1u << b;
        }
        __syncwarp();
        for (int j = lane; j < total; j += 32) dst[base + j] = stg[j];
        __syncwarp();
        base += total;
    }
}

__global__ void k_computed(Geo geo, int64_t g0, int64_t g1, int64_t covered,
                           const int32_t* __restrict__ counts, int64_t* __restrict__ computed) {
    const int64_t h = blockIdx.x;
    const int64_t groups = geo.groups();
    long long s = 0;
    for (int64_t g = g0 + threadIdx.x; g < g1; g += blockDim.x)
        s += static_cast<long long>(counts[h * groups + g]) * (geo.row_end(g) - geo.row_begin(g));
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) computed[h] = covered + s;
}

__global__ void k_add_u64(int64_t hq, int64_t covered, const unsigned long long* __restrict__ taken,
                          int64_t* __restrict__ computed) {
    const int64_t h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h < hq) computed[h] = covered + static_cast<int64_t>(taken[h]);
}

// offsets[g] = sum of middle_len over the groups before g (capacity layout):
// one thread per group and a block scan (one block covers up to 1024 groups,
// i.e. 2M tokens at step 16; beyond that a per-thread loop).
__global__ void __launch_bounds__(1024) k_offsets(Geo geo, int64_t* __restrict__ offsets) {
    __shared__ int64_t warp_sum[32];
    const int64_t G = geo.groups();
    if (G >= 1024) {
        for (int64_t g = threadIdx.x; g <= G; g += blockDim.x) {
            int64_t off = 0;
            for (int64_t h = 0; h < g; ++h) off += geo.middle_len(h);
            offsets[g] = off;
        }
        return;
    }
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    int64_t x = t < G ? geo.middle_len(t) : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sum[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int64_t v = warp_sum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        warp_sum[lane] = v;  // inclusive over warps
    }
    __syncthreads();
    const int64_t incl = x + (wid > 0 ? warp_sum[wid - 1] : 0);
    if (t < G) offsets[t + 1] = incl;
    if (t == 0) offsets[0] = 0;
}

// Caller-supplied stripe lists of the stage API (capacity layout, or a CSR
// table of list starts) -> the entries sparse_exec.cpp folds
// (b_kv <= j < window_start(g), R/src/sparse_exec.cpp:79-82; window_start(g)
// <= row_begin(g) whenever that range is non-empty, so the causal clamp
// never fires on them), in list order, duplicates kept, written to
// out_idx + out_off[h * G + g] (out_idx may be NULL: validation only).  The
// first out-of-range entry j >= n in (head, group, position) order — the one
// R/src/sparse_exec.cpp:51-56 reports — is recorded as the key
// ((h * G + g) << 32 | position) in *first_bad (atomicMin).  grid (G, hq).
__global__ void __launch_bounds__(256)
    k_filter_lists(Geo geo, const uint32_t* __restrict__ idx, const int32_t* __restrict__ counts,
                   const int64_t* __restrict__ offsets, int64_t cap, int csr,
                   const int64_t* __restrict__ out_off, uint32_t* __restrict__ out_idx,
                   int32_t* __restrict__ out_counts, unsigned long long* __restrict__ first_bad) {
    __shared__ int warp_tot[8];
    const int64_t G = geo.groups();
    const int64_t g = blockIdx.x, h = blockIdx.y, row = h * G + g;
    const int64_t cnt = counts[row];
    const uint32_t* src = idx + (csr ? offsets[row] : h * cap + offsets[g]);
    uint32_t* dst = out_idx ? out_idx + out_off[row] : nullptr;
    const int64_t lo = geo.b_kv, hi = geo.window_start(g), n = geo.n;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t base = 0;
    for (int64_t b = 0; b < cnt; b += 256) {
        const int64_t e = b + threadIdx.x;
        uint32_t j = 0;
        bool keep = false;
        if (e < cnt) {
            j = src[e];
            if (j >= n)
                atomicMin(first_bad, (static_cast<unsigned long long>(row) << 32) |
                                         static_cast<unsigned long long>(e));
            keep = j >= lo && j < hi;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) warp_tot[wid] = __popc(bal);
        __syncthreads();
        int pre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            pre += w < wid ? warp_tot[w] : 0;
            tot += warp_tot[w];
        }
        if (keep && dst) dst[base + pre + __popc(bal & ((1u << lane) - 1u))] = j;
        base += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && out_counts) out_counts[row] = static_cast<int32_t>(base);
}

}  // namespace

cudaError_t launch_filter_lists(const Geo& geo, int64_t hq, const uint32_t* idx,
                                const int32_t* counts, const int64_t* offsets, int64_t cap,
                                bool csr, const int64_t* out_off, uint32_t* out_idx,
                                int32_t* out_counts, unsigned long long* first_bad,
                                cudaStream_t s) {
    const int64_t G = geo.groups();
    if (G == 0 || hq == 0) return cudaSuccess;
    k_filter_lists<<<dim3(static_cast<unsigned>(G), static_cast<unsigned>(hq)), 256, 0, s>>>(
        geo, idx, counts, offsets, cap, csr ? 1 : 0, out_off, out_idx, out_counts, first_bad);
    return cudaGetLastError();
}

cudaError_t launch_offsets(const Geo& geo, int64_t* offsets, cudaStream_t s) {
    k_offsets<<<1, 1024, 0, s>>>(geo, offsets);
    return cudaGetLastError();
}

cudaError_t launch_compact(const Geo& geo, int64_t hq, const uint32_t* bits,
                           int64_t words_per_row, const int64_t* offsets, int64_t cap,
                           uint32_t* indices, int32_t* counts, cudaStream_t s, int64_t g0,
                           int64_t g1) {
    if (g1 < 0) g1 = geo.groups();
    const int64_t rows = (g1 - g0) * hq;
    if (rows <= 0) return cudaSuccess;
    k_compact<<<static_cast<unsigned>(rows), kCompactWarps * 32, 0, s>>>(geo, hq, g1, bits, words_per_row,
                                                                        offsets, cap, indices, counts);
    return cudaGetLastError();
}

cudaError_t launch_computed(const Geo& geo, int64_t hq, int64_t covered, const int32_t* counts,
                            int64_t* computed, cudaStream_t s, int64_t g0, int64_t g1) {
    if (g1 < 0) g1 = geo.groups();
    k_computed<<<static_cast<unsigned>(hq), 32, 0, s>>>(geo, g0, g1, covered, counts, computed);
    return cudaGetLastError();
}

cudaError_t launch_add_u64(int64_t hq, int64_t covered, const unsigned long long* taken,
                           int64_t* computed, cudaStream_t s) {
    k_add_u64<<<static_cast<unsigned>((hq + 127) / 128), 128, 0, s>>>(hq, covered, taken,
                                                                        computed);
    return cudaGetLastError();
}

}  // namespace aa
