// Kernels shared by both arithmetic paths.
#include <cuda_runtime.h>

#include "kernels.h"

namespace aa {
namespace {

// Ordered compaction of one (head, group) selection row: each thread owns one
// 32-candidate word per pass, a block-wide exclusive scan of the word
// popcounts places its keys, and keys are emitted in ascending order — the
// sorted, unique list of StripeIndex (R/include/anchorattn/stripe_identify.hpp:17-19)
// without atomics.  grid (groups, hq), block 1024.
__global__ void __launch_bounds__(1024) k_compact(Geo geo, const uint32_t* __restrict__ bits,
                                                  int64_t words_per_row,
                                                  const int64_t* __restrict__ offsets, int64_t cap,
                                                  uint32_t* __restrict__ indices,
                                                  int32_t* __restrict__ counts) {
    __shared__ int warp_tot[32];
    __shared__ int warp_excl[32];
    const int64_t g = blockIdx.x, h = blockIdx.y;
    const int64_t groups = gridDim.x;
    const int64_t len = geo.middle_len(g);
    const int64_t words = (len + 31) >> 5;
    const uint32_t* row = bits + (h * groups + g) * words_per_row;
    uint32_t* dst = indices + h * cap + offsets[g];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t base = 0;
    for (int64_t w0 = 0; w0 < words; w0 += blockDim.x) {
        const int64_t w = w0 + threadIdx.x;
        uint32_t word = w < words ? row[w] : 0u;
        if (w == words - 1 && (len & 31)) word &= (1u << (len & 31)) - 1u;
        const int c = __popc(word);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_tot[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const int t = lane < static_cast<int>(blockDim.x >> 5) ? warp_tot[lane] : 0;
            int s = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_excl[lane] = s - t;
            if (lane == 31) warp_tot[0] = s;  // block total (read after barrier)
        }
        __syncthreads();
        int64_t pos = base + warp_excl[wid] + (incl - c);
        const uint32_t key0 = static_cast<uint32_t>(geo.b_kv + (w << 5));
        while (word) {
            const int b = __ffs(word) - 1;
            dst[pos++] = key0 + static_cast<uint32_t>(b);
            word &= word - 1u;
        }
        base += warp_tot[0];
        __syncthreads();
    }
    if (threadIdx.x == 0) counts[h * groups + g] = static_cast<int32_t>(base);
}

__global__ void k_computed(Geo geo, int64_t covered, const int32_t* __restrict__ counts,
                           int64_t* __restrict__ computed) {
    const int64_t h = blockIdx.x;
    const int64_t groups = geo.groups();
    long long s = 0;
    for (int64_t g = threadIdx.x; g < groups; g += blockDim.x)
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

__global__ void k_offsets(Geo geo, int64_t* __restrict__ offsets) {
    const int64_t G = geo.groups();
    int64_t off = 0;
    for (int64_t g = 0; g < G; ++g) {
        offsets[g] = off;
        off += geo.middle_len(g);
    }
    offsets[G] = off;
}

}  // namespace

cudaError_t launch_offsets(const Geo& geo, int64_t* offsets, cudaStream_t s) {
    k_offsets<<<1, 1, 0, s>>>(geo, offsets);
    return cudaGetLastError();
}

cudaError_t launch_compact(const Geo& geo, int64_t hq, const uint32_t* bits,
                           int64_t words_per_row, const int64_t* offsets, int64_t cap,
                           uint32_t* indices, int32_t* counts, cudaStream_t s) {
    k_compact<<<dim3(static_cast<unsigned>(geo.groups()), static_cast<unsigned>(hq)), 1024, 0,
                s>>>(geo, bits, words_per_row, offsets, cap, indices, counts);
    return cudaGetLastError();
}

cudaError_t launch_computed(const Geo& geo, int64_t hq, int64_t covered, const int32_t* counts,
                            int64_t* computed, cudaStream_t s) {
    k_computed<<<static_cast<unsigned>(hq), 32, 0, s>>>(geo, covered, counts, computed);
    return cudaGetLastError();
}

cudaError_t launch_add_u64(int64_t hq, int64_t covered, const unsigned long long* taken,
                           int64_t* computed, cudaStream_t s) {
    k_add_u64<<<static_cast<unsigned>((hq + 127) / 128), 128, 0, s>>>(hq, covered, taken,
                                                                        computed);
    return cudaGetLastError();
}

}  // namespace aa
