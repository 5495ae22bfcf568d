// Fast path (AA_BF16): hand-written sm_100a kernels for b_q = b_kv = 128,
// d = 128.
//
//   K1 anchor   fa_tiles<ANCHOR>  tile list {0} ∪ [wsb(g), qb]   (Alg. 1)
//   K2 identify k_identify_fast   pooled-q · K, threshold, ballot (Alg. 2)
//   K3 sparse   fa_tiles<SPARSE>  gathered stripe tiles (TMA gather4),
//                                  merged with the K1 state       (Alg. 3)
//   D  dense    fa_tiles<DENSE>   tiles 0..qb (causal baseline)
//
// fa_tiles: one CTA = one (head, 128-row query block); 6 warps:
//   warp 0   TMA producer (Q once; K/V tile per iteration; gather4 for K3)
//   warp 1   TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5  softmax / epilogue: thread <-> query row (TMEM lane)
// TMEM (256 cols): S = Q K^T (f32) in cols [0,128), P (f16, aliasing S cols
// [0,64)) feeds O += P V from TMEM, O (f32) in cols [128,256).  96 KB smem
// and 256 TMEM columns per CTA -> two co-resident CTAs per SM, so one CTA's
// MMAs overlap the other's softmax.  Softmax is exp2-based with lazy
// rescaling (O/l only rescaled when the running max grows by > 8 in log2
// units); the state written out is exact (rescaled to the true max).
// PV runs in f16 (P in [0, 256] keeps 11 mantissa bits; V converted
// bf16 -> f16 once, exact for |v| in the f16 normal range).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <mutex>

#include "fast.h"
#include "kernels.h"
#include "sm100.cuh"

namespace aa {
namespace {

using namespace sm100;

constexpr int kB = 128;  // b_q = b_kv
constexpr int kD = 128;  // head dim
constexpr int kThreads = 192;
constexpr uint32_t kTileBytes = kB * kD * 2;   // 32 KB (bf16 / f16 tile)
constexpr uint32_t kAtomBytes = kB * 64 * 2;   // 16 KB: 128 rows x 128 B (SW128 atom column)
constexpr uint32_t kIdescQK = idesc_f16(1, 1, 0, 128, 128);  // bf16 x bf16, B K-major
constexpr uint32_t kIdescPV = idesc_f16(0, 0, 1, 128, 128);  // f16 x f16,  B MN-major
constexpr float kLog2e = 1.4426950408889634f;

enum Mode { ANCHOR = 0, SPARSE = 1, DENSE = 2 };

struct FaParams {
    int n, hq, rep, T_m, step;
    float scale_log2;  // log2(e) / sqrt(d)
    float inv_sqrt_d;
    // gather row mapping: row(kvh, j) = kvh * kv_head_rows + j * kv_row_rows
    int kv_head_rows, kv_row_rows;
    // ANCHOR outputs
    float* m_out;
    float* l_out;
    float* acc_out;
    float* qsum;
    double* msum;
    // SPARSE inputs
    const float* m_in;
    const float* l_in;
    const float* acc_in;
    const uint32_t* idx;
    const int32_t* counts;
    const int64_t* offsets;
    int64_t cap;
    int csr;
    int groups;
    // SPARSE / DENSE output
    void* out;
    int out_bf16;
};

struct Smem {
    // 1024-byte aligned tiles (SWIZZLE_128B atoms)
    uint8_t q[kTileBytes];
    uint8_t k[kTileBytes];
    uint8_t v[kTileBytes];
    uint64_t bar_q, bar_k_full, bar_k_empty, bar_v_full, bar_v_empty, bar_s_full, bar_p_full,
        bar_o_done;
    uint32_t tmem_base;
    float red[4];
};

__device__ __forceinline__ int kv_tile_of(int mode, int it, int wsb) {
    if (mode == DENSE) return it;
    return it == 0 ? 0 : wsb + it - 1;  // ANCHOR: {0} then [wsb, qb]
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 2)
    fa_tiles(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
             const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmKg,
             const __grid_constant__ CUtensorMap tmVg, const FaParams P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                       ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    // heavy-first: the last query blocks (longest tile lists) launch first
    const int bid = blockIdx.x;
    const int qb = P.T_m - 1 - bid / P.hq;
    const int h = bid % P.hq;
    const int kvh = h / P.rep;
    const int g = qb / P.step;

    // tile list
    int ntiles = 0, wsb = 0, count = 0;
    const uint32_t* list = nullptr;
    if (MODE == DENSE) {
        ntiles = qb + 1;
    } else if (MODE == ANCHOR) {
        const int rb = g * P.step * kB;
        wsb = rb < 2 * kB ? 1 : rb / kB - 1;
        ntiles = 1 + (qb >= wsb ? qb - wsb + 1 : 0);
    } else {
        count = P.counts[h * P.groups + g];
        list = P.csr ? P.idx + P.offsets[h * P.groups + g] : P.idx + h * P.cap + P.offsets[g];
        ntiles = (count + kB - 1) / kB;
    }

    if (threadIdx.x == 0) {
        mbar_init(&S.bar_q, 1);
        mbar_init(&S.bar_k_full, 1);
        mbar_init(&S.bar_k_empty, 1);
        mbar_init(&S.bar_v_full, 1);
        mbar_init(&S.bar_v_empty, 1);
        mbar_init(&S.bar_s_full, 1);
        mbar_init(&S.bar_p_full, 128);
        mbar_init(&S.bar_o_done, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&S.tmem_base, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;
    const uint32_t tS = tmem;        // S / P
    const uint32_t tO = tmem + 128;  // O

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0 && ntiles > 0) {
            mbar_expect_tx(&S.bar_q, kTileBytes);
            tma_load_3d(S.q, &tmQ, &S.bar_q, 0, qb * kB, h);
            tma_load_3d(S.q + kAtomBytes, &tmQ, &S.bar_q, 64, qb * kB, h);
        }
        if (MODE == SPARSE) {
            // Every lane gathers 4 of the tile's 128 rows (gather4 x 2 column
            // halves, for K and for V), so a tile is 4 TMA issues per lane
            // instead of 128 from one thread.  The next tile's indices are
            // fetched while this tile's loads are in flight.
            auto fetch = [&](int t, int (&j)[4]) {
                const int base = t * kB;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = base + lane * 4 + u;
                    j[u] = static_cast<int>(list[e < count ? e : base]);
                }
            };
            int j[4];
            if (ntiles > 0) fetch(0, j);
            const int vh = kvh * P.n;  // V16 scratch is packed [hkv, n, d]
            uint8_t* kdst = S.k + lane * 4 * 128;
            uint8_t* vdst = S.v + lane * 4 * 128;
            for (int it = 0; it < ntiles; ++it) {
                int rk[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) rk[u] = kvh * P.kv_head_rows + j[u] * P.kv_row_rows;
                if (lane == 0) {
                    if (it > 0) mbar_wait(&S.bar_k_empty, (it - 1) & 1);
                    mbar_expect_tx(&S.bar_k_full, kTileBytes);
                }
                __syncwarp();
                tma_gather4(kdst, &tmKg, &S.bar_k_full, 0, rk[0], rk[1], rk[2], rk[3]);
                tma_gather4(kdst + kAtomBytes, &tmKg, &S.bar_k_full, 64, rk[0], rk[1], rk[2], rk[3]);
                if (lane == 0) {
                    if (it > 0) mbar_wait(&S.bar_v_empty, (it - 1) & 1);
                    mbar_expect_tx(&S.bar_v_full, kTileBytes);
                }
                __syncwarp();
                tma_gather4(vdst, &tmVg, &S.bar_v_full, 0, vh + j[0], vh + j[1], vh + j[2], vh + j[3]);
                tma_gather4(vdst + kAtomBytes, &tmVg, &S.bar_v_full, 64, vh + j[0], vh + j[1],
                            vh + j[2], vh + j[3]);
                if (it + 1 < ntiles) fetch(it + 1, j);
            }
        } else {
            for (int it = 0; it < ntiles; ++it) {
                if (lane == 0) {
                    const int kt = kv_tile_of(MODE, it, wsb);
                    if (it > 0) mbar_wait(&S.bar_k_empty, (it - 1) & 1);
                    mbar_expect_tx(&S.bar_k_full, kTileBytes);
                    tma_load_3d(S.k, &tmK, &S.bar_k_full, 0, kt * kB, kvh);
                    tma_load_3d(S.k + kAtomBytes, &tmK, &S.bar_k_full, 64, kt * kB, kvh);
                    if (it > 0) mbar_wait(&S.bar_v_empty, (it - 1) & 1);
                    mbar_expect_tx(&S.bar_v_full, kTileBytes);
                    tma_load_3d(S.v, &tmV, &S.bar_v_full, 0, kt * kB, kvh);
                    tma_load_3d(S.v + kAtomBytes, &tmV, &S.bar_v_full, 64, kt * kB, kvh);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0 && ntiles > 0) {
            const uint32_t q0 = smem_u32(S.q), k0 = smem_u32(S.k), v0 = smem_u32(S.v);
            mbar_wait(&S.bar_q, 0);
            for (int it = 0; it < ntiles; ++it) {
                mbar_wait(&S.bar_k_full, it & 1);
                if (it > 0) mbar_wait(&S.bar_o_done, (it - 1) & 1);  // P(it-1) consumed
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kAtomBytes + (kk & 3) * 32;
                    mma_ss(tS, sdesc_sw128(q0 + off, 16, 1024), sdesc_sw128(k0 + off, 16, 1024),
                           kIdescQK, kk > 0 ? 1u : 0u);
                }
                mma_commit(&S.bar_s_full);
                mma_commit(&S.bar_k_empty);
                mbar_wait(&S.bar_p_full, it & 1);
                mbar_wait(&S.bar_v_full, it & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    mma_ts(tO, tS + kk * 8, sdesc_sw128(v0 + kk * 2048, kAtomBytes, 1024), kIdescPV,
                           (it > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(&S.bar_o_done);
                mma_commit(&S.bar_v_empty);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ softmax
        const int quad = warp & 3;                 // TMEM lane quadrant of this warp
        const int r = quad * 32 + lane;            // row within the query block
        const int row = qb * kB + r;               // global query row
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const float c = P.scale_log2;
        float m_used = -INFINITY;  // running max, log2 units (lazy)
        float m_raw = -INFINITY;   // true max of raw q.k
        float l = 0.f;

        for (int it = 0; it < ntiles; ++it) {
            // valid key columns of this tile for this row
            int lim;
            if (MODE == SPARSE) {
                lim = min(kB, count - it * kB);
            } else {
                const int kt = kv_tile_of(MODE, it, wsb);
                lim = min(kB, P.n - kt * kB);
                if (kt == qb) lim = min(lim, r + 1);
            }
            mbar_wait(&S.bar_s_full, it & 1);
            tc_fence_after();
            // pass 1: row max
            float mx = -INFINITY;
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t v[32];
                tmem_ld32(tS + lane_off + ch * 32, v);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (ch * 32 + j < lim) mx = fmaxf(mx, __uint_as_float(v[j]));
            }
            m_raw = fmaxf(m_raw, mx);
            const float mx2 = mx * c;
            bool rescale = false;
            float alpha = 1.f;
            if (mx2 > m_used + 8.f) {
                alpha = (m_used == -INFINITY) ? 0.f : ex2(m_used - mx2);
                m_used = mx2;
                rescale = it > 0;
            }
            l *= alpha;
            const float base = (m_used == -INFINITY) ? 0.f : m_used;
            // pass 2: P = 2^(s*c - m) as f16, written over S cols [0, 64)
            float lsum = 0.f;
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t v[32];
                tmem_ld32(tS + lane_off + ch * 32, v);
                tmem_wait_ld();
                uint32_t pk[16];
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    const int col = ch * 32 + j;
                    const float p0 = col < lim ? ex2(fmaf(__uint_as_float(v[j]), c, -base)) : 0.f;
                    const float p1 = col + 1 < lim ? ex2(fmaf(__uint_as_float(v[j + 1]), c, -base)) : 0.f;
                    lsum += p0 + p1;
                    pk[j >> 1] = pack_half2(p0, p1);
                }
                tmem_st16(tS + lane_off + ch * 16, pk);
            }
            l += lsum;
            if (__any_sync(0xffffffffu, rescale)) {  // tcgen05.ld/st are warp-collective
                if (!rescale) alpha = 1.f;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    uint32_t v[32];
                    tmem_ld32(tO + lane_off + ch * 32, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * alpha);
                    tmem_st32(tO + lane_off + ch * 32, v);
                }
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&S.bar_p_full);
        }

        // ------------------------------------------------------------ epilogue
        if (ntiles > 0) {
            mbar_wait(&S.bar_o_done, (ntiles - 1) & 1);
            tc_fence_after();
        }
        const bool valid_row = row < P.n;
        const size_t rowoff = (static_cast<size_t>(h) * P.n + (valid_row ? row : 0)) * kD;
        if (MODE == ANCHOR) {
            const float mt2 = m_raw * c;
            const float f = (m_used == -INFINITY) ? 0.f : ex2(m_used - mt2);
            float* acc = P.acc_out + rowoff;
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t v[32];
                tmem_ld32(tO + lane_off + ch * 32, v);
                tmem_wait_ld();
                if (valid_row) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        float4 o;
                        o.x = __uint_as_float(v[j]) * f;
                        o.y = __uint_as_float(v[j + 1]) * f;
                        o.z = __uint_as_float(v[j + 2]) * f;
                        o.w = __uint_as_float(v[j + 3]) * f;
                        *reinterpret_cast<float4*>(acc + ch * 32 + j) = o;
                    }
                }
            }
            const float m_nat = m_raw * P.inv_sqrt_d;
            if (valid_row) {
                P.m_out[static_cast<size_t>(h) * P.n + row] = m_nat;
                P.l_out[static_cast<size_t>(h) * P.n + row] = l * f;
            }
            // per-query-block partial sums for pooling (Alg. 2 inputs)
            if (P.msum != nullptr) {
                float ms = valid_row ? m_nat : 0.f;
#pragma unroll
                for (int o = 16; o; o >>= 1) ms += __shfl_xor_sync(0xffffffffu, ms, o);
                if (lane == 0) S.red[quad] = ms;
            }
            if (P.qsum != nullptr) {
                // column r of the Q tile, summed over its 128 rows (zero-filled past n)
                const int col = r;
                const uint8_t* atom = S.q + (col >> 6) * kAtomBytes;
                const int chunk = (col & 63) >> 3, e = col & 7;
                float s = 0.f;
                for (int rr = 0; rr < kB; ++rr) {
                    const __nv_bfloat16 x = *reinterpret_cast<const __nv_bfloat16*>(
                        atom + rr * 128 + ((chunk ^ (rr & 7)) << 4) + e * 2);
                    s += __bfloat162float(x);
                }
                P.qsum[(static_cast<size_t>(h) * P.T_m + qb) * kD + col] = s;
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (P.msum != nullptr && threadIdx.x == 64) {
                P.msum[static_cast<size_t>(h) * P.T_m + qb] =
                    static_cast<double>(S.red[0]) + S.red[1] + S.red[2] + S.red[3];
            }
        } else {
            // O = O_tiles / l  (DENSE)  or merged with the anchor state (SPARSE)
            float fa = 0.f, fs = 1.f, inv = 0.f;
            const float* acc_a = nullptr;
            if (MODE == SPARSE) {
                const float ma = valid_row ? P.m_in[static_cast<size_t>(h) * P.n + row] : 0.f;
                const float la = valid_row ? P.l_in[static_cast<size_t>(h) * P.n + row] : 1.f;
                const float ma2 = ma * kLog2e;
                const float M = fmaxf(ma2, m_used);
                fa = ex2(ma2 - M);
                fs = (m_used == -INFINITY) ? 0.f : ex2(m_used - M);
                inv = 1.f / (la * fa + l * fs);
                acc_a = P.acc_in + rowoff;
            } else {
                inv = 1.f / l;
            }
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t v[32];
                if (ntiles > 0) {
                    tmem_ld32(tO + lane_off + ch * 32, v);
                    tmem_wait_ld();
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = 0u;
                }
                if (valid_row) {
                float o[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) o[j] = __uint_as_float(v[j]) * fs;
                if (MODE == SPARSE) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const float4 a = *reinterpret_cast<const float4*>(acc_a + ch * 32 + j);
                        o[j] += a.x * fa;
                        o[j + 1] += a.y * fa;
                        o[j + 2] += a.z * fa;
                        o[j + 3] += a.w * fa;
                    }
                }
                if (P.out_bf16) {
                    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(P.out) + rowoff + ch * 32;
#pragma unroll
                    for (int j = 0; j < 32; j += 8) {
                        uint4 w;
                        __nv_bfloat162 t0 = __floats2bfloat162_rn(o[j] * inv, o[j + 1] * inv);
                        __nv_bfloat162 t1 = __floats2bfloat162_rn(o[j + 2] * inv, o[j + 3] * inv);
                        __nv_bfloat162 t2 = __floats2bfloat162_rn(o[j + 4] * inv, o[j + 5] * inv);
                        __nv_bfloat162 t3 = __floats2bfloat162_rn(o[j + 6] * inv, o[j + 7] * inv);
                        w.x = *reinterpret_cast<uint32_t*>(&t0);
                        w.y = *reinterpret_cast<uint32_t*>(&t1);
                        w.z = *reinterpret_cast<uint32_t*>(&t2);
                        w.w = *reinterpret_cast<uint32_t*>(&t3);
                        *reinterpret_cast<uint4*>(out + j) = w;
                    }
                } else {
                    float* out = static_cast<float*>(P.out) + rowoff + ch * 32;
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        *reinterpret_cast<float4*>(out + j) =
                            make_float4(o[j] * inv, o[j + 1] * inv, o[j + 2] * inv, o[j + 3] * inv);
                }
                }  // valid_row
                __syncwarp();
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 256);
}

// ------------------------------------------------------------------------ K2
// Alg. 2 (R/src/stripe_identify.cpp:31-46) on the tensor cores.
//
// For one KV head, the pooled queries of its GQA query heads form the rows
// r = g * rep + hh (group-major) of an A operand; 128 rows per CTA (one
// M-tile).  q_bar is f32 in the reference; it enters the MMA as an exact-ish
// split q_bar = hi + lo (two bf16 terms, residual ~2^-17 |q_bar|), so
// S = hi K^T + lo K^T is the f32 score to ~1e-5 — far inside the +-1e-3
// selection band — while K streams from HBM once per (head, M-tile).
// Each TMEM lane holds one (head, group) row, so its thread assembles the
// 32-bit selection words of 32 consecutive keys directly (no ballot).
//
// grid (chunks of key tiles, M-tiles, hkv); 192 threads: warp 0 TMA,
// warp 1 MMA, warps 2-5 threshold + bit words.  K ring of 2 stages, 2 TMEM
// accumulators.
constexpr int kIdChunk = 16;  // key tiles per CTA

struct IdSmem {
    uint8_t a_hi[kTileBytes];
    uint8_t a_lo[kTileBytes];
    uint8_t k[2][kTileBytes];
    uint64_t bar_a, bar_k_full[2], bar_k_empty[2], bar_s_full[2], bar_s_empty[2];
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(kThreads, 1)
    k_identify_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmK,
                  Geo geo, int rep, int rows_pad, const double* __restrict__ anchor, double theta,
                  uint32_t* __restrict__ bits, int64_t words_per_row) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    IdSmem& S = *reinterpret_cast<IdSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kvh = blockIdx.z;
    const int mt = blockIdx.y;
    const int groups = static_cast<int>(geo.groups());
    // key tiles relevant to this M-tile: up to the widest middle region of its groups
    const int g_last = min(groups - 1, ((mt + 1) * kB - 1) / rep);
    const int64_t span = geo.middle_end(g_last) - geo.b_kv;
    const int tiles_total = span > 0 ? static_cast<int>((span + kB - 1) / kB) : 0;
    const int t0 = blockIdx.x * kIdChunk;
    const int nt = max(0, min(kIdChunk, tiles_total - t0));
    if (nt == 0) return;

    if (threadIdx.x == 0) {
        mbar_init(&S.bar_a, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&S.bar_k_full[b], 1);
            mbar_init(&S.bar_k_empty[b], 1);
            mbar_init(&S.bar_s_full[b], 1);
            mbar_init(&S.bar_s_empty[b], 128);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&S.tmem_base, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(&S.bar_a, 2 * kTileBytes);
            const int arow = mt * kB;
            tma_load_3d(S.a_hi, &tmA, &S.bar_a, 0, arow, 2 * kvh);
            tma_load_3d(S.a_hi + kAtomBytes, &tmA, &S.bar_a, 64, arow, 2 * kvh);
            tma_load_3d(S.a_lo, &tmA, &S.bar_a, 0, arow, 2 * kvh + 1);
            tma_load_3d(S.a_lo + kAtomBytes, &tmA, &S.bar_a, 64, arow, 2 * kvh + 1);
            for (int i = 0; i < nt; ++i) {
                const int b = i & 1;
                if (i >= 2) mbar_wait(&S.bar_k_empty[b], ((i >> 1) - 1) & 1);
                mbar_expect_tx(&S.bar_k_full[b], kTileBytes);
                const int key0 = static_cast<int>(geo.b_kv) + (t0 + i) * kB;
                tma_load_3d(S.k[b], &tmK, &S.bar_k_full[b], 0, key0, kvh);
                tma_load_3d(S.k[b] + kAtomBytes, &tmK, &S.bar_k_full[b], 64, key0, kvh);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t ah = smem_u32(S.a_hi), al = smem_u32(S.a_lo);
            mbar_wait(&S.bar_a, 0);
            for (int i = 0; i < nt; ++i) {
                const int b = i & 1;
                mbar_wait(&S.bar_k_full[b], (i >> 1) & 1);
                if (i >= 2) mbar_wait(&S.bar_s_empty[b], ((i >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t kb = smem_u32(S.k[b]);
                const uint32_t d_tmem = tmem + b * 128;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kAtomBytes + (kk & 3) * 32;
                    mma_ss(d_tmem, sdesc_sw128(ah + off, 16, 1024), sdesc_sw128(kb + off, 16, 1024),
                           kIdescQK, kk > 0 ? 1u : 0u);
                }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kAtomBytes + (kk & 3) * 32;
                    mma_ss(d_tmem, sdesc_sw128(al + off, 16, 1024), sdesc_sw128(kb + off, 16, 1024),
                           kIdescQK, 1u);
                }
                mma_commit(&S.bar_s_full[b]);
                mma_commit(&S.bar_k_empty[b]);
            }
        }
        __syncwarp();
    } else {
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        const int grow = mt * kB + r;
        const int g = grow / rep, hh = kvh * rep + grow % rep;
        const bool valid = grow < groups * rep;
        int64_t mend = 0;
        float thr = 0.f;
        if (valid) {
            mend = geo.middle_end(g);
            const double ref = anchor ? anchor[static_cast<int64_t>(hh) * groups + g] : 0.0;
            // keep iff ref - s*inv_sqrt_d <= theta  <=>  s >= (ref - theta) * sqrt(d)
            thr = static_cast<float>((ref - theta) * sqrt(static_cast<double>(kD)));
        }
        uint32_t* rowbits = bits + (static_cast<int64_t>(hh) * groups + g) * words_per_row;
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        for (int i = 0; i < nt; ++i) {
            const int b = i & 1;
            mbar_wait(&S.bar_s_full[b], (i >> 1) & 1);
            tc_fence_after();
            const int64_t key0 = geo.b_kv + static_cast<int64_t>(t0 + i) * kB;
            uint32_t w[4];
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t v[32];
                tmem_ld32(tmem + b * 128 + lane_off + ch * 32, v);
                tmem_wait_ld();
                uint32_t word = 0;
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    word |= (__uint_as_float(v[c]) >= thr ? 1u : 0u) << c;
                const int64_t kfirst = key0 + ch * 32;
                if (kfirst + 32 > mend) {
                    const int64_t keep = mend - kfirst;
                    word = keep <= 0 ? 0u : (keep >= 32 ? word : word & ((1u << keep) - 1u));
                }
                w[ch] = word;
            }
            tc_fence_before();
            mbar_arrive(&S.bar_s_empty[b]);
            if (valid && key0 < mend) {
                const int64_t word0 = (key0 - geo.b_kv) >> 5;
                *reinterpret_cast<uint4*>(rowbits + word0) = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 256);
}

// q_bar (f32 [hq, G, d]) -> A operand rows r = g*rep + hh of KV head kvh as a
// two-term bf16 split: out[(2*kvh + 0), r, :] = hi, out[(2*kvh + 1), r, :] = lo.
__global__ void k_split_qbar(int groups, int rep, int rows_pad, const float* __restrict__ qbar,
                             __nv_bfloat16* __restrict__ out) {
    const int kvh = blockIdx.y;
    const int r = blockIdx.x;
    const int t = threadIdx.x;
    float x = 0.f;
    if (r < groups * rep) {
        const int g = r / rep, hh = kvh * rep + r % rep;
        x = qbar[(static_cast<int64_t>(hh) * groups + g) * kD + t];
    }
    const __nv_bfloat16 hi = __float2bfloat16(x);
    const __nv_bfloat16 lo = __float2bfloat16(x - __bfloat162float(hi));
    out[((2 * static_cast<int64_t>(kvh)) * rows_pad + r) * kD + t] = hi;
    out[((2 * static_cast<int64_t>(kvh) + 1) * rows_pad + r) * kD + t] = lo;
}

// Pooled query / anchor per group from K1's per-query-block partials
// (avgpool_rows / avgpool_vector, R/src/matrix.cpp:44-81).  grid (G, hq).
__global__ void k_pool_fast(Geo geo, int64_t q_rs, int64_t q_hs, const __nv_bfloat16* __restrict__ q,
                            const float* __restrict__ m, const float* __restrict__ qsum,
                            const double* __restrict__ msum, double* __restrict__ anchor,
                            float* __restrict__ qbar) {
    const int64_t g = blockIdx.x, h = blockIdx.y;
    const int64_t groups = gridDim.x, T = geo.q_blocks();
    const int64_t rb = geo.row_begin(g), re = geo.row_end(g);
    const int64_t qb0 = g * geo.step, qb1 = min(T, (g + 1) * geo.step);
    const double inv = 1.0 / static_cast<double>(re - rb);
    for (int t = threadIdx.x; t < kD; t += blockDim.x) {
        double s = 0.0;
        if (qsum) {
            for (int64_t b = qb0; b < qb1; ++b) s += qsum[(h * T + b) * kD + t];
        } else {
            for (int64_t i = rb; i < re; ++i) s += __bfloat162float(q[h * q_hs + i * q_rs + t]);
        }
        qbar[(h * groups + g) * kD + t] = static_cast<float>(s * inv);
    }
    if (threadIdx.x == 0 && anchor != nullptr) {
        double s = 0.0;
        if (msum) {
            for (int64_t b = qb0; b < qb1; ++b) s += msum[h * T + b];
        } else {
            for (int64_t i = rb; i < re; ++i) s += m[h * geo.n + i];
        }
        anchor[h * groups + g] = s / static_cast<double>(re - rb);
    }
}

__global__ void k_finalize_fast(int64_t total, int64_t d, const float* __restrict__ l,
                                const float* __restrict__ acc, void* out, int out_bf16) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float x = acc[e] / l[e / d];
        if (out_bf16) static_cast<__nv_bfloat16*>(out)[e] = __float2bfloat16(x);
        else static_cast<float*>(out)[e] = x;
    }
}

// V (bf16, strided) -> packed f16 [hkv, n, d] (exact for the f16 normal range).
__global__ void k_v_to_f16(int64_t n, int64_t hkv, int64_t rs, int64_t hs,
                           const __nv_bfloat16* __restrict__ v, __half* __restrict__ v16) {
    const int64_t total8 = hkv * n * (kD / 8);
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total8;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t hh = e / (n * (kD / 8));
        const int64_t rem = e % (n * (kD / 8));
        const int64_t i = rem / (kD / 8), c8 = rem % (kD / 8);
        const uint4 raw = *reinterpret_cast<const uint4*>(v + hh * hs + i * rs + c8 * 8);
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
        uint4 o;
        __half2* o2 = reinterpret_cast<__half2*>(&o);
#pragma unroll
        for (int u = 0; u < 4; ++u) o2[u] = __float22half2_rn(__bfloat1622float2(b2[u]));
        *reinterpret_cast<uint4*>(v16 + (hh * n + i) * kD + c8 * 8) = o;
    }
}

// ------------------------------------------------------------------ host side

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(p);
    });
    return fn;
}

// 3-D map {d, rows, heads} of 2-byte elements, box {64, 128, 1}, 128B swizzle.
cudaError_t make_map_3d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int64_t rows,
                        int64_t heads, int64_t row_stride, int64_t head_stride) {
    EncodeTiled enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(kD), static_cast<cuuint64_t>(rows),
                                static_cast<cuuint64_t>(heads)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(row_stride * 2),
                                   static_cast<cuuint64_t>(head_stride * 2)};
    const cuuint32_t box[3] = {64, 128, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 2-D map {d, total_rows} (row pitch d elements) for gather4, box {64, 1}.
cudaError_t make_map_gather(CUtensorMap* m, const void* base, CUtensorMapDataType dt,
                            int64_t total_rows) {
    EncodeTiled enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(kD), static_cast<cuuint64_t>(total_rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(kD * 2)};
    const cuuint32_t box[2] = {64, 1};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

constexpr size_t kSmemBytes = sizeof(Smem) + 1024;

template <int MODE>
cudaError_t launch_fa(const FastArgs& f, const void* q, const void* k, const void* v16,
                      FaParams P, cudaStream_t s) {
    CUtensorMap tq, tk, tv, tkg, tvg;
    cudaError_t e;
    const int64_t n = f.geo.n;
    if ((e = make_map_3d(&tq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, n, f.hq, f.q_rs, f.q_hs))) return e;
    if ((e = make_map_3d(&tk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, n, f.hkv, f.kv_rs, f.kv_hs))) return e;
    if ((e = make_map_3d(&tv, v16, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, n, f.hkv, kD, n * kD))) return e;
    const int64_t krows = ((f.hkv - 1) * f.kv_hs + (n - 1) * f.kv_rs) / kD + 1;
    if ((e = make_map_gather(&tkg, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, krows))) return e;
    if ((e = make_map_gather(&tvg, v16, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, f.hkv * n))) return e;
    P.n = static_cast<int>(n);
    P.hq = static_cast<int>(f.hq);
    P.rep = static_cast<int>(f.rep);
    P.T_m = static_cast<int>(f.geo.q_blocks());
    P.step = static_cast<int>(f.geo.step);
    P.groups = static_cast<int>(f.geo.groups());
    P.inv_sqrt_d = 1.0f / sqrtf(static_cast<float>(kD));
    P.scale_log2 = kLog2e * P.inv_sqrt_d;
    P.kv_head_rows = static_cast<int>(f.kv_hs / kD);
    P.kv_row_rows = static_cast<int>(f.kv_rs / kD);
    static bool attr_set[3] = {false, false, false};
    if (!attr_set[MODE]) {
        if ((e = cudaFuncSetAttribute(fa_tiles<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kSmemBytes))))
            return e;
        attr_set[MODE] = true;
    }
    const unsigned grid = static_cast<unsigned>(P.T_m * f.hq);
    fa_tiles<MODE><<<grid, kThreads, kSmemBytes, s>>>(tq, tk, tv, tkg, tvg, P);
    return cudaGetLastError();
}

cudaError_t convert_v(const FastArgs& f, const void* v, void* v16, cudaStream_t s) {
    const int64_t total8 = f.hkv * f.geo.n * (kD / 8);
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total8 + 255) / 256, 148 * 16));
    k_v_to_f16<<<blocks, 256, 0, s>>>(f.geo.n, f.hkv, f.kv_rs, f.kv_hs,
                                      static_cast<const __nv_bfloat16*>(v),
                                      static_cast<__half*>(v16));
    return cudaGetLastError();
}

}  // namespace

cudaError_t fast_convert_v(const FastArgs& f, const void* v, void* v16, cudaStream_t s) {
    return convert_v(f, v, v16, s);
}

cudaError_t fast_anchor(const FastArgs& f, const void* q, const void* k, const void* v16, float* m,
                        float* l, float* acc, float* qsum, double* msum, cudaStream_t s) {
    FaParams P{};
    P.m_out = m;
    P.l_out = l;
    P.acc_out = acc;
    P.qsum = qsum;
    P.msum = msum;
    return launch_fa<ANCHOR>(f, q, k, v16, P, s);
}

cudaError_t fast_pool(const FastArgs& f, const void* q, const float* m, const float* qsum,
                      const double* msum, double* anchor, float* qbar, cudaStream_t s) {
    k_pool_fast<<<dim3(static_cast<unsigned>(f.geo.groups()), static_cast<unsigned>(f.hq)), 128, 0,
                  s>>>(f.geo, f.q_rs, f.q_hs, static_cast<const __nv_bfloat16*>(q), m, qsum, msum,
                       anchor, qbar);
    return cudaGetLastError();
}

cudaError_t fast_identify(const FastArgs& f, const void* k, const float* qbar,
                          const double* anchor, uint32_t* bits, int64_t words_per_row,
                          cudaStream_t s) {
    const int64_t G = f.geo.groups();
    const int64_t max_end = f.geo.middle_end(G - 1);
    const int64_t span = max_end > f.geo.b_kv ? max_end - f.geo.b_kv : 0;
    const int64_t tiles = (span + kB - 1) / kB;
    if (tiles == 0) return cudaSuccess;
    if (words_per_row % 4) return cudaErrorInvalidValue;  // 16-byte word stores
    const int rows = static_cast<int>(G * f.rep);
    const int rows_pad = (rows + kB - 1) / kB * kB;
    void* split = nullptr;
    cudaError_t e;
    const size_t split_bytes = static_cast<size_t>(2 * f.hkv) * rows_pad * kD * 2;
    if ((e = cudaMallocAsync(&split, split_bytes, s))) return e;
    k_split_qbar<<<dim3(static_cast<unsigned>(rows_pad), static_cast<unsigned>(f.hkv)), kD, 0, s>>>(
        static_cast<int>(G), static_cast<int>(f.rep), rows_pad, qbar,
        static_cast<__nv_bfloat16*>(split));
    CUtensorMap ta, tk;
    if ((e = make_map_3d(&ta, split, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rows_pad, 2 * f.hkv, kD,
                         static_cast<int64_t>(rows_pad) * kD)) ||
        (e = make_map_3d(&tk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, f.geo.n, f.hkv, f.kv_rs,
                         f.kv_hs))) {
        cudaFreeAsync(split, s);
        return e;
    }
    constexpr size_t smem = sizeof(IdSmem) + 1024;
    static bool attr = false;
    if (!attr) {
        if ((e = cudaFuncSetAttribute(k_identify_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)))) {
            cudaFreeAsync(split, s);
            return e;
        }
        attr = true;
    }
    const unsigned chunks = static_cast<unsigned>((tiles + kIdChunk - 1) / kIdChunk);
    k_identify_tc<<<dim3(chunks, static_cast<unsigned>(rows_pad / kB), static_cast<unsigned>(f.hkv)),
                    kThreads, smem, s>>>(ta, tk, f.geo, static_cast<int>(f.rep), rows_pad, anchor,
                                         f.theta, bits, words_per_row);
    e = cudaGetLastError();
    cudaFreeAsync(split, s);
    return e;
}

cudaError_t fast_sparse(const FastArgs& f, const void* q, const void* k, const void* v16,
                        const float* m, const float* l, const float* acc,
                        const uint32_t* indices, const int32_t* counts, const int64_t* offsets,
                        int64_t cap, bool csr, void* out, aa_dtype out_dtype, cudaStream_t s) {
    FaParams P{};
    P.m_in = m;
    P.l_in = l;
    P.acc_in = acc;
    P.idx = indices;
    P.counts = counts;
    P.offsets = offsets;
    P.cap = cap;
    P.csr = csr ? 1 : 0;
    P.out = out;
    P.out_bf16 = out_dtype == AA_BF16;
    return launch_fa<SPARSE>(f, q, k, v16, P, s);
}

cudaError_t fast_finalize(const FastArgs& f, const float* l, const float* acc, void* out,
                          aa_dtype out_dtype, cudaStream_t s) {
    const int64_t total = f.hq * f.geo.n * kD;
    k_finalize_fast<<<static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 32)), 256,
                      0, s>>>(total, kD, l, acc, out, out_dtype == AA_BF16);
    return cudaGetLastError();
}

cudaError_t fast_dense(const FastArgs& f, const void* q, const void* k, const void* v16, void* out,
                       aa_dtype out_dtype, cudaStream_t s) {
    FaParams P{};
    P.out = out;
    P.out_bf16 = out_dtype == AA_BF16;
    return launch_fa<DENSE>(f, q, k, v16, P, s);
}

cudaError_t fast_recall(const FastArgs&, const void*, const void*, const uint32_t*, const int32_t*,
                        const int64_t*, int64_t, double*, double*, cudaStream_t) {
    return cudaErrorNotSupported;
}

}  // namespace aa
