// Fast path (AA_BF16): hand-written sm_100a kernels for b_q = b_kv = 128,
// d = 128.
//
//   K1 anchor   fa_pair<ANCHOR>  tile list {0} ∪ [wsb(g), qb]          (Alg. 1)
//   K2 identify k_identify_tc    pooled-q · K on tcgen05, threshold  (Alg. 2)
//   K3 sparse   fa_pair<SPARSE>  gathered stripe tiles (TMA gather4),
//                                merged with the K1 state             (Alg. 3)
//   D  dense    fa_pair<DENSE>   tiles 0..qb (causal baseline)
//
// fa_pair (see its comment): one CTA = two 128-row query blocks of one head
// sharing every K/V tile; TMA producer warp(s), one MMA warp issuing
// tcgen05.mma from an elected lane, two softmax warpgroups ping-ponging on the
// tensor pipe; S/P/O in TMEM.
// Softmax is exp2-based with lazy rescaling (O/l rescaled only when the
// running max grows by > 8 in log2 units); the state written out is exact
// (rescaled to the true max).  PV runs in f16 (P in [0, 256] keeps 11
// mantissa bits; V converted bf16 -> f16 once, exact for |v| in the f16
// normal range).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <mutex>

#include "fast.h"
#include "kernels.h"
#include "sm100.cuh"

namespace aa {
namespace {

using namespace sm100;

constexpr int kB = 128;  // b_q = b_kv
constexpr int kD = 128;  // head dim
constexpr int kPairThreads = 384;   // fa_pair CTA
// K ring depth of fa_pair (V keeps 2 stages): K(j + kKStages) can be fetched as
// soon as QK_B(j) has read stage j — one more tile of lead for the gathers.
#ifndef AA_K_STAGES
#define AA_K_STAGES 2
#endif
constexpr int kKStages = AA_K_STAGES;
constexpr uint32_t kTileBytes = kB * kD * 2;   // 32 KB (bf16 / f16 tile)
constexpr uint32_t kAtomBytes = kB * 64 * 2;   // 16 KB: 128 rows x 128 B (SW128 atom column)
constexpr uint32_t kIdescQK = idesc_f16(1, 1, 0, 128, 128);  // bf16 x bf16, B K-major
constexpr uint32_t kIdescPV = idesc_f16(0, 0, 1, 128, 128);  // f16 x f16,  B MN-major
constexpr float kLog2e = 1.4426950408889634f;
// Exp2 pairs per 32 columns computed by ex2_poly2 on the FMA pipe instead of
// MUFU (16 results / clock / SM on B200: one 128 x 128 tile costs >= 1100
// MUFU cycles per warp, as much as the tile's MMAs).  Measured per kernel
// (128k Llama, elect-issued MMAs): K1 0 / 2 / 4 pairs -> 3.47 / 3.28-3.33 /
// 3.26-3.28 ms; K3 0 / 2 / 4 -> 16.3 / 16.8-17.1 / 16.8-16.9 ms (the heavier
// softmax stream slows the MMA hand-off there).  So K1 offloads 4 of 16.
#ifndef AA_POLY_PAIRS
#define AA_POLY_PAIRS 0
#endif
// K3: warps issuing the K-row gathers (1: warp 0; 2: warps 0 and 2, one
// column half each)
#ifndef AA_K3_KGATHER_WARPS
#define AA_K3_KGATHER_WARPS 2
#endif
constexpr int kKGatherWarps = AA_K3_KGATHER_WARPS;
// softmax -> MMA hand-off arrivals per query tile: 128 (every thread) or 4
// (one per warp after __syncwarp: measured 0.6-0.9% slower in K3)
#ifndef AA_P_ARRIVALS
#define AA_P_ARRIVALS 128
#endif
constexpr int kPArrivals = AA_P_ARRIVALS;
// K3: warps issuing the V-row gathers (1: warp 3; 2: warps 3 and 12, one column
// half each — the CTA then has a fourth warpgroup, warps 12-15, and the
// softmax warpgroups 208 instead of 224 registers per thread)
#ifndef AA_K3_VGATHER_WARPS
#define AA_K3_VGATHER_WARPS 2
#endif
constexpr int kVGatherWarps = AA_K3_VGATHER_WARPS;
// K3 work order: 1 = KV-head-major (every item of one KV head — its groups
// heavy-first, then its query heads, then pairs — before the next KV head's),
// so the ~74 clusters running at once gather from one KV head's K / V rows
// and find them in L2: K3 DRAM read 5.06 -> 2.44 GB per layer, L2 hit rate
// 73.7 -> 82.7% (ncu, 128k Llama).  0 = group-major over all heads.
#ifndef AA_K3_KV_MAJOR
#define AA_K3_KV_MAJOR 1
#endif
#ifndef AA_POLY_PAIRS_K1
#define AA_POLY_PAIRS_K1 4
#endif

// Optional cycle accounting of the fa_pair roles (build with -DAA_PROF; read
// through aa_prof_read).  Slots: 0/1 softmax-A wait-S / compute, 2 softmax-A
// tiles, 3/4/5 MMA wait P / K / V, 6 CTA cycles, 7 epilogue (softmax A),
// 8 prologue (to the first S), 9 CTAs, 10 producer wait-empty, 11/12
// softmax-B wait-S / compute; 20/21/22 ~first CTA start / last CTA end /
// sum of CTA lifetimes (globaltimer ns).
#ifdef AA_PROF
__device__ unsigned long long g_prof[6][32];  // [fa_pair MODE | 5 = K2 identify][slot]
#define PROF(...) __VA_ARGS__
#else
#define PROF(...)
#endif

// RECALL: the dense causal QK pass without PV, accumulating per row the
// softmax mass of all keys and of the selected keys (covered ∪ stripes).
// TILEMASS: a second QK-only pass that uses RECALL's per-row (max, sum) to
// write the exact softmax mass of every (query block, key block) tile.
enum Mode { ANCHOR = 0, SPARSE = 1, DENSE = 2, RECALL = 3, TILEMASS = 4 };

template <int MODE>
constexpr bool kQkOnly = MODE == RECALL || MODE == TILEMASS;
template <int MODE>
constexpr bool kWideK3 = MODE == SPARSE && kVGatherWarps == 2;
template <int MODE>
constexpr int kThreadsOf = kWideK3<MODE> ? 512 : kPairThreads;
// register split of the wide K3 CTA (per thread; 128 x role + 128 x wg3 +
// 256 x softmax <= 65536): role warpgroup (MMA + gathers), fourth warpgroup,
// softmax warpgroups
#ifndef AA_K3_REGS_ROLE
#define AA_K3_REGS_ROLE 56
#endif
#ifndef AA_K3_REGS_WG3
#define AA_K3_REGS_WG3 40
#endif
#ifndef AA_K3_REGS_SOFTMAX
#define AA_K3_REGS_SOFTMAX 208
#endif
constexpr int kWideRegs[3] = {AA_K3_REGS_ROLE, AA_K3_REGS_WG3, AA_K3_REGS_SOFTMAX};
constexpr uint32_t kWg3Regs = kWideRegs[1];
constexpr uint32_t kWideSoftmaxRegs = kWideRegs[2];
static_assert(128 * kWideRegs[0] + 128 * kWideRegs[1] + 256 * kWideRegs[2] <= 65536, "wide K3 register split");
template <int MODE>
constexpr uint32_t kRoleRegs = kWideK3<MODE> ? kWideRegs[0] : 56;

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
    int cluster;  // K3: CTAs per cluster sharing gathered tiles (1 = none)
    int item0;    // first work item of this launch (K3 split launches)
    int g_end;    // work items cover groups [g_end - n_groups, g_end)
    int n_groups;
    // K1 -> K3 hand-off format: 0 = acc f32 unnormalised (AnchorState::acc,
    // the stage API); 1 = f16 acc / l (normalised, |.| <= max|v|: half the
    // bytes both ways; the fused chain)
    int acc_f16;
    // RECALL inputs / output
    const uint32_t* bits;   // selection bitmask [hq, G, words_per_row]
    int64_t words_per_row;
    double* row_recall;     // [hq, n]: selected / total softmax mass per row
    float2* row_stats;      // [hq, n]: (running max in log2 units, sum) — RECALL out, TILEMASS in
    float* tile_mass;       // [hq, T_m, T_n] TILEMASS output
    int T_n;
};

// Shared memory of fa_pair: two query tiles, 2-stage K and V rings.
struct PairSmem {
    uint8_t q[2][kTileBytes];
    uint8_t k[kKStages][kTileBytes];
    uint8_t v[2][kTileBytes];
    uint64_t bar_q, bar_qsum, bar_acc[2];
    uint64_t bar_k_full[kKStages], bar_k_empty[kKStages], bar_v_full[2], bar_v_empty[2];
    uint64_t bar_s_full[2], bar_p_full[2], bar_o_done[2];  // per query tile
    uint32_t tmem_base;
    float red[2][2][4];
    float row_scale[2][kB];  // K3 epilogue: per-row weight of K1's state
};

__device__ __forceinline__ int kv_tile_of(int mode, int it, int wsb) {
    if (mode == DENSE || mode == RECALL || mode == TILEMASS) return it;
    return it == 0 ? 0 : wsb + it - 1;  // ANCHOR: {0} then [wsb, qb]
}

// One CTA = two query blocks (A = qb, B = qb + 1) of one head and one group;
// they share every K/V tile (and for K3 the same gathered stripe rows), so
// each tile is loaded once for 256 query rows.  12 warps:
//   warp 0      TMA producer (Q pair once; K and V through 2-stage rings;
//               in K3 the K-row gathers only)
//   warp 1      TMEM allocator (512 columns) + MMA issuer (the whole warp runs
//               the loop with warp-uniform operands, one elected lane issues)
//   warps 2-3   K1: pooled column sums of Q; K3: warp 3 gathers the V rows
//   warps 4-7   softmax / epilogue of query tile A   (TMEM lanes 0..127)
//   warps 8-11  softmax / epilogue of query tile B
// TMEM: S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512); P_X is written
// as f16 over S_X columns [0,64) and consumed from TMEM by O_X += P_X V.
// MMA order per tile j:  PV_A(j) QK_A(j+1) PV_B(j) QK_B(j+1) — the tensor
// pipe works on one tile's MMAs while the other tile's softmax runs (FA4-style
// ping-pong); tcgen05 MMAs of one thread execute in issue order, so QK_X(j+1)
// overwriting S_X after PV_X(j) has read P_X is ordered by the pipe.
template <int MODE>
__global__ void __launch_bounds__(kThreadsOf<MODE>, 1)
    fa_pair(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
            const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmKg,
            const __grid_constant__ CUtensorMap tmVg, const FaParams P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    PairSmem& S = *reinterpret_cast<PairSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    PROF(const long long t_cta0 = clock64(); unsigned long long ns_cta0;
         asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns_cta0));)

    // work item: heavy-first (last groups first).  Within a group, the pairs of
    // one head are adjacent, then the heads of one KV head: CTAs that run
    // together gather the same stripe rows (one list per (head, group); GQA
    // siblings select mostly the same keys), so the gathers hit L2.  K3 goes
    // further and runs one KV head's items at a time (AA_K3_KV_MAJOR).
    const int ipg = (P.step + 1) / 2;  // query-block pairs per group
    const int L = blockIdx.x + P.item0;
#if AA_K3_KV_MAJOR
    // K3: KV-head-major — all of one KV head's items (heavy groups first,
    // then its query heads, then pairs) before the next KV head's, so the
    // CTAs running at once gather from one KV head's K/V (L2-resident)
    int gi, h, pi;
    if (MODE == SPARSE) {
        const int per_kv = P.n_groups * P.rep * ipg;
        const int kvb = L / per_kv, r2 = L % per_kv;
        gi = P.g_end - 1 - r2 / (P.rep * ipg);
        const int r3 = r2 % (P.rep * ipg);
        h = kvb * P.rep + r3 / ipg;
        pi = ipg - 1 - r3 % ipg;
    } else {
        gi = P.g_end - 1 - L / (ipg * P.hq);
        const int rem = L % (ipg * P.hq);
        h = rem / ipg;
        pi = ipg - 1 - rem % ipg;
    }
#else
    const int gi = P.g_end - 1 - L / (ipg * P.hq);
    const int rem = L % (ipg * P.hq);
    const int h = rem / ipg;
    const int pi = ipg - 1 - rem % ipg;
#endif
    const int kvh = h / P.rep;
    const int qA = gi * P.step + 2 * pi;
    // K3 cluster mode: a pair past the last query block of a partial group
    // still walks the group's stripe tiles (it gathers its share of every
    // multicast tile for its peer) on a query tile that lies wholly past n —
    // TMA zero-fills it and every store of it is clipped / masked by row < n.
    // Otherwise such a CTA has no work.
    if (qA >= P.T_m && !(MODE == SPARSE && P.cluster > 1)) return;
    const bool hasB = (2 * pi + 1 < P.step) && (qA + 1 < P.T_m);
    const int qB = qA + 1;

    int nA = 0, nB = 0, wsb = 0, count = 0;
    const uint32_t* list = nullptr;
    if (MODE == DENSE || kQkOnly<MODE>) {
        nA = qA + 1;
        nB = hasB ? qB + 1 : 0;
    } else if (MODE == ANCHOR) {
        const int rb = gi * P.step * kB;
        wsb = rb < 2 * kB ? 1 : rb / kB - 1;
        nA = 1 + (qA >= wsb ? qA - wsb + 1 : 0);
        nB = hasB ? 1 + (qB - wsb + 1) : 0;
    } else {
        count = P.counts[h * P.groups + gi];
        list = P.csr ? P.idx + P.offsets[h * P.groups + gi] : P.idx + h * P.cap + P.offsets[gi];
        nA = (count + kB - 1) / kB;
        nB = hasB ? nA : 0;
    }
    const int ntiles = nA > nB ? nA : nB;

    // K3 cluster mode (P.cluster = C > 1): the C CTAs of a cluster are C pairs
    // of the same (head, group) and so walk the same gathered tiles; each CTA
    // gathers 128/C rows of every tile and multicasts them to all C CTAs, and
    // a K/V stage is refilled only after all C consumers released it.
    const int C = MODE == SPARSE ? P.cluster : 1;
    const uint32_t crank = C > 1 ? cluster_ctarank() : 0;
    const uint16_t cmask = static_cast<uint16_t>((1u << C) - 1u);

    if (threadIdx.x == 0) {
        mbar_init(&S.bar_q, 1);
        mbar_init(&S.bar_qsum, 64);
        mbar_init(&S.bar_acc[0], 1);
        mbar_init(&S.bar_acc[1], 1);
        for (int b = 0; b < kKStages; ++b) {
            mbar_init(&S.bar_k_full[b], 1);
            mbar_init(&S.bar_k_empty[b], C);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&S.bar_v_full[b], 1);
            mbar_init(&S.bar_v_empty[b], C);
            mbar_init(&S.bar_s_full[b], 1);
            mbar_init(&S.bar_p_full[b], kPArrivals);
            mbar_init(&S.bar_o_done[b], 1);
        }
        fence_mbar_init();
        // The loads that need no peer: the Q pair and (contiguous-tile modes)
        // the first K / V tile go out now, overlapping the TMEM allocation
        // and the (cluster) barrier below.
        if (ntiles > 0) {
            mbar_expect_tx(&S.bar_q, hasB ? 2 * kTileBytes : kTileBytes);
            tma_load_3d(S.q[0], &tmQ, &S.bar_q, 0, qA * kB, h);
            tma_load_3d(S.q[0] + kAtomBytes, &tmQ, &S.bar_q, 64, qA * kB, h);
            if (hasB) {
                tma_load_3d(S.q[1], &tmQ, &S.bar_q, 0, qB * kB, h);
                tma_load_3d(S.q[1] + kAtomBytes, &tmQ, &S.bar_q, 64, qB * kB, h);
            }
            if (MODE != SPARSE) {
                const int kt = kv_tile_of(MODE, 0, wsb);
                mbar_expect_tx(&S.bar_k_full[0], kTileBytes);
                tma_load_3d(S.k[0], &tmK, &S.bar_k_full[0], 0, kt * kB, kvh);
                tma_load_3d(S.k[0] + kAtomBytes, &tmK, &S.bar_k_full[0], 64, kt * kB, kvh);
                if (!kQkOnly<MODE>) {
                    mbar_expect_tx(&S.bar_v_full[0], kTileBytes);
                    tma_load_3d(S.v[0], &tmV, &S.bar_v_full[0], 0, kt * kB, kvh);
                    tma_load_3d(S.v[0] + kAtomBytes, &tmV, &S.bar_v_full[0], 64, kt * kB, kvh);
                }
            }
        }
    }
    // K3 gather warps (0: K rows, 3: V rows) read the first stripe tile's row
    // indices before the (cluster) barrier; later tiles' one tile ahead
    const int g_lanes = 32 / C;
    const int g_row0 = static_cast<int>(crank) * (kB / C) + lane * 4;
    auto stripe_rows = [&](int it, bool isK, int (&r)[4]) {
        const int base = it * kB;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = base + g_row0 + u;
            const int j = lane < g_lanes ? static_cast<int>(list[e < count ? e : base]) : 0;
            r[u] = isK ? kvh * P.kv_head_rows + j * P.kv_row_rows : kvh * P.n + j;
        }
    };
    int pre_r[4] = {0, 0, 0, 0};
    if (MODE == SPARSE && ntiles > 0 && (warp == 0 || warp == 2 || warp == 3 || warp == 12))
        stripe_rows(0, warp == 0 || warp == 2, pre_r);
    if (warp == 1) tmem_alloc(&S.tmem_base, 512);
    tc_fence_before();
    if (C > 1) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;
    // register split (per warpgroup, inside each role branch): the producer /
    // MMA warpgroup needs few registers, the two softmax warpgroups hold a
    // whole S row (128 f32) each.
    // K3 split gathers: one warp streams the K rows, another the V rows of
    // every stripe tile (gather4: 4 rows x 128 B per instruction, x 2 column
    // halves); in a cluster of C each CTA gathers rows [crank*128/C, +128/C)
    // of a tile and multicasts them to the C CTAs.
    // halves: 3 = both column halves of every row; 1 / 2 = only the first /
    // second 64 columns (two warps share one operand's gathers: a warp issues
    // its lanes' gather4 ops one after another, ~70-90 cycles each, so the
    // issue rate scales with the number of issuing warps —
    // profiles/probes/gather4_rate.txt).  The warp owning half 0 arms the
    // stage's full barrier for the whole tile.
    auto gather_split = [&](bool isK, int halves) {
        const bool gl = lane < g_lanes;
        int r[4] = {pre_r[0], pre_r[1], pre_r[2], pre_r[3]};
        for (int it = 0; it < ntiles; ++it) {
            const int st = isK ? it % kKStages : it & 1;
            const int ph = isK ? it / kKStages : it >> 1;
            const int depth = isK ? kKStages : 2;
            uint64_t* full = isK ? &S.bar_k_full[st] : &S.bar_v_full[st];
            uint64_t* empty = isK ? &S.bar_k_empty[st] : &S.bar_v_empty[st];
            if (lane == 0) {
                if (it >= depth) mbar_wait(empty, (ph - 1) & 1);
                if (halves & 1) mbar_expect_tx(full, kTileBytes);
            }
            __syncwarp();
            uint8_t* dst = (isK ? S.k[st] : S.v[st]) + g_row0 * 128;
            const CUtensorMap* tm = isK ? &tmKg : &tmVg;
            if (gl) {
                if (C > 1) {
                    if (halves & 1) tma_gather4_mc(dst, tm, full, cmask, 0, r[0], r[1], r[2], r[3]);
                    if (halves & 2) tma_gather4_mc(dst + kAtomBytes, tm, full, cmask, 64, r[0], r[1], r[2], r[3]);
                } else {
                    if (halves & 1) tma_gather4(dst, tm, full, 0, r[0], r[1], r[2], r[3]);
                    if (halves & 2) tma_gather4(dst + kAtomBytes, tm, full, 64, r[0], r[1], r[2], r[3]);
                }
            }
            if (it + 1 < ntiles) stripe_rows(it + 1, isK, r);  // next tile's rows, ahead of its stage
        }
    };

    if (warp == 0) {
        setmaxnreg_dec<kRoleRegs<MODE>>();
        // ------------------------------------------------------------ producer
        // (the Q pair and the first contiguous K / V tile were issued at init)
        if (MODE == SPARSE) {
            gather_split(true, kKGatherWarps == 2 ? 1 : 3);  // K rows (warp 2: the second half)
        } else if (MODE != SPARSE) {
            for (int it = 1; it < ntiles; ++it) {
                if (lane == 0) {
                    const int st = it & 1;
                    const int sk = it % kKStages;
                    const int kt = kv_tile_of(MODE, it, wsb);
                    PROF(const long long t0 = clock64();)
                    if (it >= kKStages) mbar_wait(&S.bar_k_empty[sk], ((it / kKStages) - 1) & 1);
                    PROF(atomicAdd(&g_prof[MODE][10], clock64() - t0);)
                    mbar_expect_tx(&S.bar_k_full[sk], kTileBytes);
                    tma_load_3d(S.k[sk], &tmK, &S.bar_k_full[sk], 0, kt * kB, kvh);
                    tma_load_3d(S.k[sk] + kAtomBytes, &tmK, &S.bar_k_full[sk], 64, kt * kB, kvh);
                    if (!kQkOnly<MODE>) {
                        if (it >= 2) mbar_wait(&S.bar_v_empty[st], ((it >> 1) - 1) & 1);
                        mbar_expect_tx(&S.bar_v_full[st], kTileBytes);
                        tma_load_3d(S.v[st], &tmV, &S.bar_v_full[st], 0, kt * kB, kvh);
                        tma_load_3d(S.v[st] + kAtomBytes, &tmV, &S.bar_v_full[st], 64, kt * kB, kvh);
                    }
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        setmaxnreg_dec<kRoleRegs<MODE>>();
        // ------------------------------------------------------------ MMA issuer
        if (ntiles > 0) {  // the whole warp runs the loop; one elected lane issues
            // SW128 descriptors: the high word (SBO 1024, version, layout) is a
            // constant, the low word = start address >> 4 | LBO >> 4 << 16
            constexpr uint64_t kDescHi = sdesc_sw128_hi(1024);
            const uint32_t lq0 = sdesc_sw128_lo(smem_u32(S.q[0]), 16);
            const uint32_t lq1 = sdesc_sw128_lo(smem_u32(S.q[1]), 16);
            const uint32_t lk0 = sdesc_sw128_lo(smem_u32(S.k[0]), 16);
            const uint32_t lv0 = sdesc_sw128_lo(smem_u32(S.v[0]), kAtomBytes);
            PROF(long long pw_p = 0, pw_k = 0, pw_v = 0;)
            auto qk = [&](int X, int j) {
                const int st = j % kKStages;
                PROF(const long long t0 = clock64();)
                mbar_wait(&S.bar_k_full[st], (j / kKStages) & 1);
                PROF(pw_k += clock64() - t0;)
                tc_fence_after();
                // descriptors are built once; the k-step only moves the start
                // address field (addr >> 4, no carry below 256 KB)
                const uint32_t lq = X ? lq1 : lq0, lk = lk0 + st * (kTileBytes >> 4);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = ((kk >> 2) * kAtomBytes + (kk & 3) * 32) >> 4;
                    mma_ss_w(tmem + X * 128, kDescHi | (lq + off), kDescHi | (lk + off), kIdescQK,
                           kk > 0 ? 1u : 0u);
                }
                mma_commit_w(&S.bar_s_full[X]);
            };
            auto pv = [&](int X, int j) {
                const int st = j & 1;
                PROF(const long long t0 = clock64();)
                mbar_wait_handoff(&S.bar_p_full[X], j & 1);
                PROF(const long long t1 = clock64(); pw_p += t1 - t0;)
                if (kQkOnly<MODE>) return;  // S_X(j) consumed; no PV
                mbar_wait(&S.bar_v_full[st], (j >> 1) & 1);
                PROF(pw_v += clock64() - t1;)
                tc_fence_after();
                const uint32_t lv = lv0 + st * (kTileBytes >> 4);
                const uint32_t tS = tmem + X * 128, tO = tmem + 256 + X * 128;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts_w(tO, tS + kk * 8, kDescHi | (lv + kk * (2048 >> 4)), kIdescPV,
                           (j > 0 || kk > 0) ? 1u : 0u);
                // O_X is read only by the epilogue: one completion, after the last PV
                if (j + 1 == (X ? nB : nA)) mma_commit_w(&S.bar_o_done[X]);
            };
            // a stage is released to every producer of the cluster that fills it
            auto release = [&](uint64_t* bar) {
                if (C > 1) mma_commit_mc_w(bar, cmask); else mma_commit_w(bar);
            };
            mbar_wait(&S.bar_q, 0);
            if (nA > 0) qk(0, 0);
            if (nB > 0) qk(1, 0);
            release(&S.bar_k_empty[0]);
            for (int j = 0; j < ntiles; ++j) {
                if (j < nA) {
                    pv(0, j);
                    if (j + 1 < nA) qk(0, j + 1);
                }
                if (j < nB) {
                    pv(1, j);
                    if (j + 1 < nB) qk(1, j + 1);
                }
                if (!kQkOnly<MODE>) release(&S.bar_v_empty[j & 1]);  // no V ring in the QK-only passes
                if (j + 1 < ntiles) release(&S.bar_k_empty[(j + 1) % kKStages]);
            }
            if (C > 1) {
                // every CTA's last releases have landed here before the exit
                // cluster barrier, so no remote arrive can target a retired CTA
                const int jl = ntiles - 1;
                mbar_wait(&S.bar_k_empty[jl % kKStages], (jl / kKStages) & 1);
                mbar_wait(&S.bar_v_empty[jl & 1], (jl >> 1) & 1);
            }
            PROF(atomicAdd(&g_prof[MODE][3], pw_p); atomicAdd(&g_prof[MODE][4], pw_k); atomicAdd(&g_prof[MODE][5], pw_v);)
        }
        __syncwarp();
    } else if (warp < 4) {
        setmaxnreg_dec<kRoleRegs<MODE>>();  // warp 3: K3's V-row gathers; warps 2-3: K1's column sums
        if (MODE == SPARSE && warp == 3) gather_split(false, kWideK3<MODE> ? 1 : 3);
        if (MODE == SPARSE && kKGatherWarps == 2 && warp == 2) gather_split(true, 2);
        if (MODE == ANCHOR && P.qsum != nullptr && ntiles > 0) {
            // pooled-query partials (avgpool_rows, R/src/matrix.cpp:44-65): column
            // sums of each query tile over its 128 rows (TMA zero-fills rows past
            // n), summed in row order; thread t owns columns 2t, 2t+1.  Runs
            // beside the main loop, off the epilogue's critical path.
            const int t = threadIdx.x - 64;
            const int col = 2 * t;
            const int chunk = (col & 63) >> 3, e = col & 7;
            mbar_wait(&S.bar_q, 0);
            for (int X = 0; X < (hasB ? 2 : 1); ++X) {
                const uint8_t* atom = S.q[X] + (col >> 6) * kAtomBytes + e * 2;
                float s0 = 0.f, s1 = 0.f;
#pragma unroll 16
                for (int rr = 0; rr < kB; ++rr) {
                    const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(
                        atom + rr * 128 + ((chunk ^ (rr & 7)) << 4));
                    s0 += __low2float(x);
                    s1 += __high2float(x);
                }
                *reinterpret_cast<float2*>(P.qsum + (static_cast<size_t>(h) * P.T_m + (X ? qB : qA)) * kD + col) =
                    make_float2(s0, s1);
            }
            mbar_arrive(&S.bar_qsum);  // the epilogue reuses the Q tiles as staging
        }
    } else if (kWideK3<MODE> && warp >= 12) {
        setmaxnreg_dec<kWg3Regs>();  // K3's fourth warpgroup: the second half of the V-row gathers
        // (warps 13-15 stay idle: more issuing / polling warps measured slower,
        // profiles/r2_experiments)
        if (warp == 12) gather_split(false, 2);
    } else {
        if constexpr (kWideK3<MODE>) setmaxnreg_inc<kWideSoftmaxRegs>();
        else setmaxnreg_inc<224>();
        // ------------------------------------------------------------ softmax
        const int X = warp >= 8 ? 1 : 0;
        // P_X (or S_X consumed) -> MMA warp: one arrival per warp (after every
        // lane's own tcgen05.st / fence), or one per thread
        auto arrive_p = [&](int x) {
            if (kPArrivals == 4) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.bar_p_full[x]);
            } else {
                mbar_arrive(&S.bar_p_full[x]);
            }
        };
        const int nX = X ? nB : nA;
        const int qx = X ? qB : qA;
        if (X == 1 && !hasB) {
            // no second query block in this item
        } else {
            const int quad = warp & 3;
            const int r = quad * 32 + lane;
            const int row = qx * kB + r;
            const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
            const uint32_t tS = tmem + X * 128 + lane_off;
            const uint32_t tO = tmem + 256 + X * 128 + lane_off;
            const float c = P.scale_log2;
            float m_used = -INFINITY;  // running max, log2 units (lazy)
            float m_raw = -INFINITY;   // true max of raw q.k
            float l = 0.f;
            float l_sel = 0.f;         // RECALL: mass of the selected keys
            // RECALL: this row group's stripe bitmask row and window start
            const uint32_t* bits_x = nullptr;
            int wstart_x = 0;
            if (MODE == RECALL) {
                bits_x = P.bits + (static_cast<int64_t>(h) * P.groups + gi) * P.words_per_row;
                const int rb = gi * P.step * kB;
                const int wsbx = rb < 2 * kB ? 1 : rb / kB - 1;
                wstart_x = min(wsbx * kB, P.n);
            }

            PROF(long long ps_wait = 0, ps_comp = 0, ps_t1 = 0, ps_first = 0;)
            for (int it = 0; it < nX; ++it) {
                int lim;
                if (MODE == SPARSE) {
                    lim = min(kB, count - it * kB);
                } else {
                    const int kt = kv_tile_of(MODE, it, wsb);
                    lim = min(kB, P.n - kt * kB);
                    if (kt == qx) lim = min(lim, r + 1);
                }
                PROF(const long long ps_t0 = clock64();)
                mbar_wait_handoff(&S.bar_s_full[X], it & 1);
                PROF(ps_t1 = clock64(); ps_wait += ps_t1 - ps_t0; if (it == 0) ps_first = ps_t1;)
                tc_fence_after();
                // single pass: the whole S row in registers
                uint32_t v[128];
                // P = 2^(s*c - base) as f16 over S columns [16 ch, 16 ch + 16)
                // for S columns [32 ch, 32 ch + 32); accumulates the row sum
                auto emit_chunk = [&](int ch, float base, float2& lsum) {
                    uint32_t pk[16];
#pragma unroll
                    for (int jj = 0; jj < 32; jj += 2) {
                        const float2 x = ffma2(make_float2(__uint_as_float(v[ch * 32 + jj]),
                                                           __uint_as_float(v[ch * 32 + jj + 1])),
                                               c, -base);
                        const float2 pp = (jj >> 1) % 16 < (MODE == ANCHOR ? AA_POLY_PAIRS_K1 : AA_POLY_PAIRS)
                                              ? ex2_poly2(x)
                                                                      : make_float2(ex2(x.x), ex2(x.y));
                        lsum = fadd2(lsum, pp);
                        pk[jj >> 1] = pack_half2(pp.x, pp.y);
                    }
                    tmem_st16(tS + ch * 16, pk);
                };
                auto emit = [&](float base) -> float {
                    float2 lsum = make_float2(0.f, 0.f);
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch) emit_chunk(ch, base, lsum);
                    return lsum.x + lsum.y;
                };
                auto mask_chunk = [&](int ch) {
                    if (lim < kB) {  // causal diagonal / sequence tail / list tail
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj)
                            if (ch * 32 + jj >= lim) v[ch * 32 + jj] = 0xff800000u;  // -inf -> p = 0
                    }
                };
                tmem_ld32(tS + 0, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                tmem_ld32(tS + 64, *reinterpret_cast<uint32_t(*)[32]>(&v[64]));
                tmem_ld32(tS + 96, *reinterpret_cast<uint32_t(*)[32]>(&v[96]));
                tmem_wait_ld();
                PROF(if (lane == 0 && warp == 4) {
                    reg_fence32(&v[96]);
                    atomicAdd(&g_prof[MODE][16], clock64() - ps_t1);
                })
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) mask_chunk(ch);
                if constexpr (MODE == TILEMASS) {
                    // exact normalised mass of this (query block, key tile):
                    // per-row sum with RECALL's final (max, sum), reduced over
                    // the 128 rows of the query tile
                    float rm = 0.f;
                    if (row < P.n) {
                        const float2 st = P.row_stats[static_cast<size_t>(h) * P.n + row];
                        float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
                        for (int jj = 0; jj < kB; jj += 2) {
                            const float2 x = ffma2(make_float2(__uint_as_float(v[jj]),
                                                               __uint_as_float(v[jj + 1])),
                                                   c, -st.x);
                            acc2 = fadd2(acc2, make_float2(ex2(x.x), ex2(x.y)));
                        }
                        rm = (acc2.x + acc2.y) / st.y;
                    }
                    tc_fence_before();
                    arrive_p(X);  // S consumed
#pragma unroll
                    for (int sh = 16; sh; sh >>= 1) rm += __shfl_xor_sync(0xffffffffu, rm, sh);
                    if (lane == 0) S.red[X][it & 1][quad] = rm;
                    if (X == 0) asm volatile("bar.sync 1, 128;" ::: "memory");
                    else asm volatile("bar.sync 2, 128;" ::: "memory");
                    if (quad == 0 && lane == 0)
                        P.tile_mass[(static_cast<size_t>(h) * P.T_m + qx) * P.T_n + it] =
                            S.red[X][it & 1][0] + S.red[X][it & 1][1] + S.red[X][it & 1][2] +
                            S.red[X][it & 1][3];
                    continue;
                }
                if constexpr (MODE == RECALL) {
                    const float mx = row_max128(v);
                    m_raw = fmaxf(m_raw, mx);
                    const float mx2 = mx * c;
                    float alpha = 1.f;
                    if (mx2 > m_used + 8.f) {
                        alpha = (m_used == -INFINITY) ? 0.f : ex2(m_used - mx2);
                        m_used = mx2;
                    }
                    l *= alpha;
                    const float base = (m_used == -INFINITY) ? 0.f : m_used;
                    // selected keys of this tile for this row's group: the initial
                    // block and the local window are covered; middle keys are
                    // selected iff their stripe bit is set
                    l_sel *= alpha;
                    const int kt = it;
                    uint32_t sel[4] = {~0u, ~0u, ~0u, ~0u};
                    if (kt > 0 && kt * kB < wstart_x) {
                        const uint4 w = *reinterpret_cast<const uint4*>(bits_x + 4 * (kt - 1));
                        sel[0] = w.x, sel[1] = w.y, sel[2] = w.z, sel[3] = w.w;
                    }
                    float2 la = make_float2(0.f, 0.f), ls = make_float2(0.f, 0.f);
#pragma unroll
                    for (int jj = 0; jj < kB; jj += 2) {
                        const float2 x = ffma2(make_float2(__uint_as_float(v[jj]),
                                                           __uint_as_float(v[jj + 1])),
                                               c, -base);
                        const float2 pp = make_float2(ex2(x.x), ex2(x.y));
                        la = fadd2(la, pp);
                        const uint32_t wd = sel[jj >> 5];
                        ls = fadd2(ls, make_float2((wd >> (jj & 31)) & 1u ? pp.x : 0.f,
                                                   (wd >> ((jj + 1) & 31)) & 1u ? pp.y : 0.f));
                    }
                    l += la.x + la.y;
                    l_sel += ls.x + ls.y;
                    tc_fence_before();
                    arrive_p(X);
                    continue;
                }
                if (it == 0) {
                    // first tile: the row max sets the base
                    const float mx = row_max128(v);
                    m_raw = mx;
                    m_used = mx * c;
                    l = emit(m_used == -INFINITY ? 0.f : m_used);
                } else {
                    // Speculative: exponentials against the running (lazy) base
                    // while the row max is reduced off the critical path; P values
                    // up to 2^8 are fine in f16.  Only if the max grew by more than
                    // 2^8 (rare) is the tile redone with the new base and O / l
                    // rescaled.
                    const float lsum = emit(m_used);
                    const float mx = row_max128(v);
                    m_raw = fmaxf(m_raw, mx);
                    const float mx2 = mx * c;
                    const bool redo = mx2 > m_used + 8.f;
                    if (__any_sync(0xffffffffu, redo)) {  // tcgen05.ld/st are warp-collective
                        const float alpha = redo ? ex2(m_used - mx2) : 1.f;
                        if (redo) m_used = mx2;
                        l = l * alpha + emit(m_used);
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) {
                            uint32_t o[32];
                            tmem_ld32(tO + ch * 32, o);
                            tmem_wait_ld();
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj)
                                o[jj] = __float_as_uint(__uint_as_float(o[jj]) * alpha);
                            tmem_st32(tO + ch * 32, o);
                        }
                    } else {
                        l += lsum;
                    }
                }
                tmem_wait_st();
                tc_fence_before();
                PROF(ps_comp += clock64() - ps_t1;)
                arrive_p(X);
            }
            PROF(const long long t_epi0 = clock64();)

            // -------------------------------------------------------- epilogue
            if (kQkOnly<MODE>) {
                if (MODE == RECALL && row < P.n) {
                    P.row_recall[static_cast<size_t>(h) * P.n + row] =
                        static_cast<double>(l_sel) / static_cast<double>(l);
                    if (P.row_stats)
                        P.row_stats[static_cast<size_t>(h) * P.n + row] = make_float2(m_used, l);
                }
            } else {
            // K3 with the f16 hand-off: K1's state for this row (m, l and the
            // 256-B acc / l row) is loaded before waiting for the last PV, all
            // in flight at once, instead of chunk by chunk behind each TMEM read
            float pre_m = 0.f, pre_l = 1.f;
            const bool prefetch = MODE == SPARSE && P.acc_f16;
            // ... and (bf16 output) the acc / l tile in the coalesced order of
            // the staged pass below (thread r: 8 B at float4 slot i*128 + r)
            uint2 pre_a[2][16];
            if (prefetch) {
                if (row < P.n) {
                    const size_t ri = static_cast<size_t>(h) * P.n + row;
                    pre_m = P.m_in[ri];
                    pre_l = P.l_in[ri];
                }
                const int rows_v = P.out_bf16 ? min(kB, P.n - qx * kB) : 0;  // f32 out: TMA path
                const __half* acc_h = reinterpret_cast<const __half*>(P.acc_in) +
                                      (static_cast<size_t>(h) * P.n + qx * kB) * kD;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf)
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int rr = (i * kB + r) >> 4;
                        pre_a[hf][i] = rr < rows_v ? *reinterpret_cast<const uint2*>(
                                                         acc_h + static_cast<size_t>(rr) * kD + hf * 64 + (r & 15) * 4)
                                                   : make_uint2(0u, 0u);
                    }
            }
            if (nX > 0) {
                mbar_wait(&S.bar_o_done[X], 0);
                tc_fence_after();
            }
            PROF(if (lane == 0 && warp == 4) atomicAdd(&g_prof[MODE][13], clock64() - t_epi0);)
            if constexpr (MODE == ANCHOR) {
                // acc_out = O * f (the state rescaled to the true max) leaves
                // through shared memory so that the global stores are coalesced
                // (a warp instruction covers 512 contiguous bytes instead of 32
                // rows x 16 B)
                const bool valid_row = row < P.n;
                const float mt2 = m_raw * c;
                const float so = (m_used == -INFINITY) ? 0.f : ex2(m_used - mt2);
                // staged values: O * so (acc, f32 hand-off) or O / l (f16 hand-off)
                const float sv = P.acc_f16 ? 1.f / l : so;
                const float m_nat = m_raw * P.inv_sqrt_d;
                if (valid_row) {
                    P.m_out[static_cast<size_t>(h) * P.n + row] = m_nat;
                    P.l_out[static_cast<size_t>(h) * P.n + row] = l * so;
                }
                if (P.msum != nullptr) {
                    float ms = valid_row ? m_nat : 0.f;
#pragma unroll
                    for (int o = 16; o; o >>= 1) ms += __shfl_xor_sync(0xffffffffu, ms, o);
                    if (lane == 0) S.red[X][0][quad] = ms;
                }
                // staging: this tile's Q buffer (its last QK has completed and the
                // column sums are done), 128 rows x 64 f32 per half, 16-B chunks
                // XOR-swizzled by row
                if (P.qsum != nullptr && nX > 0) mbar_wait(&S.bar_qsum, 0);
                if (P.acc_f16) {
                    // acc / l in f16, staged in this tile's Q buffer (its last
                    // QK has completed, the column sums are done) in the
                    // 128B-swizzled layout of a TMA box {64, 128}, then two
                    // TMA stores (async; rows past n are clipped by the map)
                    uint8_t* stg = S.q[X];
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch) {
                        uint32_t v[32];
                        tmem_ld32(tO + ch * 32, v);
                        tmem_wait_ld();
#pragma unroll
                        for (int c8 = 0; c8 < 4; ++c8) {  // 8 columns = one 16-B chunk
                            const int col = ch * 32 + c8 * 8;
                            uint4 w;
                            w.x = pack_half2(__uint_as_float(v[c8 * 8 + 0]) * sv, __uint_as_float(v[c8 * 8 + 1]) * sv);
                            w.y = pack_half2(__uint_as_float(v[c8 * 8 + 2]) * sv, __uint_as_float(v[c8 * 8 + 3]) * sv);
                            w.z = pack_half2(__uint_as_float(v[c8 * 8 + 4]) * sv, __uint_as_float(v[c8 * 8 + 5]) * sv);
                            w.w = pack_half2(__uint_as_float(v[c8 * 8 + 6]) * sv, __uint_as_float(v[c8 * 8 + 7]) * sv);
                            const int chunk = (col & 63) >> 3;
                            *reinterpret_cast<uint4*>(stg + (col >> 6) * kAtomBytes + r * 128 +
                                                      ((chunk ^ (r & 7)) << 4)) = w;
                        }
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(1 + X, 128);
                    if (quad == 0 && lane == 0) {
                        tma_store_3d(&tmVg, stg, 0, qx * kB, h);
                        tma_store_3d(&tmVg, stg + kAtomBytes, 64, qx * kB, h);
                        tma_store_commit();
                        tma_store_wait_read();  // the CTA may exit once the box is read
                    }
                } else {  // f32 acc (the stage API's AnchorState::acc): coalesced LSU stores
                    float* stg = reinterpret_cast<float*>(S.q[X]);
                    const int rows_valid = min(kB, P.n - qx * kB);
                    const size_t gbase = (static_cast<size_t>(h) * P.n + qx * kB) * kD;
                    for (int half = 0; half < 2; ++half) {
                        if (half) named_bar_sync(1 + X, 128);  // half 0 drained from the staging buffer
                        uint32_t v[64];
                        tmem_ld32(tO + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                        tmem_ld32(tO + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                        tmem_wait_ld();
    #pragma unroll
                        for (int ch = 0; ch < 16; ++ch)
                            *reinterpret_cast<float4*>(stg + r * 64 + ((ch ^ (r & 15)) << 2)) = make_float4(
                                __uint_as_float(v[4 * ch]) * sv, __uint_as_float(v[4 * ch + 1]) * sv,
                                __uint_as_float(v[4 * ch + 2]) * sv, __uint_as_float(v[4 * ch + 3]) * sv);
                        named_bar_sync(1 + X, 128);
                        // thread r copies float4 i*128 + r (row idx/16, chunk idx%16): a
                        // warp instruction spans two rows' 256 contiguous bytes
                        const int ch = r & 15;
    #pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const int rr = (i * kB + r) >> 4;
                            const float4 o = *reinterpret_cast<const float4*>(stg + rr * 64 + ((ch ^ (rr & 15)) << 2));
                            if (rr < rows_valid) {
                                const size_t ge = gbase + static_cast<size_t>(rr) * kD + half * 64 + ch * 4;
                                if (P.acc_f16) {
                                    uint2 w;
                                    w.x = pack_half2(o.x, o.y);
                                    w.y = pack_half2(o.z, o.w);
                                    *reinterpret_cast<uint2*>(reinterpret_cast<__half*>(P.acc_out) + ge) = w;
                                } else {
                                    *reinterpret_cast<float4*>(P.acc_out + ge) = o;
                                }
                            }
                        }
                    }
                }
                if (P.msum != nullptr && quad == 0 && lane == 0) {
                    // S.red was written before the staging barriers above
                    P.msum[static_cast<size_t>(h) * P.T_m + qx] =
                        static_cast<double>(S.red[X][0][0]) + S.red[X][0][1] + S.red[X][0][2] + S.red[X][0][3];
                }
            } else if (MODE == SPARSE && P.acc_f16 && !P.out_bf16) {
                // merge with K1's state (f16 acc / l) entirely through TMA:
                //   out = O * (fs * inv) + acc_n * (la * fa * inv)
                // acc_n tile -> a free K stage (every QK is complete), then per
                // row (thread = TMEM lane = row) the merged f32 values go to a
                // staging buffer in the 128B-swizzled box layout {32, 128} and
                // leave by TMA store, 64 columns at a time (Q_X for columns
                // 0-63, a V stage PV no longer reads for columns 64-127)
                const float ma2 = pre_m * kLog2e;
                const float M = fmaxf(ma2, m_used);
                const float fa = ex2(ma2 - M);
                const float fs = (m_used == -INFINITY) ? 0.f : ex2(m_used - M);
                const float inv = 1.f / (pre_l * fa + l * fs);
                const float so = fs * inv, sa = pre_l * fa * inv;
                const bool issue = quad == 0 && lane == 0;
                uint8_t* accb = S.k[X];
                if (issue) {
                    mbar_expect_tx(&S.bar_acc[X], kTileBytes);
                    tma_load_3d(accb, &tmK, &S.bar_acc[X], 0, qx * kB, h);
                    tma_load_3d(accb + kAtomBytes, &tmK, &S.bar_acc[X], 64, qx * kB, h);
                }
                mbar_wait(&S.bar_acc[X], 0);
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    uint8_t* dst = half ? S.v[X ? ((nX - 1) & 1) : (nX & 1)] : S.q[X];
                    uint32_t v[64];
                    if (nX > 0) {
                        tmem_ld32(tO + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                        tmem_ld32(tO + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                        tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 64; ++jj) v[jj] = 0u;
                    }
#pragma unroll
                    for (int c8 = 0; c8 < 8; ++c8) {  // 8 columns: one 16-B f16 chunk of acc
                        const uint4 araw = *reinterpret_cast<const uint4*>(
                            accb + half * kAtomBytes + r * 128 + ((c8 ^ (r & 7)) << 4));
                        const __half2* a2 = reinterpret_cast<const __half2*>(&araw);
#pragma unroll
                        for (int u = 0; u < 2; ++u) {  // two f32 16-B chunks
                            const float2 a01 = __half22float2(a2[2 * u]);
                            const float2 a23 = __half22float2(a2[2 * u + 1]);
                            const int c = c8 * 8 + u * 4;  // column within the half (0..63)
                            const float4 o = make_float4(
                                __uint_as_float(v[c]) * so + a01.x * sa, __uint_as_float(v[c + 1]) * so + a01.y * sa,
                                __uint_as_float(v[c + 2]) * so + a23.x * sa, __uint_as_float(v[c + 3]) * so + a23.y * sa);
                            const int chunk = (c & 31) >> 2;
                            *reinterpret_cast<float4*>(dst + (c >> 5) * kAtomBytes + r * 128 +
                                                       ((chunk ^ (r & 7)) << 4)) = o;
                        }
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(1 + X, 128);
                    if (issue) {
                        tma_store_3d(&tmV, dst, half * 64, qx * kB, h);
                        tma_store_3d(&tmV, dst + kAtomBytes, half * 64 + 32, qx * kB, h);
                        tma_store_commit();
                    }
                }
                if (issue) tma_store_wait_read();  // the CTA may exit once both halves are read
            } else if (MODE == SPARSE && P.acc_f16) {
                // merge with K1's state (f16 acc / l hand-off) and leave through
                // shared memory so that loads and stores are coalesced:
                //   out = O * (fs * inv) + acc_n * (la * fa * inv)
                // the first term is staged per row (TMEM lane = row), the second
                // added in the coalesced pass (row scalar from shared memory)
                const bool valid_row = row < P.n;
                const float ma2 = pre_m * kLog2e;
                const float M = fmaxf(ma2, m_used);
                const float fa = ex2(ma2 - M);
                const float fs = (m_used == -INFINITY) ? 0.f : ex2(m_used - M);
                const float inv = 1.f / (pre_l * fa + l * fs);
                const float so = fs * inv;
                S.row_scale[X][r] = valid_row ? pre_l * fa * inv : 0.f;
                float* stg = reinterpret_cast<float*>(S.q[X]);
                const int rows_valid = min(kB, P.n - qx * kB);
                const size_t gbase = (static_cast<size_t>(h) * P.n + qx * kB) * kD;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    if (half) named_bar_sync(1 + X, 128);  // half 0 drained from the staging buffer
                    uint32_t v[64];
                    if (nX > 0) {
                        tmem_ld32(tO + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                        tmem_ld32(tO + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                        tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 64; ++jj) v[jj] = 0u;
                    }
#pragma unroll
                    for (int ch = 0; ch < 16; ++ch)
                        *reinterpret_cast<float4*>(stg + r * 64 + ((ch ^ (r & 15)) << 2)) = make_float4(
                            __uint_as_float(v[4 * ch]) * so, __uint_as_float(v[4 * ch + 1]) * so,
                            __uint_as_float(v[4 * ch + 2]) * so, __uint_as_float(v[4 * ch + 3]) * so);
                    named_bar_sync(1 + X, 128);
                    PROF(if (half == 0 && lane == 0 && warp == 4) atomicAdd(&g_prof[MODE][14], clock64() - t_epi0);)
                    // thread r covers float4 i*128 + r (row idx/16, chunk idx%16)
                    const int ch = r & 15;
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int rr = (i * kB + r) >> 4;
                        if (rr >= rows_valid) continue;
                        float4 o = *reinterpret_cast<const float4*>(stg + rr * 64 + ((ch ^ (rr & 15)) << 2));
                        const float sa = S.row_scale[X][rr];
                        const uint2 a4 = pre_a[half][i];
                        const float2 a01 = __half22float2(*reinterpret_cast<const __half2*>(&a4.x));
                        const float2 a23 = __half22float2(*reinterpret_cast<const __half2*>(&a4.y));
                        o.x += a01.x * sa;
                        o.y += a01.y * sa;
                        o.z += a23.x * sa;
                        o.w += a23.y * sa;
                        const size_t ge = gbase + static_cast<size_t>(rr) * kD + half * 64 + ch * 4;
                        if (P.out_bf16) {
                            __nv_bfloat162 t0 = __floats2bfloat162_rn(o.x, o.y);
                            __nv_bfloat162 t1 = __floats2bfloat162_rn(o.z, o.w);
                            uint2 w;
                            w.x = *reinterpret_cast<uint32_t*>(&t0);
                            w.y = *reinterpret_cast<uint32_t*>(&t1);
                            *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(P.out) + ge) = w;
                        } else {
                            *reinterpret_cast<float4*>(static_cast<float*>(P.out) + ge) = o;
                        }
                    }
                    PROF(if (half == 0 && lane == 0 && warp == 4) atomicAdd(&g_prof[MODE][15], clock64() - t_epi0);)
                }
            } else {
            const bool valid_row = row < P.n;
            const size_t rowoff = (static_cast<size_t>(h) * P.n + (valid_row ? row : 0)) * kD;
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
                    if (nX > 0) {
                        tmem_ld32(tO + ch * 32, v);
                        tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) v[jj] = 0u;
                    }
                    if (valid_row) {
                        float o[32];
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) o[jj] = __uint_as_float(v[jj]) * fs;
                        if (MODE == SPARSE) {
#pragma unroll
                            for (int jj = 0; jj < 32; jj += 4) {
                                const float4 a = *reinterpret_cast<const float4*>(acc_a + ch * 32 + jj);
                                o[jj] += a.x * fa;
                                o[jj + 1] += a.y * fa;
                                o[jj + 2] += a.z * fa;
                                o[jj + 3] += a.w * fa;
                            }
                        }
                        if (P.out_bf16) {
                            __nv_bfloat16* out = static_cast<__nv_bfloat16*>(P.out) + rowoff + ch * 32;
#pragma unroll
                            for (int jj = 0; jj < 32; jj += 8) {
                                uint4 w;
                                __nv_bfloat162 t0 = __floats2bfloat162_rn(o[jj] * inv, o[jj + 1] * inv);
                                __nv_bfloat162 t1 = __floats2bfloat162_rn(o[jj + 2] * inv, o[jj + 3] * inv);
                                __nv_bfloat162 t2 = __floats2bfloat162_rn(o[jj + 4] * inv, o[jj + 5] * inv);
                                __nv_bfloat162 t3 = __floats2bfloat162_rn(o[jj + 6] * inv, o[jj + 7] * inv);
                                w.x = *reinterpret_cast<uint32_t*>(&t0);
                                w.y = *reinterpret_cast<uint32_t*>(&t1);
                                w.z = *reinterpret_cast<uint32_t*>(&t2);
                                w.w = *reinterpret_cast<uint32_t*>(&t3);
                                *reinterpret_cast<uint4*>(out + jj) = w;
                            }
                        } else {
                            float* out = static_cast<float*>(P.out) + rowoff + ch * 32;
#pragma unroll
                            for (int jj = 0; jj < 32; jj += 4)
                                *reinterpret_cast<float4*>(out + jj) = make_float4(
                                    o[jj] * inv, o[jj + 1] * inv, o[jj + 2] * inv, o[jj + 3] * inv);
                        }
                    }
                    __syncwarp();
                }
            }
            }  // MODE != RECALL
            PROF(if (lane == 0 && (warp == 4 || warp == 8)) {
                const int o = warp == 4 ? 0 : 11;
                atomicAdd(&g_prof[MODE][o], ps_wait);
                atomicAdd(&g_prof[MODE][o + 1], ps_comp);
                if (warp == 4) {
                    atomicAdd(&g_prof[MODE][2], static_cast<unsigned long long>(nX));
                    atomicAdd(&g_prof[MODE][7], clock64() - t_epi0);
                    if (nX > 0) atomicAdd(&g_prof[MODE][8], ps_first - t_cta0);
                }
            })
        }
    }

    tc_fence_before();
    if (C > 1) cluster_sync(); else __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 512);
    PROF(if (threadIdx.x == 0) {
        atomicAdd(&g_prof[MODE][6], clock64() - t_cta0);
        atomicAdd(&g_prof[MODE][9], 1ull);
        // SM occupancy: sum of CTA lifetimes vs the launch span (globaltimer)
        unsigned long long ns1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns1));
        atomicMax(&g_prof[MODE][20], ~ns_cta0);
        atomicMax(&g_prof[MODE][21], ns1);
        atomicAdd(&g_prof[MODE][22], ns1 - ns_cta0);
    })
}

// ------------------------------------------------------------------------ K2
// Alg. 2 (R/src/stripe_identify.cpp:31-46) on the tensor cores.
//
// For one KV head, the pooled queries of its GQA query heads form the rows
// r = g * rep + hh (group-major) of an A operand, 128 rows per M-tile.  q_bar
// is f32 in the reference; it enters the MMA as an exact-ish split
// q_bar = hi + lo (two bf16 terms, residual ~2^-17 |q_bar|), so
// S = hi K^T + lo K^T is the f32 score to ~1e-5 — far inside the +-1e-3
// selection band.  Each TMEM lane holds one (head, group) row, so its thread
// assembles the 32-bit selection words of 32 consecutive keys directly.
//
// One CTA owns a KV head and a PAIR of M-tiles (both A operands resident,
// 128 KB) and walks every J-th chunk of 8 key tiles of that head, so each K
// tile is read from HBM exactly once and feeds the MMAs of both M-tiles (the
// first M-tile holds the earlier groups and stops at its shorter middle
// region).  Strided chunks balance the two-tile and one-tile parts of the
// key range across the J CTAs of a head.  K streams through a 3-stage TMA
// ring; TMEM holds 2 M-tiles x 2 accumulators.  320 threads: warp 0 TMA,
// warp 1 MMA (+ TMEM), warps 2-9 threshold + bit words (warps 2-5 M-tile 0,
// 6-9 M-tile 1; thread <-> TMEM lane <-> (head, group) row).
constexpr int kIdThreads = 320;
constexpr int kIdChunk = 8;    // key tiles per chunk
constexpr int kIdStages = 3;   // K ring depth

struct IdSmem {
    uint8_t a[2][2][kTileBytes];  // [M-tile of the pair][hi, lo]
    uint8_t k[kIdStages][kTileBytes];
    uint64_t bar_a;
    uint64_t bar_k_full[kIdStages], bar_k_empty[kIdStages];
    uint64_t bar_s_full[2][2], bar_s_empty[2][2];  // [M-tile][accumulator]
    uint32_t tmem_base;
};

struct IdWork {
    Geo geo;
    int rep, n_mt, n_pairs, J;
    int g0, gr;  // A-operand rows cover groups [g0, g0 + gr)
};

// Key tiles of M-tile mt: up to the widest middle region of its groups.
__device__ __forceinline__ int id_tiles(const IdWork& w, int mt) {
    if (mt >= w.n_mt) return 0;
    const int g_last = w.g0 + min(w.gr - 1, ((mt + 1) * kB - 1) / w.rep);
    const int64_t span = w.geo.middle_end(g_last) - w.geo.b_kv;
    return span > 0 ? static_cast<int>((span + kB - 1) / kB) : 0;
}

__global__ void __launch_bounds__(kIdThreads, 1)
    k_identify_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmK,
                  const IdWork w, const double* __restrict__ anchor, double theta,
                  uint32_t* __restrict__ bits, int64_t words_per_row) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    IdSmem& S = *reinterpret_cast<IdSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    PROF(const long long t_cta0 = clock64();)
    const int groups = static_cast<int>(w.geo.groups());
    const int j0 = blockIdx.x % w.J;
    const int pair = (blockIdx.x / w.J) % w.n_pairs;
    const int kvh = blockIdx.x / (w.J * w.n_pairs);
    const int mt0 = 2 * pair;
    const int T0 = id_tiles(w, mt0), T1 = id_tiles(w, mt0 + 1);
    const int T = max(T0, T1);
    const int nchunks = (T + kIdChunk - 1) / kIdChunk;
    const int my_chunks = nchunks > j0 ? (nchunks - j0 + w.J - 1) / w.J : 0;
    if (my_chunks == 0) return;
    const bool two = T1 > 0;
    // this CTA's i-th chunk, alternating from both ends of its list: chunks
    // where both M-tiles are live (tensor-heavy) interleave with one-tile
    // chunks (HBM-heavy), so at any moment the CTAs load both pipes
    auto chunk_at = [&](int i) { return j0 + w.J * ((i & 1) ? my_chunks - 1 - (i >> 1) : (i >> 1)); };

    if (threadIdx.x == 0) {
        mbar_init(&S.bar_a, 1);
        for (int b = 0; b < kIdStages; ++b) {
            mbar_init(&S.bar_k_full[b], 1);
            mbar_init(&S.bar_k_empty[b], 1);
        }
        for (int m = 0; m < 2; ++m)
            for (int b = 0; b < 2; ++b) {
                mbar_init(&S.bar_s_full[m][b], 1);
                mbar_init(&S.bar_s_empty[m][b], 128);
            }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&S.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(&S.bar_a, (two ? 4 : 2) * kTileBytes);
            for (int m = 0; m < (two ? 2 : 1); ++m) {
                const int arow = (mt0 + m) * kB;
                tma_load_3d(S.a[m][0], &tmA, &S.bar_a, 0, arow, 2 * kvh);
                tma_load_3d(S.a[m][0] + kAtomBytes, &tmA, &S.bar_a, 64, arow, 2 * kvh);
                tma_load_3d(S.a[m][1], &tmA, &S.bar_a, 0, arow, 2 * kvh + 1);
                tma_load_3d(S.a[m][1] + kAtomBytes, &tmA, &S.bar_a, 64, arow, 2 * kvh + 1);
            }
            int nk = 0;
            for (int ci = 0; ci < my_chunks; ++ci) {
                const int c = chunk_at(ci);
                const int t_end = min(T, (c + 1) * kIdChunk);
                for (int t = c * kIdChunk; t < t_end; ++t, ++nk) {
                    const int b = nk % kIdStages;
                    PROF(const long long t0 = clock64();)
                    if (nk >= kIdStages) mbar_wait(&S.bar_k_empty[b], ((nk / kIdStages) - 1) & 1);
                    PROF(atomicAdd(&g_prof[5][0], clock64() - t0);)
                    mbar_expect_tx(&S.bar_k_full[b], kTileBytes);
                    const int key0 = static_cast<int>(w.geo.b_kv) + t * kB;
                    tma_load_3d(S.k[b], &tmK, &S.bar_k_full[b], 0, key0, kvh);
                    tma_load_3d(S.k[b] + kAtomBytes, &tmK, &S.bar_k_full[b], 64, key0, kvh);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        {  // the whole warp runs the loop; one elected lane issues (warp-uniform operands)
            constexpr uint64_t kDescHi = sdesc_sw128_hi(1024);
            const uint32_t la0 = sdesc_sw128_lo(smem_u32(S.a[0][0]), 16);
            const uint32_t lk0 = sdesc_sw128_lo(smem_u32(S.k[0]), 16);
            mbar_wait(&S.bar_a, 0);
            int nk = 0;
            int ns[2] = {0, 0};
            for (int ci = 0; ci < my_chunks; ++ci) {
                const int c = chunk_at(ci);
                const int t_end = min(T, (c + 1) * kIdChunk);
                for (int t = c * kIdChunk; t < t_end; ++t, ++nk) {
                    const int b = nk % kIdStages;
                    PROF(const long long t0 = clock64();)
                    mbar_wait(&S.bar_k_full[b], (nk / kIdStages) & 1);
                    PROF(if (lane == 0) { atomicAdd(&g_prof[5][1], clock64() - t0); atomicAdd(&g_prof[5][9], 1ull); })
                    const uint32_t lk = lk0 + b * (kTileBytes >> 4);
#pragma unroll
                    for (int m = 0; m < 2; ++m) {
                        if (t >= (m ? T1 : T0)) continue;  // this M-tile's groups end earlier
                        const int sb = ns[m] & 1;
                        PROF(const long long t0 = clock64();)
                        if (ns[m] >= 2) mbar_wait(&S.bar_s_empty[m][sb], ((ns[m] >> 1) - 1) & 1);
                        PROF(if (lane == 0) atomicAdd(&g_prof[5][2], clock64() - t0);)
                        tc_fence_after();
                        const uint32_t lhi = la0 + m * (2 * kTileBytes >> 4), llo = lhi + (kTileBytes >> 4);
                        const uint32_t d_tmem = tmem + (2 * m + sb) * 128;
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint32_t off = ((kk >> 2) * kAtomBytes + (kk & 3) * 32) >> 4;
                            mma_ss_w(d_tmem, kDescHi | (lhi + off), kDescHi | (lk + off), kIdescQK,
                                   kk > 0 ? 1u : 0u);
                        }
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint32_t off = ((kk >> 2) * kAtomBytes + (kk & 3) * 32) >> 4;
                            mma_ss_w(d_tmem, kDescHi | (llo + off), kDescHi | (lk + off), kIdescQK, 1u);
                        }
                        mma_commit_w(&S.bar_s_full[m][sb]);
                        ++ns[m];
                    }
                    mma_commit_w(&S.bar_k_empty[b]);
                }
            }
        }
        __syncwarp();
    } else {
        const int m = (warp - 2) >> 2;  // M-tile of the pair
        const int quad = warp & 3;      // TMEM lane quadrant of this warp
        const int r = quad * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
        const int Tm = m ? T1 : T0;
        const int grow = (mt0 + m) * kB + r;
        const int g = w.g0 + grow / w.rep, hh = kvh * w.rep + grow % w.rep;
        const bool valid = grow < w.gr * w.rep;
        int64_t mend = 0;
        float thr = 0.f;
        if (valid) {
            mend = w.geo.middle_end(g);
            const double ref = anchor ? anchor[static_cast<int64_t>(hh) * groups + g] : 0.0;
            // keep iff ref - s*inv_sqrt_d <= theta  <=>  s >= (ref - theta) * sqrt(d)
            thr = static_cast<float>((ref - theta) * sqrt(static_cast<double>(kD)));
        }
        uint32_t* rowbits = bits + (static_cast<int64_t>(valid ? hh : 0) * groups + (valid ? g : 0)) * words_per_row;
        int ns = 0;
        for (int ci = 0; ci < my_chunks; ++ci) {
            const int c = chunk_at(ci);
            const int t_end = min(Tm, (c + 1) * kIdChunk);
            for (int t = c * kIdChunk; t < t_end; ++t, ++ns) {
                const int sb = ns & 1;
                PROF(const long long t0 = clock64();)
                mbar_wait(&S.bar_s_full[m][sb], (ns >> 1) & 1);
                PROF(const long long t1 = clock64(); if (lane == 0 && (warp == 2 || warp == 6)) atomicAdd(&g_prof[5][3], t1 - t0);)
                tc_fence_after();
                const int64_t key0 = w.geo.b_kv + static_cast<int64_t>(t) * kB;
                uint32_t wd[4];
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    uint32_t v[32];
                    tmem_ld32(tmem + (2 * m + sb) * 128 + lane_off + ch * 32, v);
                    tmem_wait_ld();
                    // bit cc = (s_cc >= thr): the sign bit of s - thr (+0 when
                    // equal) shifted in from the top, highest key first, so a
                    // FADD2 and one funnel shift per key; the word holds the
                    // rejected keys and is inverted once
                    uint32_t neg = 0;
#pragma unroll
                    for (int cc = 30; cc >= 0; cc -= 2) {
                        const float2 dd = fadd2(make_float2(__uint_as_float(v[cc]), __uint_as_float(v[cc + 1])),
                                                make_float2(-thr, -thr));
                        neg = __funnelshift_l(__float_as_uint(dd.y), neg, 1);
                        neg = __funnelshift_l(__float_as_uint(dd.x), neg, 1);
                    }
                    uint32_t word = ~neg;
                    const int64_t kfirst = key0 + ch * 32;
                    if (kfirst + 32 > mend) {
                        const int64_t keep = mend - kfirst;
                        word = keep <= 0 ? 0u : (keep >= 32 ? word : word & ((1u << keep) - 1u));
                    }
                    wd[ch] = word;
                }
                tc_fence_before();
                mbar_arrive(&S.bar_s_empty[m][sb]);
                if (valid && key0 < mend) {
                    const int64_t word0 = (key0 - w.geo.b_kv) >> 5;
                    *reinterpret_cast<uint4*>(rowbits + word0) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
                }
                PROF(if (lane == 0 && (warp == 2 || warp == 6)) { atomicAdd(&g_prof[5][4], clock64() - t1); atomicAdd(&g_prof[5][5], 1ull); })
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 512);
    PROF(if (threadIdx.x == 0) { atomicAdd(&g_prof[5][6], clock64() - t_cta0); atomicAdd(&g_prof[5][7], 1ull); })
}

// q_bar (f32 [hq, G, d]) -> A operand rows r = (g - g0)*rep + hh of KV head kvh
// (groups [g0, g0 + gr)) as a two-term bf16 split: out[(2*kvh + 0), r, :] = hi,
// out[(2*kvh + 1), r, :] = lo.
__global__ void k_split_qbar(int groups, int g0, int gr, int rep, int rows_pad,
                             const float* __restrict__ qbar, __nv_bfloat16* __restrict__ out) {
    const int kvh = blockIdx.y;
    const int r = blockIdx.x;
    const int t = threadIdx.x;
    float x = 0.f;
    if (r < gr * rep) {
        const int g = g0 + r / rep, hh = kvh * rep + r % rep;
        x = qbar[(static_cast<int64_t>(hh) * groups + g) * kD + t];
    }
    const __nv_bfloat16 hi = __float2bfloat16(x);
    const __nv_bfloat16 lo = __float2bfloat16(x - __bfloat162float(hi));
    out[((2 * static_cast<int64_t>(kvh)) * rows_pad + r) * kD + t] = hi;
    out[((2 * static_cast<int64_t>(kvh) + 1) * rows_pad + r) * kD + t] = lo;
}

// Pooled query / anchor per group from K1's per-query-block partials
// (avgpool_rows / avgpool_vector, R/src/matrix.cpp:44-81).  grid (G, hq).
__global__ void k_pool_fast(Geo geo, int64_t g0, int64_t q_rs, int64_t q_hs,
                            const __nv_bfloat16* __restrict__ q, const float* __restrict__ m,
                            const float* __restrict__ qsum, const double* __restrict__ msum,
                            double* __restrict__ anchor, float* __restrict__ qbar) {
    const int64_t g = g0 + blockIdx.x, h = blockIdx.y;
    const int64_t groups = geo.groups(), T = geo.q_blocks();
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

// Capacity-layout (or CSR) stripe lists -> selection bitmask rows [hq, G, W]
// (bit j - b_kv of row (h, g)); the RECALL pass reads these.
__global__ void k_scatter_bits(Geo geo, const uint32_t* __restrict__ indices,
                               const int32_t* __restrict__ counts,
                               const int64_t* __restrict__ offsets, int64_t cap,
                               uint32_t* __restrict__ bits, int64_t wpr) {
    const int64_t g = blockIdx.x, h = blockIdx.y, G = gridDim.x;
    const int64_t cnt = counts[h * G + g];
    const uint32_t* list = indices + h * cap + offsets[g];
    uint32_t* row = bits + (h * G + g) * wpr;
    const int64_t lo = geo.b_kv, hi = geo.window_start(g);
    for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) {
        const int64_t j = list[e];
        if (j < lo || j >= hi) continue;  // covered keys count once (union_mask)
        atomicOr(row + ((j - lo) >> 5), 1u << ((j - lo) & 31));
    }
}

// recall[h] = mean over rows of the per-row captured mass (metrics.cpp:8-19).
__global__ void k_recall_sum(int64_t n, const double* __restrict__ rows, double* __restrict__ recall) {
    __shared__ double red[256];
    const int64_t h = blockIdx.x;
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += rows[h * n + i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) recall[h] = red[0] / static_cast<double>(n);
}

// V (bf16, strided) -> packed f16 [hkv, n, d] (exact for the f16 normal
// range).  |v| > 65504 (or a non-finite v) does not fit f16: such values are
// counted into *overflow when it is given (the host entry reports them).
__global__ void k_v_to_f16(int64_t n, int64_t hkv, int64_t rs, int64_t hs,
                           const __nv_bfloat16* __restrict__ v, __half* __restrict__ v16,
                           unsigned* __restrict__ overflow) {
    const int64_t total8 = hkv * n * (kD / 8);
    bool bad = false;
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
        for (int u = 0; u < 4; ++u) {
            const float2 x = __bfloat1622float2(b2[u]);
            bad |= !(fabsf(x.x) <= 65504.f) || !(fabsf(x.y) <= 65504.f);
            o2[u] = __float22half2_rn(x);
        }
        *reinterpret_cast<uint4*>(v16 + (hh * n + i) * kD + c8 * 8) = o;
    }
    if (overflow != nullptr && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
        atomicAdd(overflow, 1u);
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

// 3-D map {d, rows, heads} of f32, box {32, 128, 1} (128 B rows), 128B swizzle.
cudaError_t make_map_3d_f32(CUtensorMap* m, const void* base, int64_t rows, int64_t heads) {
    EncodeTiled enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(kD), static_cast<cuuint64_t>(rows),
                                static_cast<cuuint64_t>(heads)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(kD * 4), static_cast<cuuint64_t>(rows * kD * 4)};
    const cuuint32_t box[3] = {32, 128, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
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

// Dynamic shared-memory limit of a kernel, set once per device (a process
// may drive several GPUs; the attribute is per device context).
template <class F>
cudaError_t smem_attr_once(F* fn, int bytes, unsigned long long* done_mask) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (__atomic_load_n(done_mask, __ATOMIC_ACQUIRE) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) __atomic_fetch_or(done_mask, bit, __ATOMIC_RELEASE);
    return e;
}

constexpr size_t kSmemBytes = sizeof(PairSmem) + 1024;
static_assert(kSmemBytes <= 232448, "fa_pair shared memory exceeds 227 KB");

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
    if (MODE == SPARSE && P.acc_f16 && !P.out_bf16) {
        // K3's merge epilogue moves by TMA: the tile maps of K and V (unused
        // by the gathering K3) describe K1's f16 acc / l [hq, n, d] (load) and
        // the f32 output [hq, n, d] (store)
        if ((e = make_map_3d(&tk, P.acc_in, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, n, f.hq, kD, n * kD))) return e;
        if ((e = make_map_3d_f32(&tv, P.out, n, f.hq))) return e;
    }
    if (MODE == ANCHOR && P.acc_f16) {
        // K1's f16 acc / l leaves by TMA store: the 5th map (the V gather map
        // of K3, unused here) describes acc_out [hq, n, d] f16
        if ((e = make_map_3d(&tvg, P.acc_out, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, n, f.hq, kD, n * kD)))
            return e;
    } else if ((e = make_map_gather(&tvg, v16, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, f.hkv * n))) {
        return e;
    }
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
    P.T_n = static_cast<int>((n + kB - 1) / kB);
    static unsigned long long attr_done = 0;  // per MODE instantiation, bit per device
    if ((e = smem_attr_once(fa_pair<MODE>, static_cast<int>(kSmemBytes), &attr_done))) return e;
    const int ipg = (P.step + 1) / 2;
    P.g_end = static_cast<int>(f.g1);
    P.n_groups = static_cast<int>(f.g1 - f.g0);
    const unsigned grid = static_cast<unsigned>((f.g1 - f.g0) * ipg * f.hq);
    P.cluster = 1;
    // K3: cluster the pairs of one (head, group) so each gathered tile is
    // fetched once per cluster (TMA multicast); needs the pairs of a group to
    // fill whole clusters (pairs past the end of a partial last group run as
    // gather-only members, see fa_pair).
    // Measured with split K / V gather warps (128k Llama): clusters of 2 /
    // 4 -> K3 16.3-16.4 / 17.1-17.3 ms (4-CTA clusters co-schedule on only
    // 132 of 148 SMs); AA_K3_CLUSTER overrides.
    if (MODE == SPARSE) {
        int want = 2;
        if (const char* env = getenv("AA_K3_CLUSTER")) want = atoi(env);
        for (int c : {want, 2, 1})
            if (c >= 1 && c <= 8 && ipg % c == 0) {
                P.cluster = c;
                break;
            }
    }
    if (P.cluster == 1) {
        fa_pair<MODE><<<grid, kThreadsOf<MODE>, kSmemBytes, s>>>(tq, tk, tv, tkg, tvg, P);
        return cudaGetLastError();
    }
    auto launch_cluster = [&](const FaParams& PP, unsigned g, cudaStream_t st) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(g);
        cfg.blockDim = dim3(kThreadsOf<MODE>);
        cfg.dynamicSmemBytes = kSmemBytes;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(PP.cluster);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, fa_pair<MODE>, tq, tk, tv, tkg, tvg, PP);
    };
    return launch_cluster(P, grid, s);
}

cudaError_t convert_v(const FastArgs& f, const void* v, void* v16, cudaStream_t s,
                      unsigned* overflow) {
    const int64_t total8 = f.hkv * f.geo.n * (kD / 8);
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total8 + 255) / 256, 148 * 16));
    k_v_to_f16<<<blocks, 256, 0, s>>>(f.geo.n, f.hkv, f.kv_rs, f.kv_hs,
                                      static_cast<const __nv_bfloat16*>(v),
                                      static_cast<__half*>(v16), overflow);
    return cudaGetLastError();
}

}  // namespace

cudaError_t fast_convert_v(const FastArgs& f, const void* v, void* v16, cudaStream_t s,
                           unsigned* overflow) {
    return convert_v(f, v, v16, s, overflow);
}

cudaError_t fast_anchor(const FastArgs& f, const void* q, const void* k, const void* v16, float* m,
                        float* l, float* acc, float* qsum, double* msum, cudaStream_t s, bool acc_f16) {
    FaParams P{};
    P.acc_f16 = acc_f16 ? 1 : 0;
    P.m_out = m;
    P.l_out = l;
    P.acc_out = acc;
    P.qsum = qsum;
    P.msum = msum;
    return launch_fa<ANCHOR>(f, q, k, v16, P, s);
}

cudaError_t fast_pool(const FastArgs& f, const void* q, const float* m, const float* qsum,
                      const double* msum, double* anchor, float* qbar, cudaStream_t s) {
    k_pool_fast<<<dim3(static_cast<unsigned>(f.g1 - f.g0), static_cast<unsigned>(f.hq)), 128, 0,
                  s>>>(f.geo, f.g0, f.q_rs, f.q_hs, static_cast<const __nv_bfloat16*>(q), m, qsum, msum,
                       anchor, qbar);
    return cudaGetLastError();
}

size_t fast_identify_scratch_bytes(const FastArgs& f) {
    const int64_t rows = f.geo.groups() * f.rep;
    const int64_t rows_pad = (rows + kB - 1) / kB * kB;
    return static_cast<size_t>(2 * f.hkv) * rows_pad * kD * 2;
}

cudaError_t fast_identify(const FastArgs& f, const void* k, const float* qbar,
                          const double* anchor, uint32_t* bits, int64_t words_per_row,
                          cudaStream_t s, void* scratch, size_t scratch_bytes) {
    const int64_t G = f.geo.groups();
    const int64_t Gr = f.g1 - f.g0;
    const int64_t max_end = f.geo.middle_end(f.g1 - 1);
    const int64_t span = max_end > f.geo.b_kv ? max_end - f.geo.b_kv : 0;
    const int64_t tiles = (span + kB - 1) / kB;
    if (tiles == 0) return cudaSuccess;
    if (words_per_row % 4) return cudaErrorInvalidValue;  // 16-byte word stores
    const int rows = static_cast<int>(Gr * f.rep);
    const int rows_pad = (rows + kB - 1) / kB * kB;
    void* split = scratch;
    cudaError_t e;
    const size_t split_bytes = static_cast<size_t>(2 * f.hkv) * rows_pad * kD * 2;
    const bool own = scratch == nullptr || scratch_bytes < split_bytes;
    if (own && (e = cudaMallocAsync(&split, split_bytes, s))) return e;
    k_split_qbar<<<dim3(static_cast<unsigned>(rows_pad), static_cast<unsigned>(f.hkv)), kD, 0, s>>>(
        static_cast<int>(G), static_cast<int>(f.g0), static_cast<int>(Gr), static_cast<int>(f.rep), rows_pad,
        qbar, static_cast<__nv_bfloat16*>(split));
    CUtensorMap ta, tk;
    if ((e = make_map_3d(&ta, split, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rows_pad, 2 * f.hkv, kD,
                         static_cast<int64_t>(rows_pad) * kD)) ||
        (e = make_map_3d(&tk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, f.geo.n, f.hkv, f.kv_rs,
                         f.kv_hs))) {
        if (own) cudaFreeAsync(split, s);
        return e;
    }
    constexpr size_t smem = sizeof(IdSmem) + 1024;
    static_assert(smem <= 232448, "k_identify_tc shared memory exceeds 227 KB");
    static unsigned long long attr_done = 0;
    int sms = 0, dev = 0;
    if ((e = smem_attr_once(k_identify_tc, static_cast<int>(smem), &attr_done)) ||
        (e = cudaGetDevice(&dev)) ||
        (e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev))) {
        if (own) cudaFreeAsync(split, s);
        return e;
    }
    IdWork w;
    w.geo = f.geo;
    w.rep = static_cast<int>(f.rep);
    w.n_mt = rows_pad / kB;
    w.n_pairs = (w.n_mt + 1) / 2;
    w.g0 = static_cast<int>(f.g0);
    w.gr = static_cast<int>(Gr);
    const int heads_pairs = static_cast<int>(f.hkv) * w.n_pairs;
    const int nchunks = static_cast<int>((tiles + kIdChunk - 1) / kIdChunk);
    w.J = std::max(1, std::min(nchunks, (sms > 0 ? sms : 148) / std::max(1, heads_pairs)));
    const unsigned grid = static_cast<unsigned>(heads_pairs * w.J);
    stage_mark(6, s);  // K2 kernel alone: events 6 -> 7 (inside stage 3)
    k_identify_tc<<<grid, kIdThreads, smem, s>>>(ta, tk, w, anchor, f.theta, bits, words_per_row);
    stage_mark(7, s);
    e = cudaGetLastError();
    if (own) cudaFreeAsync(split, s);
    return e;
}

cudaError_t fast_sparse(const FastArgs& f, const void* q, const void* k, const void* v16,
                        const float* m, const float* l, const float* acc,
                        const uint32_t* indices, const int32_t* counts, const int64_t* offsets,
                        int64_t cap, bool csr, void* out, aa_dtype out_dtype, cudaStream_t s,
                        bool acc_f16) {
    FaParams P{};
    P.acc_f16 = acc_f16 ? 1 : 0;
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

cudaError_t fast_recall(const FastArgs& f, const void* q, const void* k, const uint32_t* indices,
                        const int32_t* counts, const int64_t* offsets, int64_t cap,
                        double* row_captured, double* recall, cudaStream_t s) {
    const int64_t G = f.geo.groups();
    const int64_t wpr = ((f.geo.n + 31) / 32 + 3) / 4 * 4;
    const size_t bytes = static_cast<size_t>(f.hq * G * wpr) * 4;
    void* bits = nullptr;
    cudaError_t e;
    if ((e = cudaMallocAsync(&bits, bytes, s))) return e;
    if ((e = cudaMemsetAsync(bits, 0, bytes, s))) {
        cudaFreeAsync(bits, s);
        return e;
    }
    k_scatter_bits<<<dim3(static_cast<unsigned>(G), static_cast<unsigned>(f.hq)), 256, 0, s>>>(
        f.geo, indices, counts, offsets, cap, static_cast<uint32_t*>(bits), wpr);
    FaParams P{};
    P.bits = static_cast<const uint32_t*>(bits);
    P.words_per_row = wpr;
    P.row_recall = row_captured;
    // RECALL loads no V: the V maps only need a valid address
    e = launch_fa<RECALL>(f, q, k, k, P, s);
    if (e == cudaSuccess) {
        k_recall_sum<<<static_cast<unsigned>(f.hq), 256, 0, s>>>(f.geo.n, row_captured, recall);
        e = cudaGetLastError();
    }
    cudaFreeAsync(bits, s);
    return e;
}

cudaError_t fast_tile_mass(const FastArgs& f, const void* q, const void* k, float* tile_mass,
                           cudaStream_t s) {
    const int64_t G = f.geo.groups(), n = f.geo.n;
    const int64_t wpr = ((n + 31) / 32 + 3) / 4 * 4;
    const size_t bits_b = static_cast<size_t>(f.hq * G * wpr) * 4;
    const size_t rec_b = static_cast<size_t>(f.hq * n) * 8;
    const size_t st_b = static_cast<size_t>(f.hq * n) * 8;
    char* tmp = nullptr;
    cudaError_t e;
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&tmp), bits_b + rec_b + st_b, s))) return e;
    if ((e = cudaMemsetAsync(tmp, 0, bits_b, s))) {
        cudaFreeAsync(tmp, s);
        return e;
    }
    // pass 1: per-row (max, sum) of the dense causal softmax
    FaParams P{};
    P.bits = reinterpret_cast<const uint32_t*>(tmp);
    P.words_per_row = wpr;
    P.row_recall = reinterpret_cast<double*>(tmp + bits_b);
    P.row_stats = reinterpret_cast<float2*>(tmp + bits_b + rec_b);
    e = launch_fa<RECALL>(f, q, k, k, P, s);
    if (e == cudaSuccess) {
        // pass 2: normalised mass per (query block, key block) tile
        FaParams P2{};
        P2.row_stats = P.row_stats;
        P2.tile_mass = tile_mass;
        e = launch_fa<TILEMASS>(f, q, k, k, P2, s);
    }
    cudaFreeAsync(tmp, s);
    return e;
}

}  // namespace aa

#ifdef AA_PROF
extern "C" int aa_prof_read(unsigned long long* out, int reset) {
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    if (cudaMemcpyFromSymbol(out, aa::g_prof, sizeof(unsigned long long) * 192) != cudaSuccess) return -1;
    if (reset) {
        static const unsigned long long z[192] = {};
        if (cudaMemcpyToSymbol(aa::g_prof, z, sizeof(z)) != cudaSuccess) return -1;
    }
    return 0;
}
#endif
