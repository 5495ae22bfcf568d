// TMA tile::gather4 issue rate per SM (B200): one warp per CTA issues
// gather4 loads of random 128-B row segments (4 rows x 64 bf16 per op, the
// K3 stripe-gather shape) into a shared-memory ring and waits for each
// stage's bytes; reports cycles per gather4 op per SM, alone and with the
// multicast form in clusters of 2.  K3 issues 64 gather4 per tile pair per
// CTA (K and V, 64 of 128 rows each, 2 column halves), so this rate bounds
// its tile period.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_rate profiles/probes/gather4_rate.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2505_23520_b200/csrc/sm100.cuh"

using namespace aa::sm100;

constexpr int kStages = 4;
constexpr int kOpsPerStage = 32;              // 32 gather4 = 64 rows x 256 B = 16 KB
constexpr uint32_t kStageBytes = kOpsPerStage * 512;
constexpr int kIters = 512;

struct Smem {
    uint8_t ring[kStages][kStageBytes];
    uint64_t full[kStages];
};

template <bool kMc>
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap tm, int nrows, int lanes_used,
                                                int nwarps, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    Smem& S = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = kMc ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&S.full[s], 1);
        fence_mbar_init();
    }
    if (kMc) cluster_sync(); else __syncthreads();
    if (warp < nwarps) {
        uint32_t seed = 12345u + blockIdx.x * 7919u + lane * 104729u;
        long long t0 = 0;
        for (int it = 0; it < kIters; ++it) {
            if (it == 8) t0 = clock64();
            const int st = it % kStages;
            if (it >= kStages) mbar_wait(&S.full[st], ((it / kStages) - 1) & 1);
            if (lane == 0 && warp == 0) mbar_expect_tx(&S.full[st], kMc ? kStageBytes : kStageBytes);
            __syncwarp();
            // each used lane issues ops for its 4-row groups: 32 ops per stage
            // split over lanes_used lanes (in multicast mode each CTA issues
            // half and receives the peer's half)
            const int ops_here = kMc ? kOpsPerStage / 2 : kOpsPerStage;
            // ops split over nwarps warps x lanes_used lanes
            for (int o = warp * lanes_used + lane; lane < lanes_used && o < ops_here; o += nwarps * lanes_used) {
                int r[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    seed = seed * 1664525u + 1013904223u;
                    r[u] = static_cast<int>(seed % static_cast<uint32_t>(nrows));
                }
                const int oo = kMc ? o + static_cast<int>(crank) * ops_here : o;
                uint8_t* dst = S.ring[st] + (oo >> 1) * 512 + (oo & 1) * (kStageBytes / 2) * 0;
                if (kMc)
                    tma_gather4_mc(S.ring[st] + oo * 512, &tm, &S.full[st], 3, (oo & 1) * 64, r[0], r[1], r[2], r[3]);
                else
                    tma_gather4(S.ring[st] + oo * 512, &tm, &S.full[st], (oo & 1) * 64, r[0], r[1], r[2], r[3]);
                (void)dst;
            }
        }
        for (int it = kIters - kStages; it < kIters; ++it) mbar_wait(&S.full[it % kStages], (it / kStages) & 1);
        const long long t1 = clock64();
        if (lane == 0 && warp == 0) {
            out[blockIdx.x * 2] = t1 - t0;
            out[blockIdx.x * 2 + 1] = static_cast<unsigned long long>(kIters - 8) * (kMc ? kOpsPerStage / 2 : kOpsPerStage);
        }
    }
    if (kMc) cluster_sync(); else __syncthreads();
}

int main() {
    // a [rows, 128] bf16 matrix (256 B rows), like K: 8 heads x 131072 rows
    const int rows = 8 * 131072;
    void* g;
    cudaMalloc(&g, static_cast<size_t>(rows) * 256);
    cudaMemset(g, 0, static_cast<size_t>(rows) * 256);
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g, dims, strides, box, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
        printf("tensor map error %d\n", cr);
        return 1;
    }
    const int smem = sizeof(Smem) + 1024;
    cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* out;
    cudaMalloc(&out, 148 * 2 * 8);
    struct C { const char* name; bool mc; int grid; int lanes; int nrows; int warps; };
    const C cases[] = {
        {"1 CTA, 1 warp x 32 lanes, rows over 268 MB", false, 1, 32, rows, 1},
        {"148 CTAs, 1 warp x 32 lanes", false, 148, 32, rows, 1},
        {"148 CTAs, 1 warp x 32 lanes, L2-resident rows", false, 148, 32, rows / 8, 1},
        {"148 CTAs, 2 warps x 16 lanes", false, 148, 16, rows, 2},
        {"148 CTAs, 4 warps x 8 lanes", false, 148, 8, rows, 4},
        {"148 CTAs, 4 warps x 8 lanes, L2-resident rows", false, 148, 8, rows / 8, 4},
        {"clusters of 2, multicast, 1 warp x 16 lanes", true, 148, 16, rows, 1},
        {"clusters of 2, multicast, 2 warps x 8 lanes", true, 148, 8, rows, 2},
        {"clusters of 2, multicast, 4 warps x 4 lanes", true, 148, 4, rows, 4},
    };
    for (const C& c : cases) {
        cudaMemset(out, 0, 148 * 2 * 8);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c.grid);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = c.mc ? 1 : 0;
        cudaError_t e = c.mc ? cudaLaunchKernelEx(&cfg, probe<true>, tm, c.nrows, c.lanes, c.warps, out)
                             : cudaLaunchKernelEx(&cfg, probe<false>, tm, c.nrows, c.lanes, c.warps, out);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s: %s\n", c.name, cudaGetErrorString(e));
            return 1;
        }
        std::vector<unsigned long long> h(148 * 2);
        cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
        double cyc = 0;
        int nb = 0;
        for (int b = 0; b < c.grid; ++b)
            if (h[b * 2 + 1]) {
                cyc += static_cast<double>(h[b * 2]) / h[b * 2 + 1];
                ++nb;
            }
        cyc /= nb;
        printf("%-56s %6.1f cycles per issued gather4 per CTA (%.1f B/clk/SM landed)\n", c.name, cyc,
               (c.mc ? 1024.0 : 512.0) / cyc);
        fflush(stdout);
    }
    return 0;
}
