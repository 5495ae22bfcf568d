#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "sm100.cuh"
using namespace aa::sm100;
template <int N, bool TS>
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tb; __shared__ uint64_t bar;
  int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 * 2; i += blockDim.x) base[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tb, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = tb;
  constexpr uint32_t id = TS ? idesc_f16(0, 0, 1, 128, N) : idesc_f16(1, 1, 0, 128, N);
  if (warp == 0) {
    const uint32_t la = sdesc_sw128_lo((uint32_t)__cvta_generic_to_shared(base), 16);
    const uint32_t lb = sdesc_sw128_lo((uint32_t)__cvta_generic_to_shared(base + 32768), 16);
    constexpr uint64_t hi = sdesc_sw128_hi(1024);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (i & 1) * (N == 256 ? 256 : 128);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
        if (TS) mma_ts_w(tmem + 256 + (i & 1) * 128 * (N == 256 ? 0 : 1), tmem + kk * 8, hi | (lb + kk * 128), id, kk > 0 ? 1u : 0u);
        else mma_ss_w(d, hi | (la + off), hi | (lb + off), id, kk > 0 ? 1u : 0u);
      }
    }
    mma_commit_w(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}
template <int N, bool TS> void run(long long* d, int grid) {
  long long h;
  cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  for (int r = 0; r < 2; ++r) { k<N, TS><<<grid, 128, 140000>>>(d, 2048); cudaDeviceSynchronize(); }
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = h / (2048.0 * 8);
  printf("%s N=%d grid %d: %.1f cycles/MMA -> %.0f FLOP/cycle/SM (%s)\n", TS ? "TS" : "SS", N, grid, per, 2.0 * 128 * N * 16 / per, cudaGetErrorString(cudaGetLastError()));
}
int main(int argc, char** argv) {
  long long* d; cudaMalloc(&d, 64);
  int grid = argc > 1 ? atoi(argv[1]) : 148;
  run<128, false>(d, grid); run<256, false>(d, grid); run<128, true>(d, grid); run<256, true>(d, grid);
}
