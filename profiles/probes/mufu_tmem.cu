#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x){float y; asm volatile("ex2.approx.ftz.f32 %0, %1;":"=f"(y):"f"(x)); return y;}
__global__ void k_mufu(float* out, long long* clk, int iters) {
  float a[8]; for (int i=0;i<8;++i) a[i] = -0.001f*(threadIdx.x+i);
  __syncthreads();
  long long t0 = clock64();
  for (int it=0; it<iters; ++it) {
    #pragma unroll
    for (int i=0;i<8;++i) a[i] = ex2(a[i]) - 1.0f;
  }
  long long t1 = clock64();
  float s=0; for (int i=0;i<8;++i) s+=a[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
  if (threadIdx.x==0) clk[blockIdx.x]=t1-t0;
}
__global__ void k_tmem(float* out, long long* clk, int iters) {
  __shared__ uint32_t base;
  int warp = threadIdx.x/32;
  if (warp==0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"::"r"((uint32_t)__cvta_generic_to_shared(&base))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t t = base + ((uint32_t)((warp%4)*32) << 16) + (warp/4)*128;
  float acc=0;
  long long t0 = clock64();
  for (int it=0; it<iters; ++it) {
    uint32_t r[128];
    #pragma unroll
    for (int c=0;c<4;++c)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[c*32+0]),"=r"(r[c*32+1]),"=r"(r[c*32+2]),"=r"(r[c*32+3]),"=r"(r[c*32+4]),"=r"(r[c*32+5]),"=r"(r[c*32+6]),"=r"(r[c*32+7]),"=r"(r[c*32+8]),"=r"(r[c*32+9]),"=r"(r[c*32+10]),"=r"(r[c*32+11]),"=r"(r[c*32+12]),"=r"(r[c*32+13]),"=r"(r[c*32+14]),"=r"(r[c*32+15]),"=r"(r[c*32+16]),"=r"(r[c*32+17]),"=r"(r[c*32+18]),"=r"(r[c*32+19]),"=r"(r[c*32+20]),"=r"(r[c*32+21]),"=r"(r[c*32+22]),"=r"(r[c*32+23]),"=r"(r[c*32+24]),"=r"(r[c*32+25]),"=r"(r[c*32+26]),"=r"(r[c*32+27]),"=r"(r[c*32+28]),"=r"(r[c*32+29]),"=r"(r[c*32+30]),"=r"(r[c*32+31]) : "r"(t + c*32));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    #pragma unroll
    for (int i=0;i<128;++i) acc += __uint_as_float(r[i]);
  }
  long long t1 = clock64();
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc;
  if (threadIdx.x%32==0) clk[blockIdx.x*32 + warp]=t1-t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp==0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;"::"r"(base));
}
int main(){
  float* o; long long* c; cudaMalloc(&o, 1<<24); cudaMalloc(&c, 1<<20);
  long long h[1024];
  int iters=4096;
  for (int nw : {1,4,8,16}) {
    k_mufu<<<1, nw*32>>>(o,c,iters); cudaDeviceSynchronize();
    k_mufu<<<1, nw*32>>>(o,c,iters); cudaDeviceSynchronize();
    cudaMemcpy(h,c,8,cudaMemcpyDeviceToHost);
    double per = (double)h[0]/(iters*8.0);
    printf("MUFU.EX2: %2d warps: %.2f clk per warp-instr per warp -> %.2f ex2/clk/SM\n", nw, per, nw*32/per);
  }
  for (int nw : {1,4,8}) {
    k_tmem<<<1, nw*32>>>(o,c,1024); cudaDeviceSynchronize();
    k_tmem<<<1, nw*32>>>(o,c,1024); cudaDeviceSynchronize();
    cudaMemcpy(h,c,8*32,cudaMemcpyDeviceToHost);
    double per = (double)h[0]/1024;
    printf("LDTM 4x32x32b (16KB/warp) + wait + 128 FADD: %d warps: %.0f clk per iter (warp0) -> %.1f B/clk/SM\n", nw, per, nw*16384/per);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
