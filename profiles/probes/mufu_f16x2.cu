#include <cstdio>
#include <cuda_fp16.h>
__global__ void k_f16x2(float* out, long long* clk, int iters) {
  __half2 a[8]; for (int i=0;i<8;++i) a[i] = __floats2half2_rn(-0.001f*(threadIdx.x+i), -0.002f*i);
  long long t0 = clock64();
  for (int it=0; it<iters; ++it) {
    #pragma unroll
    for (int i=0;i<8;++i) { unsigned r; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(*reinterpret_cast<unsigned*>(&a[i]))); a[i] = __hsub2(*reinterpret_cast<__half2*>(&r), __floats2half2_rn(1.f,1.f)); }
  }
  long long t1 = clock64();
  float s=0; for (int i=0;i<8;++i) s+=__low2float(a[i]);
  out[threadIdx.x]=s; if (threadIdx.x==0) clk[0]=t1-t0;
}
__global__ void k_f32(float* out, long long* clk, int iters) {
  float a[8]; for (int i=0;i<8;++i) a[i] = -0.001f*(threadIdx.x+i);
  long long t0 = clock64();
  for (int it=0; it<iters; ++it) {
    #pragma unroll
    for (int i=0;i<8;++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y - 1.0f; }
  }
  long long t1 = clock64();
  float s=0; for (int i=0;i<8;++i) s+=a[i];
  out[threadIdx.x]=s; if (threadIdx.x==0) clk[0]=t1-t0;
}
int main(){
  float* o; long long* c; cudaMalloc(&o, 1<<20); cudaMalloc(&c, 64); long long h;
  for (int nw : {4, 8, 16}) {
    k_f16x2<<<1, nw*32>>>(o,c,4096); cudaDeviceSynchronize(); k_f16x2<<<1, nw*32>>>(o,c,4096); cudaDeviceSynchronize();
    cudaMemcpy(&h,c,8,cudaMemcpyDeviceToHost); double per=(double)h/(4096*8);
    printf("ex2.f16x2 %2d warps: %.2f clk/instr/warp -> %.1f results/clk/SM\n", nw, per, nw*32*2/per);
    k_f32<<<1, nw*32>>>(o,c,4096); cudaDeviceSynchronize(); k_f32<<<1, nw*32>>>(o,c,4096); cudaDeviceSynchronize();
    cudaMemcpy(&h,c,8,cudaMemcpyDeviceToHost); per=(double)h/(4096*8);
    printf("ex2.f32   %2d warps: %.2f clk/instr/warp -> %.1f results/clk/SM\n", nw, per, nw*32/per);
  }
}
