// Microbenchmark: the fusion kernel's update stream (one red.v4.f32 of a
// voxel's weighted sums + one u32 count per point) at pool sizes around the
// 126 MB L2, for the separate-array and the interleaved 32 B record layouts.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/atomics_probe2.cu -o tools/atomics_probe2
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned mix(unsigned x){x^=x>>16;x*=0x7feb352dU;x^=x>>15;x*=0x846ca68bU;x^=x>>16;return x;}
__device__ __forceinline__ void red4(float* a, float x){
  asm volatile("red.global.add.v4.f32 [%0], {%1,%1,%1,%1};"::"l"(a),"f"(x):"memory");}
// layout 0: v4 only; 1: v4 + separate u32 array; 2: 32 B record {v4, u32 @+16}
template <int L>
__global__ void upd(float* sums, unsigned* cnt, unsigned nvox, int iters){
  unsigned h=mix(threadIdx.x+blockIdx.x*977);
  for(int it=0;it<iters;++it){ h=mix(h+it); unsigned v=h%nvox;
    if(L==2){ float* r=sums+8*(size_t)v; red4(r,1.f); atomicAdd((unsigned*)(r+4),1u);} 
    else { red4(sums+4*(size_t)v,1.f); if(L==1) atomicAdd(cnt+v,1u);} }
}
int main(){
  void* big; cudaMalloc(&big, (size_t)2<<30); cudaMemset(big,0,(size_t)2<<30);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  int blocks=148*8, threads=256, iters=500; double n=(double)blocks*threads*iters;
  float* S=(float*)big; unsigned* C=(unsigned*)((char*)big+((size_t)1<<30));
  for (int mb : {8, 16, 32, 48, 64, 96, 128, 192, 256, 512}) {
    for (int L = 0; L < 3; ++L) {
      const size_t bytes_per_vox = L==0 ? 16 : (L==1 ? 20 : 32);
      unsigned nvox = (unsigned)(((size_t)mb << 20) / bytes_per_vox);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (L==0) upd<0><<<blocks,threads>>>(S,C,nvox,iters);
        if (L==1) upd<1><<<blocks,threads>>>(S,C,nvox,iters);
        if (L==2) upd<2><<<blocks,threads>>>(S,C,nvox,iters);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
      }
      printf("pool %4d MB layout %d (%s): %7.2f G points/s  %.3f ms  %s\n", mb, L,
             L==0?"v4 only     ":(L==1?"v4 + u32 arr":"32B record   "), n/ms/1e6, ms, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
