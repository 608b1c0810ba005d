// Microbenchmark: shared / global atomic throughput on this B200 (design input
// for the K4 voxel fusion).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned mix(unsigned x){x^=x>>16;x*=0x7feb352dU;x^=x>>15;x*=0x846ca68bU;x^=x>>16;return x;}
__global__ void smem_u32(unsigned* out, int iters){
  __shared__ unsigned s[8192];
  for(int i=threadIdx.x;i<8192;i+=blockDim.x) s[i]=0; __syncthreads();
  unsigned h=mix(threadIdx.x+blockIdx.x*977);
  for(int it=0;it<iters;++it){ h=mix(h+it); atomicAdd(&s[h&8191],1u);} __syncthreads();
  if(threadIdx.x==0) out[blockIdx.x]=s[0];
}
__global__ void smem_f32(unsigned* out, int iters){
  __shared__ float s[8192];
  for(int i=threadIdx.x;i<8192;i+=blockDim.x) s[i]=0; __syncthreads();
  unsigned h=mix(threadIdx.x+blockIdx.x*977);
  for(int it=0;it<iters;++it){ h=mix(h+it); atomicAdd(&s[h&8191],1.0f);} __syncthreads();
  if(threadIdx.x==0) out[blockIdx.x]=(unsigned)s[0];
}
__global__ void gmem_red_u32(unsigned* buf, unsigned mask, int iters){
  unsigned h=mix(threadIdx.x+blockIdx.x*977);
  for(int it=0;it<iters;++it){ h=mix(h+it); atomicAdd(&buf[h&mask],1u);}
}
__global__ void gmem_red_v4(float* buf, unsigned mask, int iters){
  unsigned h=mix(threadIdx.x+blockIdx.x*977);
  for(int it=0;it<iters;++it){ h=mix(h+it); float* a=buf+4*(h&mask);
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};"::"l"(a),"f"(1.f),"f"(2.f),"f"(3.f),"f"(4.f):"memory");}
}
__global__ void gmem_cas(unsigned long long* buf, unsigned mask, int iters, unsigned long long* out){
  unsigned h=mix(threadIdx.x+blockIdx.x*977); unsigned long long acc=0;
  for(int it=0;it<iters;++it){ h=mix(h+it); acc+=atomicCAS(&buf[h&mask],0ull,(unsigned long long)h);} if(acc==12345) out[0]=acc;
}
int main(){
  unsigned *o; cudaMalloc(&o, 1<<20);
  void* big; cudaMalloc(&big, (size_t)1<<30); cudaMemset(big,0,(size_t)1<<30);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  int blocks=148*8, threads=256, iters=2000; double n=(double)blocks*threads*iters;
#define T(name, launch) launch; cudaDeviceSynchronize(); cudaEventRecord(a); launch; cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b); printf("%-28s %8.2f Gop/s  %6.3f ms  err=%s\n", name, n/ms/1e6, ms, cudaGetErrorString(cudaGetLastError()));
  T("smem atomicAdd u32", (smem_u32<<<blocks,threads>>>(o,iters)));
  T("smem atomicAdd f32 (CAS)", (smem_f32<<<blocks,threads>>>(o,iters)));
  T("gmem red u32 in 1 MB", (gmem_red_u32<<<blocks,threads>>>((unsigned*)big,(1u<<18)-1,iters)));
  T("gmem red u32 in 1 GB", (gmem_red_u32<<<blocks,threads>>>((unsigned*)big,(1u<<28)-1,iters)));
  T("gmem red v4.f32 in 4 MB", (gmem_red_v4<<<blocks,threads>>>((float*)big,(1u<<18)-1,iters)));
  T("gmem red v4.f32 in 256 MB", (gmem_red_v4<<<blocks,threads>>>((float*)big,(1u<<24)-1,iters)));
  T("gmem CAS u64 in 256 MB", (gmem_cas<<<blocks,threads>>>((unsigned long long*)big,(1u<<25)-1,iters,(unsigned long long*)o)));
  return 0;
}
