// Microbenchmark: L2 reduction throughput vs the spatial pattern of a warp's
// 32 updates (random voxels / 32 voxels of one 64-voxel block / one voxel),
// for the float4 sums and the u32 counts.  Design input for the fusion kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/atomics_probe3.cu -o tools/atomics_probe3
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned mix(unsigned x){x^=x>>16;x*=0x7feb352dU;x^=x>>15;x*=0x846ca68bU;x^=x>>16;return x;}
__device__ __forceinline__ void red4(float* a, float x){
  asm volatile("red.global.add.v4.f32 [%0], {%1,%1,%1,%1};"::"l"(a),"f"(x):"memory");}
// P: 0 random voxel per lane; 1 lanes -> 32 random voxels of one random block
// (warp-uniform block); 2 lanes -> lane-th voxel of a warp-uniform block;
// 3 all lanes one voxel.  OP: 0 v4 only, 1 u32 count only, 2 both
template <int P, int OP>
__global__ void upd(float* sums, unsigned* cnt, unsigned nblk, int iters){
  const int lane = threadIdx.x & 31;
  unsigned h=mix(threadIdx.x+blockIdx.x*977), hw=mix((threadIdx.x>>5)+blockIdx.x*131);
  for(int it=0;it<iters;++it){
    h=mix(h+it); hw=mix(hw+it);
    unsigned vox;
    if (P==0) vox = h % (nblk*64);
    else if (P==1) vox = (hw % nblk)*64 + (h & 63);
    else if (P==2) vox = (hw % nblk)*64 + lane;
    else vox = (hw % nblk)*64;
    if (OP!=1) red4(sums+4*(size_t)vox,1.f);
    if (OP!=0) atomicAdd(cnt+vox,1u);
  }
}
int main(){
  void* big; cudaMalloc(&big, (size_t)1<<30); cudaMemset(big,0,(size_t)1<<30);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  int blocks=148*8, threads=256, iters=300; double n=(double)blocks*threads*iters;
  float* S=(float*)big; unsigned* C=(unsigned*)((char*)big+((size_t)512<<20));
  const char* pn[4]={"random voxel   ","block, random  ","block, lane-th ","single voxel   "};
  const char* on[3]={"v4 ","u32","v4+u32"};
  for (int mb : {16, 64}) {
    unsigned nblk = (unsigned)(((size_t)mb<<20)/(64*20));
#define RUN(P,OP) for(int rep=0;rep<2;++rep){cudaEventRecord(a); upd<P,OP><<<blocks,threads>>>(S,C,nblk,iters); cudaEventRecord(b); cudaEventSynchronize(b);} cudaEventElapsedTime(&ms,a,b); \
    printf("pool %3d MB  %s %-6s %7.2f G points/s\n", mb, pn[P], on[OP], n/ms/1e6);
    RUN(0,0) RUN(0,1) RUN(0,2) RUN(1,0) RUN(1,1) RUN(1,2) RUN(2,0) RUN(2,1) RUN(2,2) RUN(3,0) RUN(3,1)
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
