// Per-warp TMA bulk-copy pipelines: throughput vs copy size, copies per
// chunk and pipeline depth (does TMA request overhead limit small chunks?).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)
__device__ __forceinline__ uint32_t sa(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
// each warp: chunks of `chunk` bytes split into `pieces` copies, depth D stages
__global__ void k(const char* __restrict__ src, size_t nbytes, int chunk, int pieces, int D, double* out){
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bars[32][8];
  int lane=threadIdx.x&31, wib=threadIdx.x>>5, nw=blockDim.x>>5;
  size_t gw=(size_t)blockIdx.x*nw+wib, W=(size_t)gridDim.x*nw;
  char* base=sm+(size_t)wib*D*chunk;
  size_t nch=nbytes/chunk;
  if(lane==0){for(int s=0;s<D;s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;"::"r"(sa(&bars[wib][s])));}
  __syncwarp();
  auto issue=[&](size_t it){ size_t c=gw+it*W; if(c>=nch) return; int s=it%D; uint32_t b=sa(&bars[wib][s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(b),"r"(chunk):"memory");
    int ps=chunk/pieces;
    for(int p=0;p<pieces;p++) asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"::"r"(sa(base+s*chunk+p*ps)),"l"(src+c*chunk+p*ps),"r"(ps),"r"(b):"memory"); };
  if(lane==0) for(int i=0;i<D;i++) issue(i);
  double acc=0;
  for(size_t it=0;;it++){ size_t c=gw+it*W; if(c>=nch) break; int s=it%D; uint32_t b=sa(&bars[wib][s]); uint32_t ph=(it/D)&1;
    asm volatile("{.reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=;}"::"r"(b),"r"(ph):"memory");
    const double* v=(const double*)(base+s*chunk); for(int i=lane;i<chunk/8;i+=32) acc+=v[i];
    __syncwarp(); if(lane==0){ asm volatile("fence.proxy.async.shared::cta;":::"memory"); issue(it+D);} }
  if(acc==1.2345) out[0]=acc;
}
int main(){
  size_t NB=4ull<<30; char* a; CK(cudaMalloc(&a,NB)); CK(cudaMemset(a,1,NB)); double* out; CK(cudaMalloc(&out,64));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms,cudaDevAttrMultiProcessorCount,0);
  cudaFuncSetAttribute(k,cudaFuncAttributeMaxDynamicSharedMemorySize,227*1024);
  int chunks[]={512,1024,2048,4096,8192,16384}; int piecesv[]={1,5}; int Ds[]={2,4};
  for(int chunk:chunks) for(int pieces:piecesv) for(int D:Ds) for(int wpb: {4, 8}) {
    if(chunk/pieces < 16 || (chunk/pieces)%16) continue;
    size_t smem=(size_t)wpb*D*chunk; if(smem>227*1024) continue;
    int nb=0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb,k,wpb*32,smem); if(nb<1) continue;
    int grid=sms*nb;
    k<<<grid,wpb*32,smem>>>(a,NB,chunk,pieces,D,out); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); for(int r=0;r<3;r++) k<<<grid,wpb*32,smem>>>(a,NB,chunk,pieces,D,out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1); ms/=3;
    printf("chunk %6d pieces %d depth %d warps/blk %d blk/sm %d warps/sm %3d : %7.1f GB/s\n",chunk,pieces,D,wpb,nb,nb*wpb,NB/ms/1e6);
  }
  return 0;
}
