// Throwaway B200 microbenchmarks that drive the CSRC kernel design:
// streaming read BW (LDG.128 vs cp.async.bulk), fp64 red.global rates
// (coalesced / strided / mixed with streaming), memset BW.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s at %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void k_read(const double4* __restrict__ a, size_t n4, double* out){
  double s=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n4;i+=(size_t)gridDim.x*blockDim.x){
    double4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];":"=d"(v.x),"=d"(v.y),"=d"(v.z),"=d"(v.w):"l"(a+i));
    s+=v.x+v.y+v.z+v.w;}
  if(s==1.2345) out[0]=s;
}
// cp.async.bulk streaming: each CTA loops over chunks of CH bytes with S stages.
template<int CH,int S>
__global__ void k_bulk(const char* __restrict__ a, size_t nbytes, double* out){
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[S];
  size_t nch=nbytes/CH;
  if(threadIdx.x==0){for(int s=0;s<S;s++){uint32_t b=(uint32_t)__cvta_generic_to_shared(&bar[s]); asm volatile("mbarrier.init.shared.b64 [%0], 1;"::"r"(b));}}
  __syncthreads();
  int it=0; double acc=0;
  size_t c0=blockIdx.x;
  // prologue
  if(threadIdx.x==0){for(int s=0;s<S;s++){size_t c=c0+(size_t)s*gridDim.x; if(c<nch){uint32_t b=(uint32_t)__cvta_generic_to_shared(&bar[s]);uint32_t d=(uint32_t)__cvta_generic_to_shared(sm+s*CH);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;"::"r"(b),"r"(CH));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"::"r"(d),"l"(a+c*CH),"r"(CH),"r"(b):"memory");}}}
  for(size_t c=c0;c<nch;c+=gridDim.x,it++){
    int s=it%S; uint32_t ph=(it/S)&1; uint32_t b=(uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}"::"r"(b),"r"(ph));
    const double* v=(const double*)(sm+s*CH);
    for(int i=threadIdx.x;i<CH/8;i+=blockDim.x) acc+=v[i];
    __syncthreads();
    size_t cn=c+(size_t)S*gridDim.x;
    if(threadIdx.x==0 && cn<nch){uint32_t d=(uint32_t)__cvta_generic_to_shared(sm+s*CH);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;"::"r"(b),"r"(CH));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"::"r"(d),"l"(a+cn*CH),"r"(CH),"r"(b):"memory");}
  }
  if(acc==1.2345) out[0]=acc;
}
// reds: each warp handles a run of rows; per "pair" a red to y[row - off_s] (consecutive over lanes)
__global__ void k_red(double* y, size_t nrows, int nslots, const int* offs){
  size_t w=(blockIdx.x*(size_t)blockDim.x+threadIdx.x)/32; int lane=threadIdx.x&31;
  size_t nw=(size_t)gridDim.x*blockDim.x/32;
  for(size_t r0=w*32;r0<nrows;r0+=nw*32){ size_t r=r0+lane; if(r>=nrows) break;
    for(int s=0;s<nslots;s++){ long long t=(long long)r-offs[s]; if(t>=0) atomicAdd(y+t,1.0);} }
}
// reds strided: lane targets spread (stride 33 doubles)
__global__ void k_red_spread(double* y, size_t nrows, int nslots){
  size_t w=(blockIdx.x*(size_t)blockDim.x+threadIdx.x)/32; int lane=threadIdx.x&31;
  size_t nw=(size_t)gridDim.x*blockDim.x/32;
  for(size_t r0=w*32;r0<nrows;r0+=nw*32){
    for(int s=0;s<nslots;s++){ size_t t=((r0+ (size_t)lane*1031 + s*7919)*2654435761ull)%nrows; atomicAdd(y+t,1.0);} }
}
// stream + red mix: read 20B per "pair" (ja int + al,au double) with LDG, red into y[ja]
__global__ void k_mix(const int* __restrict__ ja, const double* __restrict__ al, const double* __restrict__ au, size_t k, double* y){
  for(size_t t=blockIdx.x*(size_t)blockDim.x+threadIdx.x;t<k;t+=(size_t)gridDim.x*blockDim.x){
    int j=__ldg(ja+t); double v=__ldg(al+t)+__ldg(au+t); atomicAdd(y+j,v);} }
__global__ void k_stream3(const int* __restrict__ ja, const double* __restrict__ al, const double* __restrict__ au, size_t k, double* y){
  double s=0; for(size_t t=blockIdx.x*(size_t)blockDim.x+threadIdx.x;t<k;t+=(size_t)gridDim.x*blockDim.x){
    int j=__ldg(ja+t); s+=__ldg(al+t)*__ldg(au+t)+j;} if(s==1.2345) y[0]=s; }
__global__ void k_smem_atomic(double* out, int iters){
  __shared__ double w[4096]; for(int i=threadIdx.x;i<4096;i+=blockDim.x) w[i]=0; __syncthreads();
  for(int i=0;i<iters;i++){ atomicAdd(&w[(threadIdx.x*13+i*97)&4095],1.0);} __syncthreads(); if(threadIdx.x==0) out[blockIdx.x]=w[0];
}
__global__ void k_smem_plain(double* out, int iters){
  __shared__ double w[4096]; for(int i=threadIdx.x;i<4096;i+=blockDim.x) w[i]=0; __syncthreads();
  for(int i=0;i<iters;i++){ int a=(threadIdx.x+i*97)&4095; w[a]+=1.0; __syncwarp();} __syncthreads(); if(threadIdx.x==0) out[blockIdx.x]=w[0];
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms,cudaDevAttrMultiProcessorCount,0);
  int l2; cudaDeviceGetAttribute(&l2,cudaDevAttrL2CacheSize,0);
  printf("SMs %d L2 %d\n",sms,l2);
  size_t NB=4ull<<30; char* a; CK(cudaMalloc(&a,NB)); CK(cudaMemset(a,0,NB));
  double* out; CK(cudaMalloc(&out,1<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  auto T=[&](const char* name, double bytes, double ops, auto f){ f(); cudaDeviceSynchronize(); cudaEventRecord(e0); for(int i=0;i<5;i++) f(); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); ms/=5;
    cudaError_t er=cudaGetLastError(); printf("%-40s %9.3f ms  %8.1f GB/s  %8.2f Gop/s %s\n",name,ms,bytes/ms/1e6,ops/ms/1e6, er?cudaGetErrorString(er):""); };
  for(int bpsm: {4,8,16}) { char nm[64]; snprintf(nm,64,"read ldg.v4 4GB bpsm=%d",bpsm);
    T(nm,NB,0,[&]{k_read<<<sms*bpsm,256>>>((const double4*)a,NB/32,out);}); }
  { auto kf=k_bulk<16384,4>; cudaFuncSetAttribute(kf,cudaFuncAttributeMaxDynamicSharedMemorySize,65536);
    for(int bpsm: {1,2,3}){ char nm[64]; snprintf(nm,64,"bulk 16K x4 bpsm=%d",bpsm); T(nm,NB,0,[&]{kf<<<sms*bpsm,128,65536>>>(a,NB,out);}); } }
  { auto kf=k_bulk<32768,6>; cudaFuncSetAttribute(kf,cudaFuncAttributeMaxDynamicSharedMemorySize,6*32768);
    T("bulk 32K x6 bpsm=1",NB,0,[&]{kf<<<sms,256,6*32768>>>(a,NB,out);}); }
  // memset 134MB
  T("memset 134MB",134217728.0,0,[&]{cudaMemsetAsync(a,0,134217728);});
  T("memset 1GB",1073741824.0,0,[&]{cudaMemsetAsync(a,0,1073741824);});
  // reds
  size_t nrows=16777216; double* y=(double*)a; int h_off[13]={1,255,256,257,65279,65280,65281,65535,65536,65537,65791,65792,65793}; int* offs; CK(cudaMalloc(&offs,64)); cudaMemcpy(offs,h_off,52,cudaMemcpyHostToDevice);
  for(int ns: {1,4,13}) { char nm[64]; snprintf(nm,64,"red coalesced stencil slots=%d",ns); T(nm,0,(double)nrows*ns,[&]{k_red<<<sms*8,256>>>(y,nrows,ns,offs+ (ns==1?0:0));}); }
  T("red spread 13",0,(double)nrows*13,[&]{k_red_spread<<<sms*8,256>>>(y,nrows,13);});
  // mix: k = 216M pairs
  size_t k=216338940; char* b2; CK(cudaMalloc(&b2,(size_t)5<<30)); int* ja=(int*)b2; double* al=(double*)(b2+((size_t)900<<20)); double* au=(double*)(b2+((size_t)2700<<20)); cudaMemset(b2,0,(size_t)5<<30);
  // ja = t/13 - off pattern: make targets local: fill ja with (t/13) via kernel-less memset: use zeros → worst-case same-address contention; instead fill pattern on host chunkwise
  { int* h=(int*)malloc(k*4); for(size_t t=0;t<k;t++){ size_t r=t/13+65800; h[t]=(int)(r-h_off[t%13]); } cudaMemcpy(ja,h,k*4,cudaMemcpyHostToDevice); free(h);} 
    T("stream3 20B/pair no red",20.0*k,(double)k,[&]{k_stream3<<<sms*8,256>>>(ja,al,au,k,y);});
  T("mix 20B/pair + red y[ja]",20.0*k,(double)k,[&]{k_mix<<<sms*8,256>>>(ja,al,au,k,y);});
  T("smem fp64 atomic (CAS) 1M/blk",0,(double)sms*2*256*4096,[&]{k_smem_atomic<<<sms*2,256>>>(out,4096);});
  T("smem fp64 plain rmw 1M/blk",0,(double)sms*2*256*4096,[&]{k_smem_plain<<<sms*2,256>>>(out,4096);});
  printf("done\n"); return 0;
}
