// Microbenchmarks that decide the fill-kernel design on B200 (sm_100a):
// FP64 pipe rate, conversion rate, IMAD.WIDE rate, shared/global atomic rates.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int OP> __global__ void fp64k(double* out, int iters){
  double a0=threadIdx.x*1e-3, a1=a0+1, a2=a0+2, a3=a0+3, a4=a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  double b=1.0000001, c=1e-9;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int u=0;u<8;u++){
      if(OP==0){ a0=fma(a0,b,c);a1=fma(a1,b,c);a2=fma(a2,b,c);a3=fma(a3,b,c);a4=fma(a4,b,c);a5=fma(a5,b,c);a6=fma(a6,b,c);a7=fma(a7,b,c);} 
      if(OP==1){ a0=__dadd_rn(a0,c);a1=__dadd_rn(a1,c);a2=__dadd_rn(a2,c);a3=__dadd_rn(a3,c);a4=__dadd_rn(a4,c);a5=__dadd_rn(a5,c);a6=__dadd_rn(a6,c);a7=__dadd_rn(a7,c);} 
    }
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3+a4+a5+a6+a7;
}
// conversion: u64 -> f64 -> i32 round trip
__global__ void cvtk(double* out, int iters){
  unsigned long long s[8]; double acc=0;
  for(int u=0;u<8;u++) s[u]=threadIdx.x*977ull+u*1234567ull;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int u=0;u<8;u++){ double d=(double)(s[u]>>11); acc+=d; s[u]+=0x9E3779B97F4A7C15ull; }
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc;
}
// philox-like int: 2x mul.wide + 2 lop3 per round
__global__ void imadk(unsigned* out, int iters){
  unsigned c0=threadIdx.x,c1=1,c2=2,c3=3, d0=threadIdx.x+7,d1=5,d2=6,d3=8;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int r=0;r<10;r++){
      unsigned long long p0=(unsigned long long)c0*0xD2511F53u, p1=(unsigned long long)c2*0xCD9E8D57u;
      unsigned n0=(unsigned)(p1>>32)^c1^(r*0x9E3779B9u); unsigned n1=(unsigned)p1;
      unsigned n2=(unsigned)(p0>>32)^c3^(r*0xBB67AE85u); unsigned n3=(unsigned)p0;
      c0=n0;c1=n1;c2=n2;c3=n3;
      unsigned long long q0=(unsigned long long)d0*0xD2511F53u, q1=(unsigned long long)d2*0xCD9E8D57u;
      unsigned m0=(unsigned)(q1>>32)^d1^(r*0x9E3779B9u); unsigned m1=(unsigned)q1;
      unsigned m2=(unsigned)(q0>>32)^d3^(r*0xBB67AE85u); unsigned m3=(unsigned)q0;
      d0=m0;d1=m1;d2=m2;d3=m3;
    }
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=c0^c1^c2^c3^d0^d1^d2^d3;
}
// shared atomics: random bins among NB; MODE 0 = u32 add, 1 = f64 add (CAS), 2 = f64 plain RMW (not atomic, reference for LSU)
template<int MODE> __global__ void smemk(double* out, int iters, int nb){
  extern __shared__ double sh[];
  unsigned* shu=(unsigned*)sh;
  for(int i=threadIdx.x;i<nb;i+=blockDim.x){sh[i]=0;}
  __syncthreads();
  unsigned x=threadIdx.x*2654435761u+blockIdx.x*97u+1;
  for(int i=0;i<iters;i++){
    #pragma unroll 4
    for(int u=0;u<4;u++){
      x=x*1664525u+1013904223u; unsigned b=(x>>8)%nb;
      if(MODE==0) atomicAdd(&shu[b],1u);
      if(MODE==1) atomicAdd(&sh[b],1.0);
      if(MODE==2) { volatile double* v=sh; v[b]=v[b]+1.0; }
    }
  }
  __syncthreads();
  double s=0; for(int i=threadIdx.x;i<nb;i+=blockDim.x) s+=sh[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// global f64 red: random bins among nb, shared by all CTAs
__global__ void gredk(double* bins, int iters, int nb){
  unsigned x=threadIdx.x*2654435761u+blockIdx.x*97u+1;
  for(int i=0;i<iters;i++){
    #pragma unroll 4
    for(int u=0;u<4;u++){ x=x*1664525u+1013904223u; unsigned b=(x>>8)%nb; atomicAdd(&bins[b],1.0);} 
  }
}
// global f64 red into a per-CTA private slice of nb bins (L2-resident)
__global__ void gredslk(double* bins, int iters, int nb){
  double* mine=bins+(size_t)blockIdx.x*nb;
  unsigned x=threadIdx.x*2654435761u+blockIdx.x*97u+1;
  for(int i=0;i<iters;i++){
    #pragma unroll 4
    for(int u=0;u<4;u++){ x=x*1664525u+1013904223u; unsigned b=(x>>8)%nb; atomicAdd(&mine[b],1.0);}
  }
}
// mixed: of every 8 f64 updates, R go to a per-CTA global slice (REDG), the
// rest to shared memory (CAS.SPIN) -- do the two paths add up?
template<int R> __global__ void mixk(double* gbins, double* out, int iters, int nb){
  extern __shared__ double sh[];
  double* mine=gbins+(size_t)blockIdx.x*nb;
  for(int i=threadIdx.x;i<nb;i+=blockDim.x){sh[i]=0;}
  __syncthreads();
  unsigned x=threadIdx.x*2654435761u+blockIdx.x*97u+1;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int u=0;u<8;u++){
      x=x*1664525u+1013904223u; unsigned b=(x>>8)%nb;
      if(u<R) atomicAdd(&mine[b],1.0); else atomicAdd(&sh[b],1.0);
    }
  }
  __syncthreads();
  double s=0; for(int i=threadIdx.x;i<nb;i+=blockDim.x) s+=sh[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// exp cost
__global__ void expk(double* out, int iters){
  double a=-threadIdx.x*1e-3, s=0;
  for(int i=0;i<iters;i++){
    #pragma unroll 8
    for(int u=0;u<8;u++){ s+=exp(a); a-=1e-7; }
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock(kHz) %d\n", p.name, p.multiProcessorCount, clk);
  int SM=p.multiProcessorCount; int blocks=SM*4, threads=256; 
  double* out; CK(cudaMalloc(&out, sizeof(double)*blocks*threads*4 + (1<<20)));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  auto rep=[&](const char* name, double ops){ cudaEventElapsedTime(&ms,e0,e1); printf("%-34s %8.3f ms  %10.3f Gop/s  %7.2f op/clk/SM(at %d MHz)\n", name, ms, ops/ms/1e6, ops/(ms*1e-3)/SM/(clk*1e3), clk/1000); };
  int it=2000;
  for(int w=0;w<2;w++){
  fp64k<0><<<blocks,threads>>>(out,10); cudaDeviceSynchronize();
  cudaEventRecord(e0); fp64k<0><<<blocks,threads>>>(out,it); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); rep("DFMA", (double)blocks*threads*it*64);
  cudaEventRecord(e0); fp64k<1><<<blocks,threads>>>(out,it); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); rep("DADD", (double)blocks*threads*it*64);
  cudaEventRecord(e0); cvtk<<<blocks,threads>>>(out,it); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); rep("I2F.F64.U64 (+DADD,+IADD64)", (double)blocks*threads*it*8);
  cudaEventRecord(e0); imadk<<<blocks,threads>>>((unsigned*)out,it/10); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); rep("philox round x2 (per round)", (double)blocks*threads*(it/10)*20);
  cudaEventRecord(e0); expk<<<blocks,threads>>>(out,it/8); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); rep("exp(double)", (double)blocks*threads*(it/8)*8);
  int nbs[3]={1024,8192,256};
  for(int q=0;q<3;q++){ int nb=nbs[q]; char nm[64];
    cudaFuncSetAttribute(smemk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    cudaFuncSetAttribute(smemk<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    cudaFuncSetAttribute(smemk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    cudaEventRecord(e0); smemk<0><<<blocks,threads,nb*8>>>(out,it/4,nb); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); sprintf(nm,"ATOMS u32 add nb=%d",nb); rep(nm,(double)blocks*threads*(it/4)*4);
    cudaEventRecord(e0); smemk<1><<<blocks,threads,nb*8>>>(out,it/4,nb); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); sprintf(nm,"ATOMS f64 CAS add nb=%d",nb); rep(nm,(double)blocks*threads*(it/4)*4);
    cudaEventRecord(e0); smemk<2><<<blocks,threads,nb*8>>>(out,it/4,nb); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); sprintf(nm,"LDS+STS f64 RMW nb=%d",nb); rep(nm,(double)blocks*threads*(it/4)*4);
  }
  double* bins; CK(cudaMalloc(&bins, 8*1<<20)); cudaMemset(bins,0,8<<20);
  int gnb[3]={20480, 4096, 1<<20};
  for(int q=0;q<3;q++){ char nm[64]; sprintf(nm,"REDG f64 nb=%d",gnb[q]);
    cudaEventRecord(e0); gredk<<<blocks,threads>>>(bins,it/20,gnb[q]); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); rep(nm,(double)blocks*threads*(it/20)*4);
  }
  double* sl; CK(cudaMalloc(&sl, (size_t)8*SM*8192)); cudaMemset(sl,0,(size_t)8*SM*8192);
  { char nm[64]; sprintf(nm,"REDG f64 per-CTA slice nb=8192");
    cudaEventRecord(e0); gredslk<<<SM,768>>>(sl,it/20,8192); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); rep(nm,(double)SM*768*(it/20)*4);
    cudaFuncSetAttribute(smemk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    cudaEventRecord(e0); smemk<1><<<SM,768,8192*8>>>(out,it/20,8192); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); rep("ATOMS f64 CAS 768thr 1CTA/SM nb=8192",(double)SM*768*(it/20)*4);
    cudaEventRecord(e0); smemk<0><<<SM,768,8192*8>>>(out,it/20,8192); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); rep("ATOMS u32 768thr 1CTA/SM nb=8192",(double)SM*768*(it/20)*4);
#define MIX(R) cudaFuncSetAttribute(mixk<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000); \
    cudaEventRecord(e0); mixk<R><<<SM,768,8192*8>>>(sl,out,it/40,8192); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); \
    sprintf(nm,"mix %d/8 REDG + rest CAS, 768thr",R); rep(nm,(double)SM*768*(it/40)*8);
    MIX(0) MIX(1) MIX(2) MIX(3) MIX(4)
  }
  }
  return 0;
}
