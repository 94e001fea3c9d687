#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
// MODE 0: local shared f64 atomicAdd; 1: partner CTA's shared (DSMEM); 2: R of 8 remote
template<int MODE, int R>
__global__ void __cluster_dims__(2,1,1) dsk(double* out, int iters, int nb){
  extern __shared__ double sh[];
  cg::cluster_group cl = cg::this_cluster();
  for(int i=threadIdx.x;i<nb;i+=blockDim.x) sh[i]=0;
  cl.sync();
  double* rem = cl.map_shared_rank(sh, (int)(cl.block_rank()^1));
  unsigned x=threadIdx.x*2654435761u+blockIdx.x*97u+1;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int u=0;u<8;u++){
      x=x*1664525u+1013904223u; unsigned b=(x>>8)%nb;
      if(MODE==0) atomicAdd(&sh[b],1.0);
      else if(MODE==1) atomicAdd(&rem[b],1.0);
      else { if(u<R) atomicAdd(&rem[b],1.0); else atomicAdd(&sh[b],1.0); }
    }
  }
  cl.sync();
  double s=0; for(int i=threadIdx.x;i<nb;i+=blockDim.x) s+=sh[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
template<int M,int R> int run(double* out,int SM,int clk,const char* nm){
  cudaFuncSetAttribute(dsk<M,R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int it=100;
  dsk<M,R><<<SM,768,8192*8>>>(out,10,8192); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0); dsk<M,R><<<SM,768,8192*8>>>(out,it,8192); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1); double ops=(double)SM*768*it*8;
  printf("%-32s %8.3f ms %8.1f Gop/s %6.2f op/clk/SM\n",nm,ms,ops/ms/1e6,ops/(ms*1e-3)/SM/(clk*1e3));
  return 0;
}
int main(){
  cudaDeviceProp p; cudaGetDeviceProperties(&p,0); int clk; cudaDeviceGetAttribute(&clk,cudaDevAttrClockRate,0);
  int SM=p.multiProcessorCount; double* out; CK(cudaMalloc(&out,sizeof(double)*SM*768));
  for(int r=0;r<2;r++){
  run<0,0>(out,SM,clk,"local CAS f64");
  run<1,0>(out,SM,clk,"remote (DSMEM) f64");
  run<2,1>(out,SM,clk,"1/8 remote");
  run<2,2>(out,SM,clk,"2/8 remote");
  run<2,4>(out,SM,clk,"4/8 remote");
  }
  return 0;
}
