// Microbenchmark probe: launch/graph overhead, barrier latencies, fp64 rate, HBM copy.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s at %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void empty_k(int *p){ if(p && threadIdx.x==1234567) p[0]=1; }

__global__ void block_sync_k(int iters, double *out){
  __shared__ double s[1024];
  double v = threadIdx.x;
  for(int i=0;i<iters;i++){ s[threadIdx.x]=v; __syncthreads(); v += s[(threadIdx.x+1)%blockDim.x]*1e-9; __syncthreads(); }
  if(threadIdx.x==0) out[0]=v;
}

__global__ void block_reduce_k(int iters, double *out){
  __shared__ double s[32];
  double v = threadIdx.x;
  for(int i=0;i<iters;i++){
    double x=v;
    for(int o=16;o>0;o>>=1) x+=__shfl_xor_sync(0xffffffff,x,o);
    if((threadIdx.x&31)==0) s[threadIdx.x>>5]=x;
    __syncthreads();
    double t=0; for(int w=0;w<(int)(blockDim.x>>5);w++) t+=s[w];
    __syncthreads();
    v += t*1e-12;
  }
  if(threadIdx.x==0) out[0]=v;
}

__global__ void cluster_sync_k(int iters, double *out){
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double s[1];
  double v = threadIdx.x;
  for(int i=0;i<iters;i++){
    if(threadIdx.x==0) s[0]=v;
    cl.sync();
    double *r = cl.map_shared_rank(s, (cl.block_rank()+1)%cl.num_blocks());
    v += r[0]*1e-9;
    cl.sync();
  }
  if(threadIdx.x==0 && blockIdx.x==0) out[0]=v;
}

__device__ unsigned int g_bar_count;
__device__ volatile unsigned int g_bar_gen;
__device__ __forceinline__ void grid_barrier(unsigned int nblocks){
  __syncthreads();
  if(threadIdx.x==0){
    unsigned int gen = g_bar_gen;
    __threadfence();
    unsigned int arrived = atomicAdd(&g_bar_count,1);
    if(arrived==nblocks-1){ g_bar_count=0; __threadfence(); g_bar_gen = gen+1; }
    else { while(g_bar_gen==gen){} }
    __threadfence();
  }
  __syncthreads();
}
__global__ void grid_sync_k(int iters, double *out){
  double v=threadIdx.x;
  for(int i=0;i<iters;i++){ grid_barrier(gridDim.x); v+=1e-9; }
  if(threadIdx.x==0 && blockIdx.x==0) out[0]=v;
}
__global__ void cg_grid_sync_k(int iters, double *out){
  cg::grid_group g = cg::this_grid();
  double v=threadIdx.x;
  for(int i=0;i<iters;i++){ g.sync(); v+=1e-9; }
  if(threadIdx.x==0 && blockIdx.x==0) out[0]=v;
}

__global__ void fma_k(int iters, double *out){
  double a=threadIdx.x*1e-3, b=1.0000001, c=1e-7, d=0.5, e=0.25, f=0.125, g=0.3, h=0.7;
  for(int i=0;i<iters;i++){ a=fma(a,b,c); d=fma(d,b,c); e=fma(e,b,c); f=fma(f,b,c); g=fma(g,b,c); h=fma(h,b,c);}
  out[blockIdx.x*blockDim.x+threadIdx.x]=a+d+e+f+g+h;
}

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  for(;i<n;i+=st) b[i]=a[i];
}

int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("name=%s sms=%d cc=%d.%d l2=%d smemOptin=%zu smemPerSM=%zu regsPerSM=%d coop=%d clock=%d memclk=%d busw=%d\n",
    p.name,p.multiProcessorCount,p.major,p.minor,p.l2CacheSize,p.sharedMemPerBlockOptin,p.sharedMemPerMultiprocessor,p.regsPerMultiprocessor,p.cooperativeLaunch,p.clockRate,p.memoryClockRate,p.memoryBusWidth);
  double *out; CK(cudaMalloc(&out, 1<<24));
  cudaStream_t st; CK(cudaStreamCreate(&st));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  // launch overhead
  for(int i=0;i<100;i++) empty_k<<<1,32,0,st>>>(nullptr);
  CK(cudaStreamSynchronize(st));
  cudaEventRecord(e0,st); for(int i=0;i<10000;i++) empty_k<<<1,32,0,st>>>(nullptr); cudaEventRecord(e1,st);
  CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1); printf("stream empty launch: %.3f us/launch\n", ms*1000/10000);
  // graph of 1000 empty kernels
  cudaGraph_t g; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
  for(int i=0;i<1000;i++) empty_k<<<148,128,0,st>>>(nullptr);
  CK(cudaStreamEndCapture(st,&g)); CK(cudaGraphInstantiate(&ge,g,0));
  CK(cudaGraphLaunch(ge,st)); CK(cudaStreamSynchronize(st));
  cudaEventRecord(e0,st); for(int i=0;i<10;i++) cudaGraphLaunch(ge,st); cudaEventRecord(e1,st);
  CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1); printf("graph empty node (148x128): %.3f us/node\n", ms*1000/10000);
  // block sync
  for(int nt: {256,512,1024}){
    block_sync_k<<<1,nt,0,st>>>(10,out); CK(cudaStreamSynchronize(st));
    cudaEventRecord(e0,st); block_sync_k<<<1,nt,0,st>>>(100000,out); cudaEventRecord(e1,st);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1); printf("block %d: syncthreads pair+smem: %.1f ns/iter\n", nt, ms*1e6/100000);
    cudaEventRecord(e0,st); block_reduce_k<<<1,nt,0,st>>>(100000,out); cudaEventRecord(e1,st);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1); printf("block %d: block reduce: %.1f ns/iter\n", nt, ms*1e6/100000);
  }
  // cluster sync
  CK(cudaFuncSetAttribute(cluster_sync_k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for(int cs: {2,4,8,16}){
    cudaLaunchConfig_t cfg{}; cfg.gridDim=dim3(cs); cfg.blockDim=dim3(256); cfg.stream=st;
    cudaLaunchAttribute at[1]; at[0].id=cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x=cs; at[0].val.clusterDim.y=1; at[0].val.clusterDim.z=1;
    cfg.attrs=at; cfg.numAttrs=1;
    int iters=100000;
    cudaError_t err = cudaLaunchKernelEx(&cfg, cluster_sync_k, 10, out);
    if(err!=cudaSuccess){ printf("cluster %d launch err %s\n", cs, cudaGetErrorString(err)); cudaGetLastError(); continue; }
    CK(cudaStreamSynchronize(st));
    cudaEventRecord(e0,st); CK(cudaLaunchKernelEx(&cfg, cluster_sync_k, iters, out)); cudaEventRecord(e1,st);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1); printf("cluster %d: 2x cluster.sync + dsmem: %.1f ns/iter\n", cs, ms*1e6/iters);
  }
  // grid sync (cooperative)
  for(int nb: {16, 148, 296}){
    int iters=20000; void* args[2]={&iters,&out};
    int it0=10; void* args0[2]={&it0,&out};
    CK(cudaLaunchCooperativeKernel((void*)grid_sync_k, dim3(nb), dim3(256), args0, 0, st)); CK(cudaStreamSynchronize(st));
    cudaEventRecord(e0,st); CK(cudaLaunchCooperativeKernel((void*)grid_sync_k, dim3(nb), dim3(256), args, 0, st)); cudaEventRecord(e1,st);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1); printf("grid %d: atomic grid barrier: %.1f ns/iter\n", nb, ms*1e6/iters);
    CK(cudaLaunchCooperativeKernel((void*)cg_grid_sync_k, dim3(nb), dim3(256), args0, 0, st)); CK(cudaStreamSynchronize(st));
    cudaEventRecord(e0,st); CK(cudaLaunchCooperativeKernel((void*)cg_grid_sync_k, dim3(nb), dim3(256), args, 0, st)); cudaEventRecord(e1,st);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1); printf("grid %d: cg grid.sync: %.1f ns/iter\n", nb, ms*1e6/iters);
  }
  // fp64 fma rate
  {
    int iters=20000; int nb=148*8, nt=256;
    fma_k<<<nb,nt,0,st>>>(10,out); CK(cudaStreamSynchronize(st));
    cudaEventRecord(e0,st); fma_k<<<nb,nt,0,st>>>(iters,out); cudaEventRecord(e1,st);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    double fl = 2.0*6*iters*(double)nb*nt; printf("fp64 FMA: %.2f TFLOP/s\n", fl/(ms*1e-3)/1e12);
  }
  // HBM copy
  {
    size_t n = (size_t)1<<27; // 2 GiB per buffer in double2
    double2 *a,*b; CK(cudaMalloc(&a,n*16)); CK(cudaMalloc(&b,n*16)); cudaMemset(a,0,n*16);
    for(int tpb: {256,512}){ for(int bps: {2,4,8}){
      int nb=148*bps*(1024/tpb)/2;
      copy_k<<<nb,tpb,0,st>>>(a,b,n); CK(cudaStreamSynchronize(st));
      cudaEventRecord(e0,st); for(int r=0;r<5;r++) copy_k<<<nb,tpb,0,st>>>(a,b,n); cudaEventRecord(e1,st);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
      printf("copy tpb=%d nb=%d: %.1f GB/s\n", tpb, nb, 5*2.0*n*16/(ms*1e-3)/1e9);
    }}
  }
  printf("done\n");
  return 0;
}
