// Microbenchmark: latency of one cluster-wide fp64 sum for different schemes.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void st_async(uint32_t ra, double v, uint32_t rm) { asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" :: "r"(ra), "d"(v), "r"(rm) : "memory"); }
__device__ __forceinline__ void mbar_init(uint32_t m) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(m) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint32_t m, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(m), "r"(b) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t m, uint32_t p) { asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" :: "r"(m), "r"(p) : "memory"); }
__device__ __forceinline__ double wsum(double v) { for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o); return v; }

template <int MODE>
__global__ void k(int iters, double* out) {
  __shared__ __align__(16) double slots[2][16 * 32];
  __shared__ double wp[32];
  __shared__ __align__(8) unsigned long long mb[2];
  const int K = cg::this_cluster().num_blocks(), rank = cg::this_cluster().block_rank();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) { mbar_init(sa(&mb[0])); mbar_init(sa(&mb[1])); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  cg::this_cluster().sync();
  double v = 1e-3 * threadIdx.x + rank;
  uint32_t ph[2] = {0, 0};
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    double t = wsum(v);
    if (MODE == 0) {          // per-warp push
      if (lane < K) st_async(mapa(sa(&slots[b][rank * nw + wid]), lane), t, mapa(sa(&mb[b]), lane));
      if (threadIdx.x == 0) mbar_expect(sa(&mb[b]), 8u * K * nw);
      mbar_wait(sa(&mb[b]), ph[b]); ph[b] ^= 1;
      double s = 0.0;
      for (int j = lane; j < K * nw; j += 32) s += slots[b][j];
      t = wsum(s);
    } else if (MODE == 1) {   // CTA pre-reduce, per-CTA push
      if (lane == 0) wp[wid] = t;
      __syncthreads();
      if (wid == 0) {
        double u = wsum(lane < nw ? wp[lane] : 0.0);
        if (lane < K) st_async(mapa(sa(&slots[b][rank]), lane), u, mapa(sa(&mb[b]), lane));
      }
      if (threadIdx.x == 0) mbar_expect(sa(&mb[b]), 8u * K);
      mbar_wait(sa(&mb[b]), ph[b]); ph[b] ^= 1;
      t = wsum(lane < K ? slots[b][lane] : 0.0);
    } else {                  // cluster.sync with DSMEM push
      if (lane == 0) wp[wid] = t;
      __syncthreads();
      if (wid == 0) {
        double u = wsum(lane < nw ? wp[lane] : 0.0);
        if (lane < K) cg::this_cluster().map_shared_rank(&slots[b][0], lane)[rank] = u;
      }
      cg::this_cluster().sync();
      t = wsum(lane < K ? slots[b][lane] : 0.0);
    }
    v = v + 1e-20 * t;
  }
  if (threadIdx.x == 0 && rank == 0) out[0] = v;
}

int main() {
  double* o; cudaMalloc(&o, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode)
    for (int K : {1, 2, 4, 8, 16})
      for (int nt : {288, 512}) {
        void (*f)(int, double*) = mode == 0 ? k<0> : (mode == 1 ? k<1> : k<2>);
        cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(K); cfg.blockDim = dim3(nt);
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = K; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        int it = 10; cudaLaunchKernelEx(&cfg, f, it, o); cudaDeviceSynchronize();
        it = 20000;
        cudaEventRecord(a); cudaLaunchKernelEx(&cfg, f, it, o); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("mode %d K %2d threads %d: %.1f ns per reduction (%s)\n", mode, K, nt, ms * 1e6 / it, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
