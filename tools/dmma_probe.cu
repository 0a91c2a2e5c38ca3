// DMMA (mma.m8n8k4.f64) latency / throughput probe vs DFMA on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k_mma(double* out, long long* cyc, int n) {
  double d[CH][2];
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-3 + c;
  double a = 1.0000001, b = 0.9999999;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH>
__global__ void k_fma(double* out, long long* cyc, int n) {
  double d[CH];
  for (int c = 0; c < CH; ++c) d[c] = threadIdx.x * 1e-3 + c;
  double a = 1.0000001, b = 0.9999999;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) d[c] = fma(d[c], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += d[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 148 * 1024 * 8 * 4); cudaMalloc(&cyc, 8);
  const int n = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  // latency: 1 warp, 1 chain
  k_mma<1><<<1, 32>>>(out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DMMA dependent latency: %.1f cycles\n", (double)h / n);
  k_fma<1><<<1, 32>>>(out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cycles\n", (double)h / n);
  for (int warps : {4, 8, 16, 32}) {
    k_mma<4><<<148, 32 * warps>>>(out, cyc, n);
    cudaEventRecord(e0); k_mma<4><<<148, 32 * warps>>>(out, cyc, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 4 * n * (double)warps * 148;
    printf("DMMA %2d warps/SM x 4 chains: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
    k_fma<8><<<148, 32 * warps>>>(out, cyc, n);
    cudaEventRecord(e0); k_fma<8><<<148, 32 * warps>>>(out, cyc, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 32 * 8 * n * (double)warps * 148;
    printf("DFMA %2d warps/SM x 8 chains: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  return 0;
}
