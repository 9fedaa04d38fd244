// FP64 throughput microbenchmark (development tool): scalar DFMA vs DMMA
// (mma.sync.aligned.m8n8k4.f64) on one SM, 12 warps.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dfma(double* out, long long* cyc, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_dmma(double* out, long long* cyc, int iters) {
  double d[8][2];
  for (int k = 0; k < 8; ++k) d[k][0] = d[k][1] = 0.0;
  const double a = 1e-3 * threadIdx.x, b = 2e-3;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(d[k][0], d[k][1], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  double s = 0;
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  out[threadIdx.x] = s;
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 1 << 16);
  cudaMalloc(&c, 64);
  const int iters = 4096;
  for (int nw : {1, 4, 12, 32}) {
    k_dfma<<<1, 32 * nw>>>(o, c, iters);
    k_dmma<<<1, 32 * nw>>>(o, c, iters);
    long long h[2];
    cudaDeviceSynchronize();
    cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    const double fma_dfma = 32.0 * nw * 8 * iters, fma_dmma = 256.0 * nw * 8 * iters;
    printf("warps=%2d  DFMA: %.1f FMA/clk/SM   DMMA: %.1f FMA/clk/SM\n", nw, fma_dfma / h[0], fma_dmma / h[1]);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
