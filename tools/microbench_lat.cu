// Latency microbenchmark (development tool): dependent DADD / DFMA chains,
// dependent shared-memory loads, __syncthreads at 256 threads, the double
// warp butterfly sum, SHFL.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void lat(long long* out, double a, int iters) {
  __shared__ int chase[1024];
  __shared__ double red[64];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) chase[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  double x = a, y = a * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x + y;  // dependent DADD
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) y = fma(y, x, 1e-9);  // dependent DFMA
  long long t2 = clock64();
  int p = threadIdx.x & 1023;
  for (int i = 0; i < iters; ++i) p = chase[p];  // dependent LDS
  long long t3 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t4 = clock64();
  double s = x;
  for (int i = 0; i < iters; ++i) s = warp_sum(s) * 1e-3;
  long long t5 = clock64();
  // block reduce pattern: warp sum, smem write, barrier, read 8
  double b = y;
  for (int i = 0; i < iters; ++i) {
    double v = warp_sum(b);
    if ((threadIdx.x & 31) == 0) red[(i & 1) * 32 + (threadIdx.x >> 5)] = v;
    __syncthreads();
    double t = red[(i & 1) * 32];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) t += red[(i & 1) * 32 + k];
    b = t * 1e-3;
  }
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; out[5] = t6 - t5;
    out[6] = (long long)(x + y + p + s + b);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  const int iters = 1000;
  for (int nt : {32, 256, 512}) {
    lat<<<1, nt>>>(d, 1.0, iters);
    lat<<<1, nt>>>(d, 1.0, iters);
    long long h[8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads %d: DADD %.1f  DFMA %.1f  LDS %.1f  BAR %.1f  warp_sum(double) %.1f  block_sum %.1f cycles\n", nt,
           h[0] / (double)iters, h[1] / (double)iters, h[2] / (double)iters, h[3] / (double)iters, h[4] / (double)iters,
           h[5] / (double)iters);
  }
  return 0;
}
