// Microbenchmark of the dense-path primitives (development tool): times each
// device primitive of kd_dense.cu in isolation with clock64 on one SM.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2603_16536_b200/csrc/kd_dense.cu"

using namespace kd;

__global__ void bench(double* g, long long* out) {
  extern __shared__ double sm[];
  __shared__ int fail;
  __shared__ double rinv_s[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // SPD 32x32 packed diag tile: I*40 + small
  for (int e = tid; e < 528 * 8; e += blockDim.x) sm[e] = 0.001 * ((e * 7919) % 13);
  __syncthreads();
  if (tid < 32)
    for (int r = 0; r < 32; ++r) sm[tri(r) + r] = 40.0;
  __syncthreads();
  long long t0 = clock64();
  if (wid == 0) diag_factor_invert(sm, 32, lane, &fail, rinv_s);
  __syncthreads();
  long long t1 = clock64();
  // panel rows: 32 rows of an off-diag tile at sm+600 using Linv at sm
  if (wid == 0) panel_tile(sm, 1, 0, 96);
  __syncthreads();
  long long t2 = clock64();
  if (wid == 0) syrk_tile(sm, 1, 1, 0, 96, lane);  // uses tiles of an n=96 layout
  __syncthreads();
  long long t3 = clock64();
  // 12 warps each one syrk tile concurrently (same tile reads; different targets ok for timing)
  syrk_tile(sm, 2, 1, 0, 96, lane);
  __syncthreads();
  long long t4 = clock64();
  if (tid == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    out[2] = t3 - t2;
    out[3] = t4 - t3;
  }
  if (tid == 0) g[0] = sm[5] + fail;
}

template <int NT>
__global__ void bench_solve(double* g, long long* out, int n) {
  extern __shared__ double sm[];
  const int T = (n + 31) / 32;
  const int nlen = n * (n + 1) / 2;
  double* L = sm;
  double* b = sm + ((nlen + 1) & ~1);
  double* w = b + 32 * T;
  for (int e = threadIdx.x; e < nlen; e += NT) L[e] = 1e-3 * ((e * 31) % 7);
  for (int e = threadIdx.x; e < 32 * T; e += NT) b[e] = 1.0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < 10; ++it) inv_solve<NT>(L, b, w, n, T);
  long long t1 = clock64();
  double a = 0, b2 = 0, c = 0;
  double red[64];
  long long t2 = clock64();
  for (int it = 0; it < 10; ++it) {
    a = threadIdx.x * 1.0 + it;
    b2 = a * 0.5;
    c = a * 0.25;
    __shared__ double rs[3 * NT / 32];
    block_max3<NT>(a, b2, c, rs);
    __syncthreads();
  }
  long long t3 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / 10;
    out[1] = (t3 - t2) / 10;
    g[1] = b[3] + a + b2 + c + red[0] * 0;
  }
}

int main() {
  double* g;
  long long* o;
  cudaMalloc(&g, 64);
  cudaMalloc(&o, 64);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(bench_solve<384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 230000);
  for (int rep = 0; rep < 3; ++rep) {
    bench<<<1, 384, 200000>>>(g, o);
    long long h[4];
    cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
    printf("diag_factor_invert %lld  panel(tile, DMMA) %lld  syrk(1 warp) %lld  syrk(12 warps) %lld cycles\n", h[0],
           h[1], h[2], h[3]);
  }
  for (int n : {64, 128, 214, 232}) {
    bench_solve<384><<<1, 384, 230000>>>(g, o, n);
    long long h[2];
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("n=%d inv_solve %lld cycles  block_max3 %lld cycles\n", n, h[0], h[1]);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
