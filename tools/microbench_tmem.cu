// TMEM read-bandwidth microbenchmark (development tool): can tensor memory
// serve the PADMM solve's fp64 tile rows faster than shared memory?
// One CTA of 256 threads per SM (8 warps, two per TMEM lane quarter); every
// lane streams 32-double tile rows and folds them into FMAs.
//   mode 0: shared memory, lane r reads row r of a 32 x 33 tile (LDS.64)
//   mode 1: TMEM, tcgen05.ld.32x32b.x16 (8 doubles per lane), a wait per load
//   mode 2: TMEM, two x16 loads per wait
//   mode 3: TMEM, four x16 loads (a whole 32-double row) per wait
//   mode 4: mode 0 and mode 2 interleaved (both data paths at once)
// Measured on a B200: shared memory 122 B/clk/SM, TMEM 256-264 B/clk/SM, and
// the two overlap (mode 4 runs at the shared-memory time).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbt tools/microbench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define LD16(taddr, r)                                                                                        \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),     \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) \
               : "r"(taddr))

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ double dbl(uint32_t lo, uint32_t hi) {
  return __hiloint2double((int)hi, (int)lo);
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) bench(double* out, long long* cyc, int iters) {
  __shared__ double tile[4][32 * 33];
  __shared__ uint32_t tbase;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < 4 * 32 * 33; e += 256) (&tile[0][0])[e] = 1e-3 * (e % 97);
  if (MODE >= 1) {
    if (wid == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  } else {
    __syncthreads();
  }
  const uint32_t tb = MODE >= 1 ? tbase : 0u;
  const uint32_t lanebase = (uint32_t)(32 * (wid & 3)) << 16;
  // each warp of a quarter uses its own 256 columns (4 tiles of 64 columns)
  const uint32_t colbase = (wid >> 2) * 256;
  double v[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = 1.0 + 1e-6 * c;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int t = it & 3;
    if (MODE == 0 || MODE == 4) {
      const double* row = &tile[(wid + t) & 3][lane * 33];
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        a0 += row[c] * v[c];
        a1 += row[c + 1] * v[c + 1];
        a2 += row[c + 2] * v[c + 2];
        a3 += row[c + 3] * v[c + 3];
      }
    }
    if (MODE == 1) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t r[16];
        LD16(tb + lanebase + colbase + 64 * t + 16 * q, r);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          a0 += dbl(r[2 * k], r[2 * k + 1]) * v[8 * q + k];
          a1 += dbl(r[2 * k + 2], r[2 * k + 3]) * v[8 * q + k + 1];
        }
      }
    }
    if (MODE == 2 || MODE == 4) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        uint32_t r[32];
        LD16(tb + lanebase + colbase + 64 * t + 32 * q, r);
        LD16(tb + lanebase + colbase + 64 * t + 32 * q + 16, (r + 16));
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          a2 += dbl(r[2 * k], r[2 * k + 1]) * v[16 * q + k];
          a3 += dbl(r[2 * k + 2], r[2 * k + 3]) * v[16 * q + k + 1];
        }
      }
    }
    if (MODE == 3) {
      uint32_t r[64];
#pragma unroll
      for (int q = 0; q < 4; ++q) LD16(tb + lanebase + colbase + 64 * t + 16 * q, (r + 16 * q));
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        a0 += dbl(r[2 * k], r[2 * k + 1]) * v[k];
        a1 += dbl(r[2 * k + 2], r[2 * k + 3]) * v[k + 1];
      }
    }
  }
  const long long t1 = clock64();
  __syncthreads();
  if (MODE >= 1) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
  }
  out[blockIdx.x * 256 + threadIdx.x] = (a0 + a1) + (a2 + a3);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int M>
void run(const char* name, double* out, long long* cyc, int iters, double bytes_per_iter_per_sm) {
  bench<M><<<148, 256>>>(out, cyc, iters);
  bench<M><<<148, 256>>>(out, cyc, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += h[i] / 148.0;
  printf("%-34s %10.0f cycles  %7.1f B/clk/SM  %6.1f cycles per 8 KB tile per warp\n", name, mean,
         bytes_per_iter_per_sm * iters / mean, mean / iters * 8.0 / (bytes_per_iter_per_sm / 8192.0));
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 256 * 8);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  const double tile_bytes = 8 * 8192.0;  // 8 warps x one 32 x 32 fp64 tile per iteration
  run<0>("smem LDS.64 rows", out, cyc, iters, tile_bytes);
  run<1>("tmem 32x32b.x16, wait per load", out, cyc, iters, tile_bytes);
  run<2>("tmem 2 x x16, wait per pair", out, cyc, iters, tile_bytes);
  run<3>("tmem 4 x x16, one wait", out, cyc, iters, tile_bytes);
  run<4>("smem rows + tmem (both)", out, cyc, iters, 2 * tile_bytes);
  return 0;
}
