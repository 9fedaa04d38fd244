// Block-reduction latency variants at 256 threads (development tool).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int V>
__global__ void red(long long* out, double a, int iters) {
  __shared__ __align__(16) double buf[2][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, NW = blockDim.x >> 5;
  double b = a + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double* bb = buf[i & 1];
    if (V == 0) {  // warp_sum, STS, BAR, 8 serial loads+adds
      double v = warp_sum(b);
      if (lane == 0) bb[wid] = v;
      __syncthreads();
      double t = bb[0];
      for (int k = 1; k < NW; ++k) t += bb[k];
      b = t * 1e-3;
    } else if (V == 1) {  // STS, BAR, LDS only
      if (lane == 0) bb[wid] = b;
      __syncthreads();
      b = bb[(i + 1) & 7] * 1e-3;
    } else if (V == 2) {  // warp_sum, STS, BAR, vector loads + tree
      double v = warp_sum(b);
      if (lane == 0) bb[wid] = v;
      __syncthreads();
      const double2* q = reinterpret_cast<const double2*>(bb);
      double2 q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
      b = (((q0.x + q0.y) + (q1.x + q1.y)) + ((q2.x + q2.y) + (q3.x + q3.y))) * 1e-3;
    } else if (V == 3) {  // warp_sum, STS, BAR, lane-parallel load + warp_sum
      double v = warp_sum(b);
      if (lane == 0) bb[wid] = v;
      __syncthreads();
      b = warp_sum(lane < NW ? bb[lane] : 0.0) * 1e-3;
    } else if (V == 4) {  // warp_sum only
      b = warp_sum(b) * 1e-3;
    } else if (V == 5) {  // BAR only
      __syncthreads();
      b = b * 1.0000001;
    } else if (V == 6) {  // smem warp stage: STS, syncwarp, 16 LDS.128 broadcast + tree; STS, BAR, LDS.128 tree
      __shared__ __align__(16) double wb[2][512];
      double* w = wb[i & 1] + 32 * wid;
      w[lane] = b;
      __syncwarp();
      const double2* q = reinterpret_cast<const double2*>(w);
      double p[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) { const double2 t = q[k]; p[k] = t.x + t.y; }
#pragma unroll
      for (int st = 8; st > 0; st >>= 1)
#pragma unroll
        for (int k = 0; k < st; ++k) p[k] = p[k] + p[k + st];
      if (lane == 0) bb[wid] = p[0];
      __syncthreads();
      const double2* r = reinterpret_cast<const double2*>(bb);
      double2 q0 = r[0], q1 = r[1], q2 = r[2], q3 = r[3];
      b = (((q0.x + q0.y) + (q1.x + q1.y)) + ((q2.x + q2.y) + (q3.x + q3.y))) * 1e-3;
    } else if (V == 7) {  // 2 shuffle levels (xor 1, 2) then smem stage over 8 quads
      __shared__ __align__(16) double wc[2][128];
      double v = b;
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      double* w = wc[i & 1] + 8 * wid;
      if ((lane & 3) == 0) w[lane >> 2] = v;
      __syncwarp();
      const double2* q = reinterpret_cast<const double2*>(w);
      const double2 a0 = q[0], a1 = q[1], a2 = q[2], a3 = q[3];
      const double ws = ((a0.x + a0.y) + (a1.x + a1.y)) + ((a2.x + a2.y) + (a3.x + a3.y));
      if (lane == 0) bb[wid] = ws;
      __syncthreads();
      const double2* r = reinterpret_cast<const double2*>(bb);
      double2 q0 = r[0], q1 = r[1], q2 = r[2], q3 = r[3];
      b = (((q0.x + q0.y) + (q1.x + q1.y)) + ((q2.x + q2.y) + (q3.x + q3.y))) * 1e-3;
    } else if (V == 8) {  // all partials to smem, BAR, each thread reads its quarter... : STS, BAR, 8 LDS.128 of 16-sums
      __shared__ __align__(16) double wd[2][512];
      double* w = wd[i & 1];
      w[threadIdx.x] = b;
      __syncthreads();
      // every thread sums all NT values with 16-wide vector loads (NT=256 -> 128 LDS.128): too many; use 8 lanes x
      const double2* q = reinterpret_cast<const double2*>(w);
      double acc = 0.0;
#pragma unroll 8
      for (int k = 0; k < 128; ++k) { const double2 t = q[k]; acc += t.x + t.y; }
      b = acc * 1e-3;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = (long long)b;
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  const char* names[] = {"warp_sum+STS+BAR+8 serial", "STS+BAR+LDS", "warp_sum+STS+BAR+LDS.128 tree",
                         "warp_sum+STS+BAR+warp_sum", "warp_sum only", "BAR only", "smem warp stage + LDS.128 tree",
                         "2 shfl + smem quads + LDS.128 tree", "all partials, 128 LDS.128"};
  for (int nt : {256, 512}) {
    for (int v = 0; v < 9; ++v) {
      long long h[2];
      for (int rep = 0; rep < 2; ++rep) {
        switch (v) {
          case 0: red<0><<<1, nt>>>(d, 1.0, 1000); break;
          case 1: red<1><<<1, nt>>>(d, 1.0, 1000); break;
          case 2: red<2><<<1, nt>>>(d, 1.0, 1000); break;
          case 3: red<3><<<1, nt>>>(d, 1.0, 1000); break;
          case 4: red<4><<<1, nt>>>(d, 1.0, 1000); break;
          case 5: red<5><<<1, nt>>>(d, 1.0, 1000); break;
          case 6: red<6><<<1, nt>>>(d, 1.0, 1000); break;
          case 7: red<7><<<1, nt>>>(d, 1.0, 1000); break;
          case 8: red<8><<<1, nt>>>(d, 1.0, 1000); break;
        }
      }
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("threads %d  %-32s %.1f cycles\n", nt, names[v], h[0] / 1000.0);
    }
  }
  return 0;
}
