// kd_device.cuh — device helpers shared by the step kernels.
#pragma once

#include <cuda_runtime.h>

#include <atomic>

#include "kd_layout.h"
#include "kd_math.cuh"

namespace kd {

// Opt-in to more than 48 KB of dynamic shared memory for kernel `fn` on the
// current device.  The attribute is per device, so the largest size already
// configured is cached per device (one slot per device ordinal, updated with a
// compare-exchange: safe when host threads drive different GPUs at once).
struct SmemAttrCache {
  static constexpr int kMaxDevices = 64;
  std::atomic<size_t> bytes[kMaxDevices];
  SmemAttrCache() {
    for (auto& b : bytes) b.store(0);
  }
};
inline cudaError_t ensure_smem_attr(const void* fn, size_t smem, SmemAttrCache& cache) {
  if (smem <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const bool cached = dev >= 0 && dev < SmemAttrCache::kMaxDevices;
  if (cached && cache.bytes[dev].load() >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess || !cached) return e;
  size_t cur = cache.bytes[dev].load();
  while (cur < smem && !cache.bytes[dev].compare_exchange_weak(cur, smem)) {
  }
  return cudaSuccess;
}

__device__ __forceinline__ V3 ld3(const double* p) { return V3{p[0], p[1], p[2]}; }
__device__ __forceinline__ Q4 ldq(const double* p) { return Q4{p[0], p[1], p[2], p[3]}; }
__device__ __forceinline__ M3 ldm(const double* p) {
  M3 m;
#pragma unroll
  for (int i = 0; i < 9; ++i) m.m[i] = p[i];
  return m;
}
__device__ __forceinline__ void st3(double* p, V3 v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}
__device__ __forceinline__ void stm(double* p, const M3& m) {
#pragma unroll
  for (int i = 0; i < 9; ++i) p[i] = m.m[i];
}

// Exact warp maximum of non-negative doubles.  With the sign bit cleared,
// IEEE bit patterns of non-negative doubles order like their values, so two
// 32-bit REDUX reductions (high words, then the low words of the lanes that
// hold the maximal high word) give the maximum without a shuffle tree.
__device__ __forceinline__ double warp_max_nonneg(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffull;
  const unsigned hi = (unsigned)(u >> 32), lo = (unsigned)u;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  return __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
}

// Warp exclusive prefix sum; returns the warp total.
__device__ __forceinline__ int warp_exclusive_sum(int v, int lane, int& excl) {
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  excl = incl - v;
  return __shfl_sync(0xffffffffu, incl, 31);
}

// Per-body incidence lists of a world's rows in ascending row order (the
// accumulation order of apply_jacobian_transpose, constraints.cpp:121-129, and
// of MatrixFreeDelassus::apply, delassus.cpp:108-113), built by one warp: a
// counting sort over the incidence codes 2r + side, 32 codes per pass; lanes
// holding the same body in a pass are grouped by __match_any_sync, so every
// body's list comes out in ascending code (= row) order.  rb: 2 body ids per
// row (-1: none).  Writes cptr[0..nb] (cptr[b]..cptr[b+1] = body b's codes in
// clist) except cptr[nb], which the caller sets to the returned total.
__device__ __forceinline__ int warp_incidence_lists(const int32_t* rb, int n, int nb, int32_t* cptr, int32_t* clist,
                                                    int lane) {
  const int ncode = 2 * n;
  for (int b = lane; b <= nb; b += 32) cptr[b] = 0;
  __syncwarp();
  for (int c0 = 0; c0 < ncode; c0 += 32) {  // counts into cptr[b + 1]
    const int code = c0 + lane;
    const int body = code < ncode ? rb[code] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, body);
    if (body >= 0 && lane == __ffs(grp) - 1) cptr[body + 1] += __popc(grp);
    __syncwarp();
  }
  int run = 0;  // exclusive scan over indices 1..nb: cptr[b + 1] = start of body b
  for (int base = 1; base <= nb; base += 32) {
    const int b = base + lane;
    const int cnt = b <= nb ? cptr[b] : 0;
    int excl;
    const int tot = warp_exclusive_sum(cnt, lane, excl);
    __syncwarp();
    if (b <= nb) cptr[b] = run + excl;
    run += tot;
  }
  __syncwarp();
  // cptr[b + 1] is body b's cursor while filling: it ends at the start of body
  // b + 1, which is its final value (cptr[0] = 0)
  for (int c0 = 0; c0 < ncode; c0 += 32) {
    const int code = c0 + lane;
    const int body = code < ncode ? rb[code] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, body);
    if (body >= 0) clist[cptr[body + 1] + __popc(grp & ((1u << lane) - 1))] = code;
    __syncwarp();
    if (body >= 0 && lane == __ffs(grp) - 1) cptr[body + 1] += __popc(grp);
    __syncwarp();
  }
  return run;
}

// max is exactly associative/commutative: any reduction order gives the
// reference's serial lpNorm<Infinity> result bit for bit.
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-order (deterministic) butterfly sum.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 1/sqrt(d) for the positive pivots of the factorizations: the hardware fp64
// estimate (MUFU.RSQ64H, relative error < 1e-6) and one third-order
// correction y (1 + e/2 + 3e^2/8), e = 1 - d y^2 (error O(e^3) < 1e-18, so the
// result is within the final rounding; max 2.4e-16 relative to 1/sqrt(d)
// rounded twice, tmp microbenchmark).  49 cycles of latency on B200 vs 123 for
// a float seed plus two Newton steps and 66 for the generic rsqrt.  Subnormal
// inputs flush to zero (a pivot that small has failed anyway).
__device__ __forceinline__ double fast_rsqrt(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-d * y, y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}

// 1/x and sqrt(x) for the PADMM projection: the hardware fp64 estimate plus
// one third-order correction y (1 + e + e^2), e = 1 - x y (the generic fp64
// division costs ~1.5k cycles of latency on the PADMM critical path,
// measured).  Outside [1e-30, 1e30] the exact operation is used.
__device__ __forceinline__ double fast_rcp(double x) {
  const double ax = fabs(x);
  if (!(ax > 1e-30 && ax < 1e30)) return 1.0 / x;
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}
// y / x from the estimate above plus one residual correction (q + r (y - x q)):
// the correctly rounded quotient except in rare last-bit cases.
__device__ __forceinline__ double fast_div(double y, double x) {
  const double r = fast_rcp(x);
  const double q = y * r;
  return fma(fma(-x, q, y), r, q);
}
__device__ __forceinline__ double fast_sqrt(double x) {
  if (!(x > 1e-30 && x < 1e30)) return x == 0.0 ? x : sqrt(x);  // sqrt(+-0) = +-0 without the slow path
  return x * fast_rsqrt(x);
}

// Projection of one contact triple onto the friction cone of slope mu
// (project_cone, padmm.cpp:19-37): inside -> identity, polar cone -> 0, else
// tau = (w_n + mu |w_t|) / (1 + mu^2), y = (tau, mu tau w_t / |w_t|).
// inv_1pmu2 = 1 / (1 + mu^2) is precomputed per contact.
__device__ __forceinline__ void project_soc(const double w[3], double mu, double inv_1pmu2, double y[3]) {
  const double wn = w[0];
  const double tn = fast_sqrt(w[1] * w[1] + w[2] * w[2]);
  y[0] = w[0];
  y[1] = w[1];
  y[2] = w[2];
  if (tn <= mu * wn) return;
  if (mu * tn <= -wn) {
    y[0] = y[1] = y[2] = 0.0;
    return;
  }
  const double tau = (wn + mu * tn) * inv_1pmu2;
  y[0] = tau;
  if (tn > 0) {
    const double s = mu * tau * fast_rcp(tn);
    y[1] = s * w[1];
    y[2] = s * w[2];
  } else {
    y[1] = y[2] = 0.0;
  }
}

}  // namespace kd
