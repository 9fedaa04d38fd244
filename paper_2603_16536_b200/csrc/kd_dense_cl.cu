// kd_dense_cl.cu — K2c: the dense PADMM loop of a hand-off world on a CTA
// pair (thread-block cluster of 2), two pairs' CTAs resident per SM.
//
// The fused dense kernel K2 keeps X = L^-1 (~200 KB on DR-Legs) in one CTA's
// shared memory, so one world runs per SM and its PADMM loop is bound by one
// SM's shared-memory pipe and by the latency of its serial phases (the per-unit
// projection, the residual reduction, the barriers), during which the pipe
// idles.  Here K2 only forms X and writes its nonzero tiles to an HBM slab;
// K2c splits the tile rows of X between the two CTAs of a cluster (about
// 100 KB each), so an SM hosts half of two different worlds and one world's
// serial phases overlap the other's solve passes.
//
// Per PADMM iteration (padmm.cpp:87-159), each CTA:
//   pass 1  w_i = sum_j X_ij b_j for its own tile rows i (item partials per
//           tile, summed in ascending j);
//   pass 2  per own tile (i, j), lane = column: X_ij^T w_i, stored in its own
//           and (DSMEM) in the peer CTA's shared memory;
//   one cluster barrier, then every unit's x = sum over the tiles of its
//           column in ascending i (both CTAs hold every partial, so both form
//           the same x bit for bit);
//   units   both CTAs run every cone unit (projection padmm.cpp:10-42, dual
//           update, residuals, Nesterov, the next right-hand side) on
//           identical data, so they reach identical decisions without
//           exchanging anything else; rank 0 writes the outputs.
// The CTA's tiles arrive by one TMA bulk copy (cp.async.bulk, mbarrier
// transaction count) from the slab.
#include <cooperative_groups.h>

#include "kd_device.cuh"

namespace cg = cooperative_groups;

namespace kd {

namespace {

constexpr int CL_NT = 256;
constexpr int CL_NW = CL_NT / 32;
constexpr int CL_LDT = 33;           // off-diagonal tile row stride (doubles), as in K2
constexpr int CL_MAX_ITEMS = 36;     // tiles of X for T <= 8
constexpr int CL_OFF = 32 * CL_LDT;  // slab doubles of an off-diagonal tile
constexpr int CL_DIAG = 528;         // slab doubles of a (packed) diagonal tile

__device__ __forceinline__ int cl_rows(int ti, int n) { return min(32, n - 32 * ti); }
__device__ __forceinline__ int cl_tri(int r) { return (r * (r + 1)) >> 1; }
__device__ __forceinline__ bool cl_tile(unsigned long long m, int ti, int tj) {
  return (m >> (ti * (ti + 1) / 2 + tj)) & 1ull;
}

struct ClTables {
  int n_items[2];                    // tiles per CTA (CTA 0: rows < split)
  int ij[2][CL_MAX_ITEMS];           // i << 4 | j, row-major per CTA
  int off[CL_MAX_ITEMS];             // own tiles: shared-memory offset (doubles)
  int col_n[8];                      // per tile column: tiles in it (both CTAs)
  int col_src[8][8];                 // ascending i: cta << 8 | item index in that CTA's list
  int row_n[8];                      // own tile rows (relative): tiles in it
  int row_items[8][8];               // ascending j: own item index
  int start, len;                    // own tiles in the slab (doubles)
  int pp_off[2];                     // per CTA: offset (doubles) of its PP buffer
  unsigned long long bar;            // bulk-copy completion
  double red[CL_NW];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(CL_NT, 2)
    dense_cl_kernel(BatchView bv, StepParams sp, const int32_t* bin_worlds) {
  extern __shared__ __align__(16) double smem[];
  __shared__ ClTables S;
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int w = bin_worlds[blockIdx.x >> 1];
  WorldStep& ws = bv.wstep[w];
  const DevWorld W = bv.worlds[w];
  // both CTAs of the pair read the same words: identical decisions
  if (ws.backend != BE_DENSE_SN || W.xslab_off < 0 || ws.fail) return;
  const DevSnPlan SP = bv.snplan[W.model];
  const int n = SP.S, T = (n + 31) >> 5, ks = SP.cl_split;
  const unsigned long long xm = ((unsigned long long)(uint32_t)SP.xmask_hi << 32) | (uint32_t)SP.xmask_lo;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int lo = q ? ks : 0, hi = q ? T : ks;
  const int npad = 32 * T;

  // ---- tables (thread 0) and the bulk copy of this CTA's tiles
  if (tid == 0) {
    int cnt[2] = {0, 0}, len[2] = {0, 0};
    for (int i = 0; i < T; ++i)
      for (int j = 0; j <= i; ++j)
        if (cl_tile(xm, i, j)) {
          const int c = i >= ks;
          S.ij[c][cnt[c]++] = (i << 4) | j;
          len[c] += i == j ? CL_DIAG : CL_OFF;
        }
    S.n_items[0] = cnt[0];
    S.n_items[1] = cnt[1];
    int o = 0;
    for (int k = 0; k < cnt[q]; ++k) {
      const int ij = S.ij[q][k];
      S.off[k] = o;
      o += (ij >> 4) == (ij & 15) ? CL_DIAG : CL_OFF;
    }
    for (int j = 0; j < T; ++j) {
      int m = 0;
      for (int c = 0; c < 2; ++c)
        for (int k = 0; k < cnt[c]; ++k)
          if ((S.ij[c][k] & 15) == j) S.col_src[j][m++] = (c << 8) | k;
      S.col_n[j] = m;
    }
    for (int i = lo; i < hi; ++i) {
      int m = 0;
      for (int k = 0; k < cnt[q]; ++k)
        if ((S.ij[q][k] >> 4) == i) S.row_items[i - lo][m++] = k;
      S.row_n[i - lo] = m;
    }
    S.start = q ? len[0] : 0;
    S.len = len[q];
    for (int c = 0; c < 2; ++c) S.pp_off[c] = ((len[c] + 1) & ~1) + 32 * cnt[c];
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const unsigned bytes = 8u * (unsigned)len[q];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&S.bar)), "r"(bytes)
                 : "memory");
    const char* src = reinterpret_cast<const char*>(bv.xslab + W.xslab_off + S.start);
    char* dst = reinterpret_cast<char*>(smem);
    constexpr unsigned CHUNK = 32768;
    for (unsigned o2 = 0; o2 < bytes; o2 += CHUNK) {
      const unsigned sz = min(CHUNK, bytes - o2);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(dst + o2)),
          "l"(src + o2), "r"(sz), "r"(smem_u32(&S.bar))
          : "memory");
    }
  }
  __syncthreads();
  const int n_own = S.n_items[q], n_peer = S.n_items[q ^ 1];
  const double* X = smem;
  double* P = smem + ((S.len + 1) & ~1);  // own tile partials (pass 1, then pass 2), 32 per item
  double* PP = P + 32 * n_own;            // the peer's pass-2 partials, 32 per peer item
  double* b = PP + 32 * n_peer;           // right-hand side (full length, both CTAs)
  double* wv = b + npad;                  // w = X b (own tile rows)
  // the peer's PP buffer (DSMEM) holds this CTA's items, in P's order
  double* PPr = cl.map_shared_rank(smem + S.pp_off[q ^ 1], q ^ 1);

  // ---- unit state (one cone unit per thread, as in K2)
  const int64_t R0 = W.row_off;
  const int n_jd = ws.n_rows - ws.n_limits - 3 * ws.n_contacts;
  const int first_contact = n_jd + ws.n_limits;
  const int n_units = first_contact + ws.n_contacts;
  const bool has_unit = tid < n_units;
  const int row0 = tid < first_contact ? tid : first_contact + 3 * (tid - first_contact);
  const int kind = !has_unit ? ROW_BILATERAL : (tid < n_jd ? ROW_BILATERAL : (tid < first_contact ? ROW_LIMIT : ROW_CONTACT));
  const int nr = !has_unit ? 0 : (kind == ROW_CONTACT ? 3 : 1);
  const double mu = has_unit ? bv.rmu[R0 + row0] : 0.0;
  int pos[3] = {0, 0, 0};
#pragma unroll
  for (int d = 0; d < 3; ++d)
    if (d < nr) pos[d] = bv.sn_r2p[W.snr2p_off + row0 + d];
  const double inv_1pmu2 = 1.0 / (1.0 + mu * mu);
  const double eta = sp.eta, rho = sp.rho;
  const double inv_rho = 1.0 / rho;
  double v[3] = {0, 0, 0}, x[3] = {0, 0, 0}, y[3] = {0, 0, 0}, z[3] = {0, 0, 0}, yh[3], zh[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (d < nr) {
      v[d] = bv.vf[R0 + row0 + d];
      x[d] = bv.x0[R0 + row0 + d];
      z[d] = bv.z0[R0 + row0 + d];
    }
  }
  if (kind == ROW_CONTACT) project_soc(x, mu, inv_1pmu2, y);
  else if (kind == ROW_LIMIT) y[0] = fmax(0.0, x[0]);
  else y[0] = x[0];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    yh[d] = y[d];
    zh[d] = z[d];
  }
  for (int r = tid; r < npad; r += CL_NT) b[r] = wv[r] = 0.0;  // padding and unused positions
  __syncthreads();
  auto write_rhs = [&]() {  // rhs = -(v_f + s - eta x - rho y_hat - z_hat)   (padmm.cpp:116-117)
    const double s0 = kind == ROW_CONTACT ? mu * fast_sqrt(zh[1] * zh[1] + zh[2] * zh[2]) : 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d < nr) b[pos[d]] = -((((v[d] + (d == 0 ? s0 : 0.0)) - eta * x[d]) - rho * yh[d]) - zh[d]);
  };
  write_rhs();
  // the tiles have landed (phase 0 of the bulk-copy barrier), and the peer CTA
  // is running (its shared memory exists) before any DSMEM store
  {
    unsigned ok = 0;
    while (!ok)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(smem_u32(&S.bar))
          : "memory");
  }
  cl.sync();

  double prev = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  double rp = 0.0, dmax = 0.0, rc = 0.0;
  int restarts = 0, it = 1, m = 0;
  bool converged = false;
  const int hcap = bv.hist_cap;
#ifdef KD_PROF_CL
  long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tq = clock64();
  auto ps = [&](int k) {
    const long long t = clock64();
    pacc[k] += t - tq;
    tq = t;
  };
#else
  auto ps = [](int) {};
#endif
  for (it = 1; it <= sp.max_iters; ++it) {
    ps(7);
    __syncthreads();  // b complete
    ps(0);
    // ---- pass 1: item partials of w = X b, lane = row
    for (int k = wid; k < n_own; k += CL_NW) {
      const int ij = S.ij[q][k], i = ij >> 4, j = ij & 15;
      const int ri = cl_rows(i, n), r = lane;
      const double* Xt = X + S.off[k];
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      if (r < ri) {
        if (i == j) {
          const double* drow = Xt + cl_tri(r);
          const double2* bi = reinterpret_cast<const double2*>(b + 32 * i);
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const double2 bb = bi[c / 2];
            if (c <= r) a0 += drow[c] * bb.x;
            if (c + 1 <= r) a1 += drow[c + 1] * bb.y;
          }
        } else {
          const double* row = Xt + r * CL_LDT;
          const double2* bj = reinterpret_cast<const double2*>(b + 32 * j);
#pragma unroll
          for (int c = 0; c < 32; c += 4) {
            const double2 b01 = bj[c / 2], b23 = bj[c / 2 + 1];
            a0 += row[c] * b01.x;
            a1 += row[c + 1] * b01.y;
            a2 += row[c + 2] * b23.x;
            a3 += row[c + 3] * b23.y;
          }
        }
      }
      P[32 * k + lane] = (a0 + a1) + (a2 + a3);
    }
    __syncthreads();
    ps(1);
    // ---- w_i = sum of the row's item partials, ascending j
    for (int t = tid; t < 32 * (hi - lo); t += CL_NT) {
      const int il = t >> 5, r = t & 31;
      const int nk = S.row_n[il];
      double s = nk ? P[32 * S.row_items[il][0] + r] : 0.0;
      for (int mm = 1; mm < nk; ++mm) s += P[32 * S.row_items[il][mm] + r];
      wv[32 * (lo + il) + r] = s;
    }
    __syncthreads();
    ps(2);
    // the peer has read the previous iteration's partials out of its PP
    if (it > 1) cl.barrier_wait();
    ps(3);
    // ---- pass 2: item partials of x = X^T w, lane = column; to P and the peer's PP
    for (int k = wid; k < n_own; k += CL_NW) {
      const int ij = S.ij[q][k], i = ij >> 4, j = ij & 15;
      const int c = lane, rj = cl_rows(j, n);
      const double* Xt = X + S.off[k];
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      if (c < rj) {
        if (i == j) {
          const double2* wj = reinterpret_cast<const double2*>(wv + 32 * j);
#pragma unroll
          for (int r = 0; r < 32; r += 2) {
            const double2 ww = wj[r / 2];
            if (r >= c && r < rj) a0 += Xt[cl_tri(r) + c] * ww.x;
            if (r + 1 >= c && r + 1 < rj) a1 += Xt[cl_tri(r + 1) + c] * ww.y;
          }
        } else {
          const int ri = cl_rows(i, n);
          const double* A = Xt + c;
          const double2* wi = reinterpret_cast<const double2*>(wv + 32 * i);
          if (ri == 32) {
#pragma unroll
            for (int r = 0; r < 32; r += 4) {
              const double2 w01 = wi[r / 2], w23 = wi[r / 2 + 1];
              a0 += A[r * CL_LDT] * w01.x;
              a1 += A[(r + 1) * CL_LDT] * w01.y;
              a2 += A[(r + 2) * CL_LDT] * w23.x;
              a3 += A[(r + 3) * CL_LDT] * w23.y;
            }
          } else {
#pragma unroll
            for (int r = 0; r < 32; r += 4) {
              const double2 w01 = wi[r / 2], w23 = wi[r / 2 + 1];
              if (r < ri) a0 += A[r * CL_LDT] * w01.x;
              if (r + 1 < ri) a1 += A[(r + 1) * CL_LDT] * w01.y;
              if (r + 2 < ri) a2 += A[(r + 2) * CL_LDT] * w23.x;
              if (r + 3 < ri) a3 += A[(r + 3) * CL_LDT] * w23.y;
            }
          }
        }
      }
      const double val = (a0 + a1) + (a2 + a3);
      P[32 * k + lane] = val;
      PPr[32 * k + lane] = val;
    }
    ps(4);
    cl.barrier_arrive();  // release: P and the peer's PP hold every pass-2 partial
    cl.barrier_wait();
    ps(5);
    // ---- x of this thread's unit: its column's tile partials in ascending i
    const double beta = sp.acceleration ? sp.nest_beta[m] : 0.0;
    double yp[3], zp[3], wvv[3], yn[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (d < nr) {
        const int p = pos[d], j = p >> 5, c = p & 31;
        const int nk = S.col_n[j];
        double s = 0.0;
        for (int mm = 0; mm < nk; ++mm) {
          const int src = S.col_src[j][mm];
          const double* buf = (src >> 8) == q ? P : PP;
          const double val = buf[32 * (src & 255) + c];
          s = mm ? s + val : val;
        }
        x[d] = s;
      }
      wvv[d] = x[d] - zh[d] * inv_rho;
      yp[d] = y[d];
      zp[d] = z[d];
    }
    cl.barrier_arrive();  // this CTA is done reading its PP
    if (kind == ROW_CONTACT) project_soc(wvv, mu, inv_1pmu2, yn);
    else {
      yn[0] = kind == ROW_LIMIT ? fmax(0.0, wvv[0]) : wvv[0];
      yn[1] = yn[2] = 0.0;
    }
    double ymax = 0.0, zmax = 0.0;
    rp = dmax = rc = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (d < nr) {
        const double zn = zh[d] - rho * (x[d] - yn[d]);
        rp = fmax(rp, fabs(x[d] - yn[d]));
        dmax = fmax(dmax, fabs(yn[d] - y[d]));
        ymax = fmax(ymax, fabs(yn[d]));
        zmax = fmax(zmax, fabs(zn));
        y[d] = yn[d];
        z[d] = zn;
      }
    }
    if (kind != ROW_BILATERAL) rc = fmin(ymax, zmax);
    // max(r_p, r_d, r_c) (padmm.cpp:128-131), one reduction (rho > 0)
    ps(6);
    double combined;
    {
      double vmax = warp_max_nonneg(fmax(rp, fmax(rho * dmax, rc)));
      if (lane == 0) S.red[wid] = vmax;
      __syncthreads();
      combined = S.red[0];
#pragma unroll
      for (int k = 1; k < CL_NW; ++k) combined = fmax(combined, S.red[k]);
    }
    if (q == 0 && tid == 0 && it <= hcap) bv.hist[(int64_t)w * hcap + it - 1] = combined;
    if (!sp.fixed_mode && combined < sp.eps) {
      converged = true;
      break;
    }
    if (sp.acceleration) {  // nesterov_update (padmm.cpp:58-71)
      const bool restart = sp.restart && combined > prev;
      if (restart) {
        m = 0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          yh[d] = y[d];
          zh[d] = z[d];
        }
        ++restarts;
      } else {
        ++m;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          yh[d] = y[d] + beta * (y[d] - yp[d]);
          zh[d] = z[d] + beta * (z[d] - zp[d]);
        }
      }
    } else {
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        yh[d] = y[d];
        zh[d] = z[d];
      }
    }
    prev = combined;
    write_rhs();  // (S.red is rewritten only after the next iteration's barriers)
  }
  if (it > 1 || converged) cl.barrier_wait();  // pairs the last arrive: no DSMEM traffic remains
  // the last iteration's r_p, r_d, r_c (padmm.cpp:147-157)
  __syncthreads();
  {
    double a = warp_max_nonneg(rp), bb = warp_max_nonneg(dmax), c = warp_max_nonneg(rc);
    __shared__ double red3[3 * CL_NW];
    if (lane == 0) {
      red3[3 * wid] = a;
      red3[3 * wid + 1] = bb;
      red3[3 * wid + 2] = c;
    }
    __syncthreads();
    a = red3[0];
    bb = red3[1];
    c = red3[2];
#pragma unroll
    for (int k = 1; k < CL_NW; ++k) {
      a = fmax(a, red3[3 * k]);
      bb = fmax(bb, red3[3 * k + 1]);
      c = fmax(c, red3[3 * k + 2]);
    }
    rp = a;
    dmax = bb;
    rc = c;
  }
  if (q != 0) return;
#ifdef KD_PROF_CL
  // [0] barrier before pass 1, [1] pass 1, [2] row combine, [3] wait for the
  // peer's release of PP, [4] pass 2, [5] cluster barrier, [6] units,
  // [7] reduction + Nesterov + rhs
  if (tid == 0)
    for (int k = 0; k < 8; ++k) ws.phase_cycles[k] = pacc[k];
#endif
  const double r_p = rp, r_d = rho * dmax, r_c = rc;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (d < nr) {
      bv.lam[R0 + row0 + d] = y[d];
      bv.zo[R0 + row0 + d] = z[d];
    }
  }
  if (tid == 0) {
    const int done = min(it, sp.max_iters);
    ws.iterations = done;
    ws.r_p = r_p;
    ws.r_d = r_d;
    ws.r_c = r_c;
    ws.restarts = restarts;
    ws.converged = (converged || fmax(r_p, fmax(r_d, r_c)) < sp.eps) ? 1 : 0;
    ws.cr_iterations = 0;
    ws.cr_breakdown = 0;
    for (int i = done; i < hcap; ++i) bv.hist[(int64_t)w * hcap + i] = -1.0;
  }
}

// Shared memory of a K2c CTA for a plan: the larger CTA's tiles, both CTAs'
// partials, b and w (the static tables are separate).
size_t dense_cl_smem_bytes(int own_len, int n_items, int T) {
  return 8 * ((size_t)((own_len + 1) & ~1) + 32 * (size_t)n_items + 2 * 32 * (size_t)T);
}

size_t dense_cl_static_bytes() { return sizeof(ClTables) + 8 * 3 * CL_NW; }

cudaError_t launch_dense_cluster(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count,
                                 size_t smem, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  static SmemAttrCache attr;
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(dense_cl_kernel), smem, attr);
    if (e != cudaSuccess) return e;
  }
  static std::atomic<int> carve{0};
  if (!carve.load()) {
    const cudaError_t e = cudaFuncSetAttribute(dense_cl_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    carve.store(1);
  }
  dense_cl_kernel<<<2 * count, CL_NT, smem, s>>>(bv, sp, worlds);
  return cudaGetLastError();
}

}  // namespace kd
