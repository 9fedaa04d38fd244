// kd_dense.cu — K2: fused per-world dense Delassus path, one CTA per world.
//
// One CTA keeps one world resident on chip for the whole solve:
//   1. assemble_dense (delassus.cpp:67-104): D = P (J M^-1 J^T + R) P + (eta+rho) I
//      from the per-body Gram blocks, summed in ascending body order;
//   2. blocked Cholesky D = L L^T (DenseDelassus::factorize, delassus.cpp:59-63)
//      over 32x32 tiles, right-looking, with each diagonal tile replaced by its
//      inverse so the triangular solves are dependency-light mat-vecs;
//   3. the PADMM loop (padmm_solve, padmm.cpp:87-159): De Saxce shift, the two
//      triangular solves, cone projection (padmm.cpp:10-42), dual update,
//      residual triple with warp-shuffle max-reductions, Nesterov with restart.
//      Each thread owns one cone unit (a bilateral/limit row or a contact
//      triple) and keeps y, z, y_hat, z_hat, v_f in registers across iterations.
//
// Factor storage (n(n+1)/2 doubles, no padding): tile row ti holds ti full
// 32-wide off-diagonal tiles (rows(ti) x 32, XOR-swizzled so row and column
// walks are bank-conflict free for 8-byte words) followed by the diagonal tile
// packed row-major lower.  In GLOBAL_L mode the same layout lives in a per-world
// HBM slab (worlds whose n exceeds the shared-memory capacity, n <= 300).
#include "kd_device.cuh"

namespace kd {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int swz(int r) { return (r & 15) ^ ((r >> 4) << 2); }
__device__ __forceinline__ int tile_rows(int ti, int n) { return min(32, n - 32 * ti); }
__device__ __forceinline__ int tile_row_base(int ti) { return 512 * ti * (ti - 1) + 528 * ti; }
__device__ __forceinline__ int off_tile(int ti, int tj, int n) { return tile_row_base(ti) + tj * 32 * tile_rows(ti, n); }
__device__ __forceinline__ int diag_tile(int ti, int n) { return tile_row_base(ti) + ti * 32 * tile_rows(ti, n); }
__device__ __forceinline__ int tri(int r) { return (r * (r + 1)) >> 1; }
// element (i, j), i >= j
__device__ __forceinline__ int lidx(int i, int j, int n) {
  const int ti = i >> 5, tj = j >> 5, r = i & 31, c = j & 31;
  if (ti == tj) return diag_tile(ti, n) + tri(r) + c;
  return off_tile(ti, tj, n) + r * 32 + (c ^ swz(r));
}

// ---------------------------------------------------------------- reductions
template <int NT>
__device__ __forceinline__ void block_max3(double& a, double& b, double& c, double* red) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  a = warp_max(a);
  b = warp_max(b);
  c = warp_max(c);
  if (lane == 0) {
    red[3 * wid] = a;
    red[3 * wid + 1] = b;
    red[3 * wid + 2] = c;
  }
  __syncthreads();
  a = red[0];
  b = red[1];
  c = red[2];
#pragma unroll
  for (int k = 1; k < NW; ++k) {
    a = fmax(a, red[3 * k]);
    b = fmax(b, red[3 * k + 1]);
    c = fmax(c, red[3 * k + 2]);
  }
}

// ---------------------------------------------------------------- Cholesky pieces
// Factor the packed diagonal tile in place and overwrite it with L_kk^{-1}.
// One warp; lane r owns row r of the tile.  Pivots use one rsqrt each
// (L_cc = d * rsqrt(d), L_rc = a_rc * rsqrt(d)), and the reciprocal of every
// pivot is kept so the inverse needs no divisions.
__device__ void diag_factor_invert(double* T, int rk, int lane, int* fail) {
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = (lane < rk && c <= lane) ? T[tri(lane) + c] : (c == lane ? 1.0 : 0.0);
  bool bad = false;
  double my_rinv = 1.0;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const double dcc = __shfl_sync(FULL, a[c], c);
    if (!(dcc > 0.0)) bad = true;
    const double rinv = rsqrt(dcc);
    const double lc = lane > c ? a[c] * rinv : (lane == c ? dcc * rinv : a[c]);
    if (lane == c) my_rinv = rinv;
    a[c] = lc;
#pragma unroll
    for (int j = 1; j < 32; ++j) {
      if (j > c) {
        const double ljc = __shfl_sync(FULL, lc, j);
        if (j <= lane) a[j] -= lc * ljc;
      }
    }
  }
  if (bad && lane == 0) *fail = 1;
  // stash L_kk (rows < rk), then invert column-wise: lane c owns column c of
  // X = L^{-1}: X_rc = (d_rc - sum_{k<r} L_rk X_kc) / L_rr
#pragma unroll
  for (int c = 0; c < 32; ++c)
    if (lane < rk && c <= lane) T[tri(lane) + c] = a[c];
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = 0.0;
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const double rr = __shfl_sync(FULL, my_rinv, r);
    if (r < rk) {
      double s0 = (lane == r) ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      const double* row = T + tri(r);
#pragma unroll
      for (int k = 0; k + 3 < r; k += 4) {
        s0 -= row[k] * a[k];
        s1 -= row[k + 1] * a[k + 1];
        s2 -= row[k + 2] * a[k + 2];
        s3 -= row[k + 3] * a[k + 3];
      }
#pragma unroll
      for (int k = r & ~3; k < r; ++k) s0 -= row[k] * a[k];
      a[r] = (lane <= r) ? ((s0 + s1) + (s2 + s3)) * rr : 0.0;
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 32; ++r)
    if (r < rk && lane <= r) T[tri(r) + lane] = a[r];
  __syncwarp();
}

// Panel: L_ik = A_ik Linv_kk^T for one row of tile (ti, k); in place.
__device__ __forceinline__ void panel_row(double* row, int r, const double* Linv) {
  double a[32];
  const int f = swz(r);
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = row[c ^ f];
#pragma unroll
  for (int c = 31; c >= 0; --c) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q <= c; ++q) s += a[q] * Linv[tri(c) + q];
    a[c] = s;
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) row[c ^ f] = a[c];
}

// Trailing update of tile (i, j) (k < j <= i): A_ij -= L_ik L_jk^T.
// Lane owns a 4 x 8 block: rows 4*(lane/4)+t, cols 8*(lane%4)+v.
__device__ __forceinline__ void syrk_tile(double* L, int i, int j, int k, int n, int lane) {
  const int ri = tile_rows(i, n), rj = tile_rows(j, n);
  const double* Pi = L + off_tile(i, k, n);
  const double* Pj = L + off_tile(j, k, n);
  const int rg = lane >> 2, cg = lane & 3;
  double acc[4][8];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[t][v] = 0.0;
  int rowi[4], rowj[8];
#pragma unroll
  for (int t = 0; t < 4; ++t) rowi[t] = min(4 * rg + t, ri - 1);
#pragma unroll
  for (int v = 0; v < 8; ++v) rowj[v] = min(8 * cg + v, rj - 1);
#pragma unroll 4
  for (int q = 0; q < 32; ++q) {
    double li[4], lj[8];
#pragma unroll
    for (int t = 0; t < 4; ++t) li[t] = Pi[rowi[t] * 32 + (q ^ swz(rowi[t]))];
#pragma unroll
    for (int v = 0; v < 8; ++v) lj[v] = Pj[rowj[v] * 32 + (q ^ swz(rowj[v]))];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int v = 0; v < 8; ++v) acc[t][v] += li[t] * lj[v];
  }
  if (i == j) {
    double* D = L + diag_tile(i, n);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int r = 4 * rg + t;
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int c = 8 * cg + v;
        if (r < ri && c <= r) D[tri(r) + c] -= acc[t][v];
      }
    }
  } else {
    double* A = L + off_tile(i, j, n);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int r = 4 * rg + t;
      if (r >= ri) continue;
      const int f = swz(r);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int c = 8 * cg + v;
        if (c < rj) A[r * 32 + (c ^ f)] -= acc[t][v];
      }
    }
  }
}

// ---------------------------------------------------------------- L^{-1}
// 4x8 register blocks over a 32x32 tile: lane owns rows 4*(lane>>2)+t, cols 8*(lane&3)+v.
// X_kj = Linv_kk * B_kj (in place; B_kj rows rk, full 32 columns)
__device__ __forceinline__ void trmm_left(double* L, int k, int j, int n, int lane) {
  const int rk = tile_rows(k, n);
  const double* Li = L + diag_tile(k, n);
  double* C = L + off_tile(k, j, n);
  const int rg = lane >> 2, cg = lane & 3;
  double acc[4][8];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[t][v] = 0.0;
#pragma unroll 4
  for (int q = 0; q < 32; ++q) {
    if (q >= rk) break;
    double li[4], cq[8];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int r = 4 * rg + t;
      li[t] = (q <= r && r < rk) ? Li[tri(r) + q] : 0.0;
    }
    const int f = swz(q);
#pragma unroll
    for (int v = 0; v < 8; ++v) cq[v] = C[q * 32 + ((8 * cg + v) ^ f)];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int v = 0; v < 8; ++v) acc[t][v] += li[t] * cq[v];
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int r = 4 * rg + t;
    if (r >= rk) continue;
    const int f = swz(r);
#pragma unroll
    for (int v = 0; v < 8; ++v) C[r * 32 + ((8 * cg + v) ^ f)] = acc[t][v];
  }
  __syncwarp();
}

// B_ik = -L_ik * Linv_kk (in place; tile (i, k), k < i, Linv_kk full 32x32)
__device__ __forceinline__ void trmm_right_neg(double* L, int i, int k, int n, int lane) {
  const int ri = tile_rows(i, n);
  const double* Li = L + diag_tile(k, n);
  double* C = L + off_tile(i, k, n);
  const int rg = lane >> 2, cg = lane & 3;
  double acc[4][8];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[t][v] = 0.0;
  int rowi[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) rowi[t] = min(4 * rg + t, ri - 1);
#pragma unroll 4
  for (int q = 0; q < 32; ++q) {
    double cr[4], lq[8];
#pragma unroll
    for (int t = 0; t < 4; ++t) cr[t] = C[rowi[t] * 32 + (q ^ swz(rowi[t]))];
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int c = 8 * cg + v;
      lq[v] = c <= q ? Li[tri(q) + c] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int v = 0; v < 8; ++v) acc[t][v] += cr[t] * lq[v];
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int r = 4 * rg + t;
    if (r >= ri) continue;
    const int f = swz(r);
#pragma unroll
    for (int v = 0; v < 8; ++v) C[r * 32 + ((8 * cg + v) ^ f)] = -acc[t][v];
  }
  __syncwarp();
}

// C_ij -= A_ik * X_kj  (all off-diagonal; k < T-1 so A and X have 32 columns)
__device__ __forceinline__ void gemm_sub(double* L, int i, int j, int k, int n, int lane) {
  const int ri = tile_rows(i, n);
  const double* A = L + off_tile(i, k, n);
  const double* X = L + off_tile(k, j, n);
  double* C = L + off_tile(i, j, n);
  const int rg = lane >> 2, cg = lane & 3;
  double acc[4][8];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[t][v] = 0.0;
  int rowi[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) rowi[t] = min(4 * rg + t, ri - 1);
#pragma unroll 4
  for (int q = 0; q < 32; ++q) {
    double a[4], x[8];
#pragma unroll
    for (int t = 0; t < 4; ++t) a[t] = A[rowi[t] * 32 + (q ^ swz(rowi[t]))];
    const int f = swz(q);
#pragma unroll
    for (int v = 0; v < 8; ++v) x[v] = X[q * 32 + ((8 * cg + v) ^ f)];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int v = 0; v < 8; ++v) acc[t][v] += a[t] * x[v];
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int r = 4 * rg + t;
    if (r >= ri) continue;
    const int f = swz(r);
#pragma unroll
    for (int v = 0; v < 8; ++v) C[r * 32 + ((8 * cg + v) ^ f)] -= acc[t][v];
  }
}

// Overwrite the Cholesky factor (diag tiles already inverted) with X = L^{-1}
// by right-looking block forward substitution on L X = I.
template <int NT>
__device__ void tri_inverse(double* L, int n, int T) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = 1; k < T; ++k) {
    // the column-(k-1) contributions B_i,k-1 = -L_i,k-1 Linv_k-1 (phase 3 of step k-1)
    // and B_ij -= L_i,k-1 X_k-1,j (phase 2) are applied below, in order.
    const int kk = k - 1;
    // phase 1 (step kk): X_kk,j = Linv_kk B_kk,j for j < kk
    for (int u = wid; u < kk; u += NW) trmm_left(L, kk, u, n, lane);
    __syncthreads();
    // phase 2 (step kk): B_ij -= L_i,kk X_kk,j for i > kk, j < kk
    const int below = T - kk - 1;
    for (int u = wid; u < below * kk; u += NW) gemm_sub(L, kk + 1 + u / kk, u % kk, kk, n, lane);
    __syncthreads();
    // phase 3 (step kk): B_i,kk = -L_i,kk Linv_kk for i > kk
    for (int u = wid; u < below; u += NW) trmm_right_neg(L, kk + 1 + u, kk, n, lane);
    __syncthreads();
  }
  // final step T-1: X_T-1,j = Linv B for j < T-1
  for (int u = wid; u < T - 1; u += NW) trmm_left(L, T - 1, u, n, lane);
  __syncthreads();
}

// x = X^T X b with X = L^{-1} (so x = D^{-1} b).  Warp i owns tile row i for
// w = X b (lane = row, a dot product over the whole tile row) and tile column
// i for x = X^T w (lane = column): no cross-warp reduction, two barriers.
template <int NT>
__device__ void inv_solve(const double* X, double* b, double* w, int n, int T) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  __syncthreads();
  for (int i = wid; i < T; i += NT / 32) {
    const int ri = tile_rows(i, n);
    const int r = lane;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (r < ri) {
      const int f = swz(r);
      for (int j = 0; j < i; ++j) {
        const double* row = X + off_tile(i, j, n) + r * 32;
        const double* bj = b + 32 * j;
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          a0 += row[c ^ f] * bj[c];
          a1 += row[(c + 1) ^ f] * bj[c + 1];
          a2 += row[(c + 2) ^ f] * bj[c + 2];
          a3 += row[(c + 3) ^ f] * bj[c + 3];
        }
      }
      const double* drow = X + diag_tile(i, n) + tri(r);
      const double* bi = b + 32 * i;
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        if (c <= r) a0 += drow[c] * bi[c];
        if (c + 1 <= r) a1 += drow[c + 1] * bi[c + 1];
      }
      w[32 * i + r] = (a0 + a1) + (a2 + a3);
    }
  }
  __syncthreads();
  for (int j = wid; j < T; j += NT / 32) {
    const int c = lane;
    const int rj = tile_rows(j, n);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (c < rj) {
      const double* D = X + diag_tile(j, n);
      const double* wj = w + 32 * j;
#pragma unroll
      for (int r = 0; r < 32; r += 2) {
        if (r >= c && r < rj) a0 += D[tri(r) + c] * wj[r];
        if (r + 1 >= c && r + 1 < rj) a1 += D[tri(r + 1) + c] * wj[r + 1];
      }
      for (int i = j + 1; i < T; ++i) {
        const int ri = tile_rows(i, n);
        const double* A = X + off_tile(i, j, n);
        const double* wi = w + 32 * i;
        if (ri == 32) {
#pragma unroll
          for (int r = 0; r < 32; r += 4) {
            a0 += A[r * 32 + (c ^ swz(r))] * wi[r];
            a1 += A[(r + 1) * 32 + (c ^ swz(r + 1))] * wi[r + 1];
            a2 += A[(r + 2) * 32 + (c ^ swz(r + 2))] * wi[r + 2];
            a3 += A[(r + 3) * 32 + (c ^ swz(r + 3))] * wi[r + 3];
          }
        } else {
          for (int r = 0; r < ri; ++r) a0 += A[r * 32 + (c ^ swz(r))] * wi[r];
        }
      }
      b[32 * j + c] = (a0 + a1) + (a2 + a3);
    }
  }
  __syncthreads();
}

// SOC projection of one contact triple (padmm.cpp:19-37)
__device__ __forceinline__ void project_soc(const double w[3], double mu, double y[3]) {
  const double wn = w[0];
  const double tn = sqrt(w[1] * w[1] + w[2] * w[2]);
  y[0] = w[0];
  y[1] = w[1];
  y[2] = w[2];
  if (tn <= mu * wn) return;
  if (mu * tn <= -wn) {
    y[0] = y[1] = y[2] = 0.0;
    return;
  }
  const double tau = (wn + mu * tn) / (1.0 + mu * mu);
  y[0] = tau;
  if (tn > 0) {
    y[1] = mu * tau * w[1] / tn;
    y[2] = mu * tau * w[2] / tn;
  } else {
    y[1] = y[2] = 0.0;
  }
}

}  // namespace

template <int NT, bool GLOBAL_L>
__global__ void __launch_bounds__(NT, 1) dense_kernel(BatchView bv, StepParams sp, const int32_t* bin_worlds) {
  extern __shared__ __align__(16) double smem[];
  const int w = bin_worlds[blockIdx.x];
  WorldStep& ws = bv.wstep[w];
  if (ws.backend != (GLOBAL_L ? BE_DENSE_GLOBAL : BE_DENSE_SMEM)) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = NT / 32;
  const DevWorld W = bv.worlds[w];
  const int n = ws.n_rows;
  const int T = (n + 31) >> 5;
  const int nlen = n * (n + 1) / 2;
  const int npad = 32 * T;
  double* L = GLOBAL_L ? bv.lslab + W.lslab_off : smem;
  double* xv = smem + (GLOBAL_L ? 0 : ((nlen + 1) & ~1));
  double* P = xv + npad;
  double* wv_s = P + npad;         // intermediate w = L^{-1} b
  double* red = wv_s + npad;       // 3 * NW
  int* rbs = reinterpret_cast<int*>(red + 3 * NW + 1);  // 2n body ids
  __shared__ int fail;
  const int64_t R0 = W.row_off;
  const RowJ* rj = bv.rowj + R0;
  const int32_t* rb = bv.rbody + 2 * R0;
  const double* regg = bv.reg + R0;
  const double eta_rho = sp.eta + sp.rho;

  long long t_prev = clock64();
  auto stamp = [&](int k) {
    if (tid == 0) {
      const long long t = clock64();
      ws.phase_cycles[k] = t - t_prev;
      t_prev = t;
    }
  };
  if (tid == 0) fail = 0;
  for (int r = tid; r < n; r += NT) {
    P[r] = bv.scale[R0 + r];
    rbs[2 * r] = rb[2 * r];
    rbs[2 * r + 1] = rb[2 * r + 1];
  }
  for (int e = tid; e < nlen; e += NT) L[e] = 0.0;
  __syncthreads();

  // ---- 1. D = sum_b Gram_b, ascending body order: phase 0 stores the term of
  // the smallest shared body, phase 1 adds the term of the larger one.
  {
    const int nb = W.nb;
    const int32_t* cptr = bv.csr_ptr + W.body_off + w;
    const int32_t* clist = bv.csr + 2 * R0;
    for (int phase = 0; phase < 2; ++phase) {
      for (int b = wid; b < nb; b += NW) {
        const int beg = cptr[b], end = cptr[b + 1];
        for (int pc = beg; pc < end; pc += 32) {
          const int p = pc + lane;
          double gm[6];
          int ip = -1;
          if (p < end) {
            const int e = clist[p];
            ip = e >> 1;
            const double* jm = rj[ip].JM + 6 * (e & 1);
#pragma unroll
            for (int k = 0; k < 6; ++k) gm[k] = jm[k];
          } else {
#pragma unroll
            for (int k = 0; k < 6; ++k) gm[k] = 0.0;
          }
          for (int qc = beg; qc <= pc; qc += 32) {
            const int q = qc + lane;
            double g[6];
            int iq = -1;
            if (q < end) {
              const int e = clist[q];
              iq = e >> 1;
              const double* jj = rj[iq].J + 6 * (e & 1);
#pragma unroll
              for (int k = 0; k < 6; ++k) g[k] = jj[k];
            } else {
#pragma unroll
              for (int k = 0; k < 6; ++k) g[k] = 0.0;
            }
            for (int qq = 0; qq < 32; ++qq) {
              const int jrow = __shfl_sync(FULL, iq, qq);
              double gq[6];
#pragma unroll
              for (int k = 0; k < 6; ++k) gq[k] = __shfl_sync(FULL, g[k], qq);
              if (ip < 0 || jrow < 0 || jrow > ip) continue;  // lower triangle, rows ascending
              // shared bodies of rows ip and jrow
              const int a0 = rbs[2 * ip], a1 = rbs[2 * ip + 1], c0 = rbs[2 * jrow], c1 = rbs[2 * jrow + 1];
              const bool s0 = a0 >= 0 && (a0 == c0 || a0 == c1);
              const bool s1 = a1 >= 0 && (a1 == c0 || a1 == c1);
              const int smin = (s0 && s1) ? min(a0, a1) : (s0 ? a0 : a1);
              const bool two = s0 && s1;
              const bool mine = phase == 0 ? (b == smin) : (two && b == max(a0, a1));
              if (!mine) continue;
              double s = 0.0;
#pragma unroll
              for (int k = 0; k < 6; ++k) s += gm[k] * gq[k];
              const int o = lidx(ip, jrow, n);
              if (phase == 0) L[o] = s;
              else L[o] += s;
            }
          }
        }
      }
      __syncthreads();
    }
  }
  stamp(0);
  // diagonal += R; P D P; += (eta + rho) I   (delassus.cpp:96-100)
  {
    const int ntiles = T * (T + 1) / 2;
    for (int u = wid; u < ntiles; u += NW) {
      int ti = 0;
      while ((ti + 1) * (ti + 2) / 2 <= u) ++ti;
      const int tj = u - ti * (ti + 1) / 2;
      const int rows = tile_rows(ti, n);
      if (ti == tj) {
        double* D = L + diag_tile(ti, n);
        for (int e = lane; e < tri(rows); e += 32) {
          int r = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
          while (tri(r + 1) <= e) ++r;
          while (tri(r) > e) --r;
          const int i = 32 * ti + r, j = 32 * ti + (e - tri(r));
          double d = D[e];
          if (i == j) d += regg[i];
          d = (P[i] * d) * P[j];
          if (i == j) d += eta_rho;
          D[e] = d;
        }
      } else {
        double* A = L + off_tile(ti, tj, n);
        const double pj = P[32 * tj + lane];
        for (int r = 0; r < rows; ++r) {
          const int o = r * 32 + (lane ^ swz(r));
          A[o] = (P[32 * ti + r] * A[o]) * pj;
        }
      }
    }
  }
  __syncthreads();
  stamp(1);
  // ---- 2. blocked right-looking Cholesky with look-ahead; diagonal tiles
  // become L_kk^{-1}.  While warps 1.. run the trailing update of step k,
  // warp 0 updates and factors diagonal tile k+1 (the critical path).
  if (wid == 0) diag_factor_invert(L + diag_tile(0, n), tile_rows(0, n), lane, &fail);
  __syncthreads();
  for (int k = 0; k < T; ++k) {
    const double* Linv = L + diag_tile(k, n);
    for (int i = 32 * (k + 1) + tid; i < n; i += NT) {
      const int ti = i >> 5, r = i & 31;
      panel_row(L + off_tile(ti, k, n) + r * 32, r, Linv);
    }
    __syncthreads();
    if (k + 1 < T) {
      const int m = T - k - 1;
      const int units = m * (m + 1) / 2;
      if (wid == 0) {
        syrk_tile(L, k + 1, k + 1, k, n, lane);
        __syncwarp();
        diag_factor_invert(L + diag_tile(k + 1, n), tile_rows(k + 1, n), lane, &fail);
      } else {
        for (int u = wid; u < units; u += NW - 1) {  // unit 0, tile (k+1, k+1), is warp 0's
          int ii = 0;
          while ((ii + 1) * (ii + 2) / 2 <= u) ++ii;
          const int jj = u - ii * (ii + 1) / 2;
          syrk_tile(L, k + 1 + ii, k + 1 + jj, k, n, lane);
        }
      }
      __syncthreads();
    }
  }
  if (fail) {
    if (tid == 0) {
      ws.fail = 1;
      atomicAdd(bv.error_count, 1);
    }
  }
  stamp(2);
  // ---- 2b. X = L^{-1}: every PADMM solve becomes two parallel mat-vecs
  tri_inverse<NT>(L, n, T);
  stamp(3);

  // ---- 3. PADMM (padmm.cpp:87-159), one cone unit per thread
  const int n_jd = ws.n_rows - ws.n_limits - 3 * ws.n_contacts;
  const int first_contact = n_jd + ws.n_limits;
  const int n_units = first_contact + ws.n_contacts;
  const bool has_unit = tid < n_units;
  const int row0 = tid < first_contact ? tid : first_contact + 3 * (tid - first_contact);
  const int kind = !has_unit ? ROW_BILATERAL : (tid < n_jd ? ROW_BILATERAL : (tid < first_contact ? ROW_LIMIT : ROW_CONTACT));
  const int nr = !has_unit ? 0 : (kind == ROW_CONTACT ? 3 : 1);
  const double mu = has_unit ? bv.rmu[R0 + row0] : 0.0;
  const double eta = sp.eta, rho = sp.rho;
  double v[3] = {0, 0, 0}, x[3] = {0, 0, 0}, y[3] = {0, 0, 0}, z[3] = {0, 0, 0}, yh[3], zh[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (d < nr) {
      v[d] = bv.vf[R0 + row0 + d];
      x[d] = bv.x0[R0 + row0 + d];
      z[d] = bv.z0[R0 + row0 + d];
    }
  }
  // y = Pi_K(x0)
  if (kind == ROW_CONTACT) project_soc(x, mu, y);
  else if (kind == ROW_LIMIT) y[0] = fmax(0.0, x[0]);
  else y[0] = x[0];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    yh[d] = y[d];
    zh[d] = z[d];
  }
  double a = 1.0, prev = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  double r_p = 0, r_d = 0, r_c = 0;
  int restarts = 0, it = 1;
  bool converged = false;
  const int hcap = bv.hist_cap;
  // rhs = -(v_f + s - eta x - rho y_hat - z_hat)   (padmm.cpp:116-117)
  auto write_rhs = [&]() {
    const double s0 = kind == ROW_CONTACT ? mu * hypot(zh[1], zh[2]) : 0.0;  // desaxce_shift (padmm.cpp:44-52)
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d < nr) xv[row0 + d] = -((((v[d] + (d == 0 ? s0 : 0.0)) - eta * x[d]) - rho * yh[d]) - zh[d]);
  };
  write_rhs();
  for (it = 1; it <= sp.max_iters; ++it) {
    inv_solve<NT>(L, xv, wv_s, n, T);
    double rp = 0.0, dmax = 0.0, rc = 0.0;
    double yp[3], zp[3], wv[3], yn[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (d < nr) x[d] = xv[row0 + d];
      wv[d] = x[d] - zh[d] / rho;
      yp[d] = y[d];
      zp[d] = z[d];
    }
    if (kind == ROW_CONTACT) project_soc(wv, mu, yn);
    else {
      yn[0] = kind == ROW_LIMIT ? fmax(0.0, wv[0]) : wv[0];
      yn[1] = yn[2] = 0.0;
    }
    double ymax = 0.0, zmax = 0.0;
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
    block_max3<NT>(rp, dmax, rc, red);
    r_p = rp;
    r_d = rho * dmax;
    r_c = rc;
    const double combined = fmax(r_p, fmax(r_d, r_c));
    if (tid == 0 && it <= hcap) bv.hist[(int64_t)w * hcap + it - 1] = combined;
    if (!sp.fixed_mode && combined < sp.eps) {
      converged = true;
      break;
    }
    if (sp.acceleration) {  // nesterov_update (padmm.cpp:58-71)
      const bool restart = sp.restart && combined > prev;
      if (restart) {
        a = 1.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          yh[d] = y[d];
          zh[d] = z[d];
        }
        ++restarts;
      } else {
        const double an = 0.5 * (1.0 + sqrt(1.0 + 4.0 * a * a));
        const double beta = (a - 1.0) / an;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          yh[d] = y[d] + beta * (y[d] - yp[d]);
          zh[d] = z[d] + beta * (z[d] - zp[d]);
        }
        a = an;
      }
    } else {
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        yh[d] = y[d];
        zh[d] = z[d];
      }
    }
    prev = combined;
    write_rhs();
  }
  stamp(4);
  // outputs (padmm.cpp:147-157)
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

// Shared-memory bytes the dense kernel needs for n rows with NT threads.
size_t dense_smem_bytes(int n, int nt, bool global_l) {
  const int T = (n + 31) / 32;
  const size_t nlen = global_l ? 0 : (size_t)((n * (n + 1) / 2 + 1) & ~1);
  return 8 * (nlen + 3 * (size_t)(32 * T) + 3 * (nt / 32) + 1) + 4 * 2 * (size_t)(32 * T) + 64;
}

template <int NT, bool G>
static cudaError_t launch_t(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, int cap,
                            cudaStream_t s) {
  const size_t smem = dense_smem_bytes(cap, NT, G);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    const cudaError_t e = cudaFuncSetAttribute(dense_kernel<NT, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  dense_kernel<NT, G><<<count, NT, smem, s>>>(bv, sp, worlds);
  return cudaGetLastError();
}

cudaError_t launch_dense(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, int cap, int nt,
                         bool global_l, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  if (global_l) return launch_t<384, true>(bv, sp, worlds, count, cap, s);
  switch (nt) {
    case 64: return launch_t<64, false>(bv, sp, worlds, count, cap, s);
    case 128: return launch_t<128, false>(bv, sp, worlds, count, cap, s);
    case 256: return launch_t<256, false>(bv, sp, worlds, count, cap, s);
    default: return launch_t<384, false>(bv, sp, worlds, count, cap, s);
  }
}

}  // namespace kd
