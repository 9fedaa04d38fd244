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

// Off-diagonal tiles are stored row-major with a padded row stride of 33
// doubles: element (r, c) at r*33 + c.  Since 33 = 1 (mod 16 bank pairs), a
// column walk (lane = row) and a row walk (lane = column) are both
// bank-conflict free for 8-byte words, and every address is base + constant
// (no per-element swizzle arithmetic in the mat-vec loops).
constexpr int LDT = 33;
__device__ __forceinline__ int tile_rows(int ti, int n) { return min(32, n - 32 * ti); }
__device__ __forceinline__ int tile_row_base(int ti) { return 528 * ti * ti; }
__device__ __forceinline__ int off_tile(int ti, int tj, int n) { return tile_row_base(ti) + tj * LDT * tile_rows(ti, n); }
__device__ __forceinline__ int diag_tile(int ti, int n) { return tile_row_base(ti) + ti * LDT * tile_rows(ti, n); }
__device__ __forceinline__ int tri(int r) { return (r * (r + 1)) >> 1; }
// element (i, j), i >= j
__device__ __forceinline__ int lidx(int i, int j, int n) {
  const int ti = i >> 5, tj = j >> 5, r = i & 31, c = j & 31;
  if (ti == tj) return diag_tile(ti, n) + tri(r) + c;
  return off_tile(ti, tj, n) + r * LDT + c;
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

// Block maximum of one non-negative value per thread (one barrier).
template <int NT>
__device__ __forceinline__ double block_max_nonneg(double v, double* red) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_max_nonneg(v);
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double m[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) m[k] = red[k];
#pragma unroll
  for (int s = 1; s < NW; s *= 2)
#pragma unroll
    for (int k = 0; k + s < NW; k += 2 * s) m[k] = fmax(m[k], m[k + s]);
  return m[0];
}

// ---------------------------------------------------------------- Cholesky pieces
// Factor the packed diagonal tile in place and overwrite it with L_kk^{-1}.
// One warp; lane r owns row r in registers (fully unrolled so every register
// index is static; the kernel calls this from exactly one site to keep a
// single copy of the code in the instruction cache).  Pivots use one
// reciprocal square root each (L_cc = d r, L_rc = a_rc r, r = 1/sqrt(d)); the
// reciprocals are kept so the inverse is division-free.
__device__ __noinline__ void diag_factor_invert(double* T, int rk, int lane, int* fail, double* col) {
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = (lane < rk && c <= lane) ? T[tri(lane) + c] : (c == lane ? 1.0 : 0.0);
  bool bad = false;
  double my_rinv = 1.0;
  // pivot c: column c goes through shared memory (one store, broadcast reads)
  // instead of 31 shuffles, and 1/sqrt(d) is a float seed plus two Newton
  // steps instead of the generic rsqrt; both were the diagonal chain's cost
  // (tools/microbench_chain.cu: 16.5k -> 11.7k cycles per tile)
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    col[lane] = a[c];
    __syncwarp();
    const double dcc = col[c];
    if (!(dcc > 0.0)) bad = true;
    const double rinv = fast_rsqrt(dcc);
    const double lc = lane > c ? a[c] * rinv : (lane == c ? dcc * rinv : a[c]);
    if (lane == c) my_rinv = rinv;
    a[c] = lc;
#pragma unroll
    for (int j = c + 1; j < 32; ++j) {
      const double ljc = col[j] * rinv;  // = lane j's L_jc
      if (j <= lane) a[j] -= lc * ljc;
    }
    __syncwarp();
  }
  if (bad && lane == 0) *fail = 1;
#pragma unroll
  for (int c = 0; c < 32; ++c)
    if (lane < rk && c <= lane) T[tri(lane) + c] = a[c];
  __syncwarp();
  // lane c owns column c of X = L^{-1}: X_rc = (d_rc - sum_{k<r} L_rk X_kc) / L_rr
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

// Overwrite a packed lower diagonal tile that holds L_rc (c < r) and 1/L_rr on
// its diagonal (the supernodal factor's hand-off format) with L_kk^{-1}; the
// same column-parallel substitution as the second half of diag_factor_invert.
__device__ __noinline__ void diag_invert_rinv(double* T, int rk, int lane) {
  const double my_rinv = lane < rk ? T[tri(lane) + lane] : 1.0;
  double a[32];
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

// ---------------------------------------------------------------- DMMA tile products
// One warp computes a 32x32 tile product with FP64 tensor-core MMAs
// (mma.sync m8n8k4 f64: 256 FMA per instruction; tcgen05 has no fp64 kind).
// Fragment layout: A (8x4 row) lane l -> A[l>>2][l&3]; B (4x8 col) lane l ->
// B[l&3][l>>2]; C (8x8) lane l -> C[l>>2][2(l&3)+{0,1}].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// element loaders (rows beyond `rows` read as 0)
struct OffT {  // off-diagonal tile, swizzled
  const double* p;
  int rows;
  __device__ __forceinline__ double operator()(int r, int c) const { return r < rows ? p[r * LDT + c] : 0.0; }
};
struct OffTT {  // transpose of an off-diagonal tile
  const double* p;
  int rows;
  __device__ __forceinline__ double operator()(int r, int c) const { return c < rows ? p[c * LDT + r] : 0.0; }
};
struct DiagL {  // packed lower diagonal tile
  const double* p;
  int rows;
  __device__ __forceinline__ double operator()(int r, int c) const { return (r < rows && c <= r) ? p[tri(r) + c] : 0.0; }
};
struct DiagLT {  // transpose of a packed lower diagonal tile (upper)
  const double* p;
  int rows;
  __device__ __forceinline__ double operator()(int r, int c) const { return (c < rows && r <= c) ? p[tri(c) + r] : 0.0; }
};

// acc[mb][nb][h] += sum_k A(8mb+l/4, k) B(k, 8nb+2(l%4)+h), k < 32
// kmask: the 4-wide k steps to execute (a step whose A columns are all
// structurally zero adds exact zeros: skipping it leaves the result bitwise equal)
template <class LA, class LB>
__device__ __forceinline__ void mma_tile(double acc[4][4][2], const LA& la, const LB& lb, unsigned kmask = 0xffu) {
  const int lane = threadIdx.x & 31, qr = lane >> 2, qc = lane & 3;
#pragma unroll 2
  for (int ks = 0; ks < 8; ++ks) {
    if (!((kmask >> ks) & 1u)) continue;
    double a[4], b[4];
#pragma unroll
    for (int mb = 0; mb < 4; ++mb) a[mb] = la(8 * mb + qr, 4 * ks + qc);
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) b[nb] = lb(4 * ks + qc, 8 * nb + qr);
#pragma unroll
    for (int mb = 0; mb < 4; ++mb)
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb][0], acc[mb][nb][1], a[mb], b[nb]);
  }
}

__device__ __forceinline__ void zero_acc(double acc[4][4][2]) {
#pragma unroll
  for (int mb = 0; mb < 4; ++mb)
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) acc[mb][nb][0] = acc[mb][nb][1] = 0.0;
}

// C (off-diagonal, rows) = alpha * acc + beta * C
__device__ __forceinline__ void store_off(double* C, int rows, const double acc[4][4][2], double alpha, bool accumulate) {
  const int lane = threadIdx.x & 31, qr = lane >> 2, qc = lane & 3;
#pragma unroll
  for (int mb = 0; mb < 4; ++mb) {
    const int r = 8 * mb + qr;
    if (r >= rows) continue;
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int o = r * LDT + 8 * nb + 2 * qc + h;
        C[o] = accumulate ? C[o] + alpha * acc[mb][nb][h] : alpha * acc[mb][nb][h];
      }
  }
}

// C (packed lower diagonal, rows) -= acc (lower part only)
__device__ __forceinline__ void sub_diag(double* C, int rows, const double acc[4][4][2]) {
  const int lane = threadIdx.x & 31, qr = lane >> 2, qc = lane & 3;
#pragma unroll
  for (int mb = 0; mb < 4; ++mb) {
    const int r = 8 * mb + qr;
    if (r >= rows) continue;
#pragma unroll
    for (int nb = 0; nb <= mb; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 8 * nb + 2 * qc + h;
        if (c <= r) C[tri(r) + c] -= acc[mb][nb][h];
      }
  }
}

// Trailing update of tile (i, j) (k < j <= i): A_ij -= L_ik L_jk^T.
__device__ __forceinline__ void syrk_tile(double* L, int i, int j, int k, int n, int lane) {
  double acc[4][4][2];
  zero_acc(acc);
  mma_tile(acc, OffT{L + off_tile(i, k, n), tile_rows(i, n)}, OffTT{L + off_tile(j, k, n), tile_rows(j, n)});
  if (i == j) sub_diag(L + diag_tile(i, n), tile_rows(i, n), acc);
  else store_off(L + off_tile(i, j, n), tile_rows(i, n), acc, -1.0, true);
}

// Panel tile: L_ik = A_ik Linv_kk^T (in place).
__device__ __forceinline__ void panel_tile(double* L, int i, int k, int n) {
  double acc[4][4][2];
  zero_acc(acc);
  double* A = L + off_tile(i, k, n);
  const int ri = tile_rows(i, n);
  mma_tile(acc, OffT{A, ri}, DiagLT{L + diag_tile(k, n), 32});
  __syncwarp();
  store_off(A, ri, acc, 1.0, false);
}

// One 8-row block mb of a tile product: acc[nb][h] += sum_k A(8mb+l/4, k)
// B(k, 8nb+2(l%4)+h) — the same DMMAs, in the same order, as mma_tile's row
// block mb, so a tile computed as four row-block jobs is bitwise the same.
template <class LA, class LB>
__device__ __forceinline__ void mma_rows(double acc[4][2], int mb, const LA& la, const LB& lb, unsigned kmask = 0xffu) {
  const int lane = threadIdx.x & 31, qr = lane >> 2, qc = lane & 3;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    if (!((kmask >> ks) & 1u)) continue;
    const double a = la(8 * mb + qr, 4 * ks + qc);
    double b[4];
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) b[nb] = lb(4 * ks + qc, 8 * nb + qr);
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) dmma(acc[nb][0], acc[nb][1], a, b[nb]);
  }
}

// rows 8mb..8mb+7 of C (off-diagonal, rows) = alpha * acc + beta * C
__device__ __forceinline__ void store_rows(double* C, int rows, const double acc[4][2], double alpha, bool accumulate,
                                           int mb) {
  const int lane = threadIdx.x & 31, qr = lane >> 2, qc = lane & 3;
  const int r = 8 * mb + qr;
  if (r >= rows) return;
#pragma unroll
  for (int nb = 0; nb < 4; ++nb)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int o = r * LDT + 8 * nb + 2 * qc + h;
      C[o] = accumulate ? C[o] + alpha * acc[nb][h] : alpha * acc[nb][h];
    }
}

// ---------------------------------------------------------------- L^{-1}
// X_kj = Linv_kk * B_kj (in place)
__device__ __forceinline__ void trmm_left(double* L, int k, int j, int n, int lane) {
  double acc[4][4][2];
  zero_acc(acc);
  const int rk = tile_rows(k, n);
  double* C = L + off_tile(k, j, n);
  mma_tile(acc, DiagL{L + diag_tile(k, n), rk}, OffT{C, rk});
  __syncwarp();
  store_off(C, rk, acc, 1.0, false);
}

// B_ik = -L_ik * Linv_kk (in place)
__device__ __forceinline__ void trmm_right_neg(double* L, int i, int k, int n, int lane, unsigned km = 0xffu) {
  double acc[4][4][2];
  zero_acc(acc);
  const int ri = tile_rows(i, n);
  double* C = L + off_tile(i, k, n);
  mma_tile(acc, OffT{C, ri}, DiagL{L + diag_tile(k, n), 32}, km);
  __syncwarp();
  store_off(C, ri, acc, -1.0, false);
}

// C_ij -= A_ik * X_kj
__device__ __forceinline__ void gemm_sub(double* L, int i, int j, int k, int n, int lane, unsigned km = 0xffu) {
  double acc[4][4][2];
  zero_acc(acc);
  mma_tile(acc, OffT{L + off_tile(i, k, n), tile_rows(i, n)}, OffT{L + off_tile(k, j, n), 32}, km);
  store_off(L + off_tile(i, j, n), tile_rows(i, n), acc, -1.0, true);
}

// Row-block jobs of the two phases whose output rows depend only on the same
// rows of their left operand (so the four jobs of a tile may run on different
// warps, in place): a single warp's 32x32 DMMA product is bound by its
// sub-partition's FP64 tensor rate, so a phase with fewer tiles than warps
// finishes sooner split into row blocks.
__device__ __forceinline__ void gemm_sub_rows(double* L, int i, int j, int k, int n, int mb, unsigned km) {
  const int ri = tile_rows(i, n);
  if (8 * mb >= ri) return;
  double acc[4][2];
#pragma unroll
  for (int nb = 0; nb < 4; ++nb) acc[nb][0] = acc[nb][1] = 0.0;
  mma_rows(acc, mb, OffT{L + off_tile(i, k, n), ri}, OffT{L + off_tile(k, j, n), 32}, km);
  store_rows(L + off_tile(i, j, n), ri, acc, -1.0, true, mb);
}
__device__ __forceinline__ void trmm_right_neg_rows(double* L, int i, int k, int n, int mb, unsigned km) {
  const int ri = tile_rows(i, n);
  if (8 * mb >= ri) return;
  double acc[4][2];
#pragma unroll
  for (int nb = 0; nb < 4; ++nb) acc[nb][0] = acc[nb][1] = 0.0;
  double* C = L + off_tile(i, k, n);
  mma_rows(acc, mb, OffT{C, ri}, DiagL{L + diag_tile(k, n), 32}, km);
  __syncwarp();
  store_rows(C, ri, acc, -1.0, false, mb);
}
#ifndef KD_INV_SPLIT
#define KD_INV_SPLIT 1
#endif


// Overwrite the Cholesky factor (diag tiles already inverted) with X = L^{-1}
// by right-looking block forward substitution on L X = I.
// lmask / xmask: bit ti(ti+1)/2 + tj set for every tile of L / of X that can
// be nonzero (all ones unless the factor came from a supernodal plan).  A zero
// tile L_i,kk contributes nothing to phases 2 and 3; a structurally zero tile
// X_kk,j is never formed (phase 1) nor used (phase 2).
// (masks exist only for supernodal hand-off factors, T <= 8; an all-ones mask
// means "every tile", valid for any T)
__device__ __forceinline__ bool mtile(unsigned long long mask, int ti, int tj) {
  return mask == ~0ull || ((mask >> (ti * (ti + 1) / 2 + tj)) & 1ull);
}
template <int NT>
__device__ void tri_inverse(double* L, int n, int T, unsigned long long lmask, unsigned long long xmask,
                            const uint8_t* kmask = nullptr, long long* prof = nullptr) {
  auto km = [&](int i, int k) -> unsigned { return kmask ? kmask[i * (i + 1) / 2 + k] : 0xffu; };
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto nth_bit = [](unsigned m, int q) {  // position of the q-th set bit
    for (int t = 0; t < q; ++t) m &= m - 1;
    return __ffs(m) - 1;
  };
  const bool full = lmask == ~0ull && xmask == ~0ull;  // dense factor: every tile, any T
#ifdef KD_PROF_INV
  long long c1 = 0, c2 = 0, c3 = 0, cq = clock64();
#endif
  for (int k = 1; k < T; ++k) {
    // the column-(k-1) contributions B_i,k-1 = -L_i,k-1 Linv_k-1 (phase 3 of step k-1)
    // and B_ij -= L_i,k-1 X_k-1,j (phase 2) are applied below, in order.
    const int kk = k - 1;
    unsigned rows = 0, cols = 0;  // rows i > kk with L_i,kk != 0; columns j < kk with X_kk,j != 0
    int below = T - 1 - kk, nc = kk;
    if (!full) {
      for (int i = kk + 1; i < T; ++i)
        if (mtile(lmask, i, kk)) rows |= 1u << i;
      for (int j = 0; j < kk; ++j)
        if (mtile(xmask, kk, j)) cols |= 1u << j;
      below = __popc(rows);
      nc = __popc(cols);
    }
    auto row_at = [&](int q) { return full ? kk + 1 + q : nth_bit(rows, q); };
    auto col_at = [&](int q) { return full ? q : nth_bit(cols, q); };
    // phase 1 (step kk): X_kk,j = Linv_kk B_kk,j for j < kk.  Its output rows
    // mix every row of B_kk,j, so row-block jobs (one per warp) compute into
    // registers and store after a barrier.
    if (KD_INV_SPLIT && nc > 0 && 4 * nc <= NW) {
      const int t = wid >> 2, mb = wid & 3;
      const int rk = tile_rows(kk, n);
      double acc[4][2];
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) acc[nb][0] = acc[nb][1] = 0.0;
      double* C = t < nc ? L + off_tile(kk, col_at(t), n) : nullptr;
      if (C && 8 * mb < rk) mma_rows(acc, mb, DiagL{L + diag_tile(kk, n), rk}, OffT{C, rk});
      __syncthreads();
      if (C && 8 * mb < rk) store_rows(C, rk, acc, 1.0, false, mb);
    } else {
      for (int u = wid; u < nc; u += NW) trmm_left(L, kk, col_at(u), n, lane);
    }
    __syncthreads();
#ifdef KD_PROF_INV
    { const long long t = clock64(); c1 += t - cq; cq = t; }
#endif
    // phase 2 (step kk): B_ij -= L_i,kk X_kk,j for i > kk, j < kk
    if (KD_INV_SPLIT && below * nc < NW) {  // fewer tiles than warps: row-block jobs
      for (int u = wid; u < 4 * below * nc; u += NW) {
        const int t = u >> 2, i = row_at(t / nc);
        gemm_sub_rows(L, i, col_at(t % nc), kk, n, u & 3, km(i, kk));
      }
    } else {
      for (int u = wid; u < below * nc; u += NW) {
        const int i = row_at(u / nc);
        gemm_sub(L, i, col_at(u % nc), kk, n, lane, km(i, kk));
      }
    }
    __syncthreads();
#ifdef KD_PROF_INV
    { const long long t = clock64(); c2 += t - cq; cq = t; }
#endif
    // phase 3 (step kk): B_i,kk = -L_i,kk Linv_kk for i > kk
    if (KD_INV_SPLIT && below < NW) {
      for (int u = wid; u < 4 * below; u += NW) {
        const int i = row_at(u >> 2);
        trmm_right_neg_rows(L, i, kk, n, u & 3, km(i, kk));
      }
    } else {
      for (int u = wid; u < below; u += NW) {
        const int i = row_at(u);
        trmm_right_neg(L, i, kk, n, lane, km(i, kk));
      }
    }
    __syncthreads();
#ifdef KD_PROF_INV
    { const long long t = clock64(); c3 += t - cq; cq = t; }
#endif
  }
  // final step T-1: X_T-1,j = Linv B for j < T-1
  for (int u = wid; u < T - 1; u += NW)
    if (mtile(xmask, T - 1, u)) trmm_left(L, T - 1, u, n, lane);
  __syncthreads();
#ifdef KD_PROF_INV
  if (prof && threadIdx.x == 0) {
    prof[5] = c1;  // phase 1 (incl. its barriers)
    prof[6] = c2;  // phase 2
    prof[7] = c3;  // phase 3
    prof[1] = clock64() - cq;  // final step
  }
#endif
}

// x = X^T X b with X = L^{-1} (so x = D^{-1} b).  Warp i owns tile row i for
// w = X b (lane = row, a dot product over the whole tile row) and tile column
// i for x = X^T w (lane = column): no cross-warp reduction, two barriers.
// Padded tiles give both walks constant offsets and no bank conflicts; the
// broadcast vector operand is read as double2 (one wavefront per two entries).
template <int NT>
__device__ void inv_solve(const double* X, double* b, double* w, int n, int T, unsigned long long xmask,
                          long long* prof = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  __syncthreads();
#ifdef KD_PROF_PADMM
  long long q0 = clock64();
#endif
#ifdef KD_PROF_WARP
  const long long qw0 = clock64();
#endif
  for (int i = wid; i < T; i += NT / 32) {
    const int ri = tile_rows(i, n), r = lane;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (r < ri) {
      for (int j = 0; j < i; ++j) {
        if (!mtile(xmask, i, j)) continue;  // structurally zero tile of L^-1
        const double* row = X + off_tile(i, j, n) + r * LDT;
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
      const double* drow = X + diag_tile(i, n) + tri(r);
      const double2* bi = reinterpret_cast<const double2*>(b + 32 * i);
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        const double2 bb = bi[c / 2];
        if (c <= r) a0 += drow[c] * bb.x;
        if (c + 1 <= r) a1 += drow[c + 1] * bb.y;
      }
      w[32 * i + r] = (a0 + a1) + (a2 + a3);
    }
  }
#ifdef KD_PROF_WARP
  __syncwarp();
  if (KD_PROF_WARP == 1 && prof) prof[4 + wid] += clock64() - qw0;
#endif
  __syncthreads();
#ifdef KD_PROF_WARP
  const long long qw1 = clock64();
#endif
#ifdef KD_PROF_PADMM
  long long q1 = clock64();
  prof[0] += q1 - q0;
#endif
  for (int j = wid; j < T; j += NT / 32) {
    const int c = lane, rj = tile_rows(j, n);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (c < rj) {
      const double* D = X + diag_tile(j, n);
      const double2* wj = reinterpret_cast<const double2*>(w + 32 * j);
#pragma unroll
      for (int r = 0; r < 32; r += 2) {
        const double2 ww = wj[r / 2];
        if (r >= c && r < rj) a0 += D[tri(r) + c] * ww.x;
        if (r + 1 >= c && r + 1 < rj) a1 += D[tri(r + 1) + c] * ww.y;
      }
      for (int i = j + 1; i < T; ++i) {
        if (!mtile(xmask, i, j)) continue;
        const int ri = tile_rows(i, n);
        const double* A = X + off_tile(i, j, n) + c;
        const double2* wi = reinterpret_cast<const double2*>(w + 32 * i);
        if (ri == 32) {
#pragma unroll
          for (int r = 0; r < 32; r += 4) {
            const double2 w01 = wi[r / 2], w23 = wi[r / 2 + 1];
            a0 += A[r * LDT] * w01.x;
            a1 += A[(r + 1) * LDT] * w01.y;
            a2 += A[(r + 2) * LDT] * w23.x;
            a3 += A[(r + 3) * LDT] * w23.y;
          }
        } else {  // the last tile row: same walk, rows >= ri predicated off
#pragma unroll
          for (int r = 0; r < 32; r += 4) {
            const double2 w01 = wi[r / 2], w23 = wi[r / 2 + 1];
            if (r < ri) a0 += A[r * LDT] * w01.x;
            if (r + 1 < ri) a1 += A[(r + 1) * LDT] * w01.y;
            if (r + 2 < ri) a2 += A[(r + 2) * LDT] * w23.x;
            if (r + 3 < ri) a3 += A[(r + 3) * LDT] * w23.y;
          }
        }
      }
      b[32 * j + c] = (a0 + a1) + (a2 + a3);
    }
  }
#ifdef KD_PROF_WARP
  __syncwarp();
  if (KD_PROF_WARP == 2 && prof) prof[4 + wid] += clock64() - qw1;
#endif
  __syncthreads();
#ifdef KD_PROF_PADMM
  prof[1] += clock64() - q1;
#endif
}


// Release / acquire flags in shared memory (CTA scope).
__device__ __forceinline__ void flag_release(int* f, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(f)), "r"(v) : "memory");
}
__device__ __forceinline__ int flag_acquire(const int* f) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(f)) : "memory");
  return v;
}

// Register-resident tiles of X for the dataflow solve.  During PADMM most of
// the 255 registers the L^-1 formation needed are free; each warp parks up to
// KD_DF_REG tiles of X there, in the orientation of the pass that uses them
// (pass 1: lane = row, pass 2: lane = column, 32 doubles per lane, zeros
// outside the tile's triangle / rows).  A register tile costs the pass only
// its 16 broadcast wavefronts instead of 80 (64 for the tile + 16), and the
// tiles chosen are the ones on the dataflow critical path: the pass-2 tile of
// the last tile row (published last) and the first tiles of the warp's own
// tile row.  The dot products run in the same order with the same
// accumulators as from shared memory (bitwise the same up to the sign of
// exact zeros).
#ifndef KD_TMEM
#define KD_TMEM 1
#endif
#ifndef KD_DF_REG
#define KD_DF_REG (KD_TMEM ? 1 : 2)  // with TMEM tiles one register tile per warp measured best
#endif
constexpr int DF_NC = KD_DF_REG;
struct RegTiles {
  double v[DF_NC > 0 ? DF_NC : 1][32];
  int id[DF_NC > 0 ? DF_NC : 1];  // pass << 8 | i << 4 | j, or -1
};
__device__ __forceinline__ int rt_id(int pass, int i, int j) { return (pass << 8) | (i << 4) | j; }

// slot of tile (pass, i, j) in R, or -1
__device__ __forceinline__ int rt_slot(const RegTiles& R, int pass, int i, int j) {
  const int q = rt_id(pass, i, j);
  int s = -1;
#pragma unroll
  for (int k = 0; k < DF_NC; ++k)
    if (R.id[k] == q) s = k;
  return s;
}

// the t-th register-tile candidate of warp wid: 1. the pass-2 tile of the
// last tile row in this warp's column, 2. the first tiles of this warp's tile
// row (pass 1)
__device__ __forceinline__ int rt_cand(int wid, int t, int T, unsigned long long xmask) {
  if (wid >= T) return -1;
  if (wid < T - 1 && mtile(xmask, T - 1, wid)) {
    if (t == 0) return rt_id(2, T - 1, wid);
    --t;
  }
  for (int j = 0; j <= wid; ++j)
    if (mtile(xmask, wid, j)) {
      if (t == 0) return rt_id(1, wid, j);
      --t;
    }
  return -1;
}

// pick and load warp `wid`'s register tiles (after X is final; warp-uniform)
__device__ void rt_load(RegTiles& R, const double* X, int n, int T, unsigned long long xmask) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int s = 0; s < DF_NC; ++s) R.id[s] = rt_cand(wid, s, T, xmask);  // static slot index: R stays in registers
#pragma unroll
  for (int s = 0; s < DF_NC; ++s) {
    const int q = R.id[s];
    if (q < 0) {
#pragma unroll
      for (int e = 0; e < 32; ++e) R.v[s][e] = 0.0;
      continue;
    }
    const int pass = q >> 8, i = (q >> 4) & 15, j = q & 15;
    const int ri = tile_rows(i, n);
    if (i == j) {
      const double* D = X + diag_tile(i, n);
      if (pass == 1) {  // lane = row r: X[r][c], c <= r
#pragma unroll
        for (int c = 0; c < 32; ++c) R.v[s][c] = (lane < ri && c <= lane) ? D[tri(lane) + c] : 0.0;
      } else {  // lane = column c: X[r][c], r >= c
#pragma unroll
        for (int r = 0; r < 32; ++r) R.v[s][r] = (lane < ri && r >= lane && r < ri) ? D[tri(r) + lane] : 0.0;
      }
    } else {
      const double* A = X + off_tile(i, j, n);
      if (pass == 1) {
#pragma unroll
        for (int c = 0; c < 32; ++c) R.v[s][c] = lane < ri ? A[lane * LDT + c] : 0.0;
      } else {
#pragma unroll
        for (int r = 0; r < 32; ++r) R.v[s][r] = r < ri ? A[r * LDT + lane] : 0.0;
      }
    }
  }
}

// acc += tile . v (4-accumulator off-diagonal order / 2-accumulator diagonal order)
__device__ __forceinline__ void rt_dot_off(const double* t, const double* v, double& a0, double& a1, double& a2,
                                           double& a3) {
  const double2* v2 = reinterpret_cast<const double2*>(v);
#pragma unroll
  for (int c = 0; c < 32; c += 4) {
    const double2 p = v2[c / 2], q = v2[c / 2 + 1];
    a0 += t[c] * p.x;
    a1 += t[c + 1] * p.y;
    a2 += t[c + 2] * q.x;
    a3 += t[c + 3] * q.y;
  }
}
__device__ __forceinline__ void rt_dot_diag(const double* t, const double* v, double& a0, double& a1) {
  const double2* v2 = reinterpret_cast<const double2*>(v);
#pragma unroll
  for (int c = 0; c < 32; c += 2) {
    const double2 p = v2[c / 2];
    a0 += t[c] * p.x;
    a1 += t[c + 1] * p.y;
  }
}
template <int S>
struct RtDispatch {  // static register indexing: slot k -> R.v[k]
  __device__ __forceinline__ static void off(const RegTiles& R, int k, const double* v, double& a0, double& a1,
                                             double& a2, double& a3) {
    if (k == S - 1) rt_dot_off(R.v[S - 1], v, a0, a1, a2, a3);
    else RtDispatch<S - 1>::off(R, k, v, a0, a1, a2, a3);
  }
  __device__ __forceinline__ static void diag(const RegTiles& R, int k, const double* v, double& a0, double& a1) {
    if (k == S - 1) rt_dot_diag(R.v[S - 1], v, a0, a1);
    else RtDispatch<S - 1>::diag(R, k, v, a0, a1);
  }
};
template <>
struct RtDispatch<0> {
  __device__ __forceinline__ static void off(const RegTiles&, int, const double*, double&, double&, double&,
                                             double&) {}
  __device__ __forceinline__ static void diag(const RegTiles&, int, const double*, double&, double&) {}
};

// Tensor-memory tiles of X for the dataflow solve.  The tile visits of the
// solve passes that do not fit the register tiles are parked in TMEM (512
// columns x 128 lanes, allocated per CTA for the PADMM loop; one K2 CTA per
// SM), in the orientation of the pass that reads them: lane = row (pass 1) or
// column (pass 2), 32 doubles = 64 columns per tile.  A warp reaches only its
// lane quarter (warp % 4), which it shares with warp ^ 4: each quarter holds 8
// tiles, split between its two warps by need.  tcgen05.ld streams a tile row
// at ~256 B/clk/SM on a path separate from shared memory's 128 B/clk
// (tools/microbench_tmem.cu), so a TMEM visit costs the shared-memory pipe
// only its vector broadcast.  Same dot-product order as the register tiles.
struct TmTiles {
  unsigned m1, m2;  // bit j: pass-1 tile (wid, j) in TMEM; bit i: pass-2 tile (i, wid)
  uint32_t c1, c2;  // TMEM address of the first pass-1 / pass-2 tile
  unsigned r1, r2;  // bit j: tile (wid, j), j < wid, of X nonzero; bit i: tile (i, wid), i > wid, nonzero
};
// the warp's nonzero off-diagonal tiles of its tile row / tile column (the
// solve passes walk these bits instead of testing the mask per tile)
__device__ __forceinline__ void df_masks(TmTiles& M, int T, unsigned long long xmask) {
  const int v = threadIdx.x >> 5;
  unsigned row = 0u, col = 0u;
  if (v < T) {
    if (xmask == ~0ull) {
      row = (1u << v) - 1u;
      col = ((1u << T) - 1u) & ~((2u << v) - 1u);
    } else {
      row = (unsigned)(xmask >> (v * (v + 1) / 2)) & ((1u << v) - 1u);
      for (int i = v + 1; i < T; ++i) col |= (unsigned)((xmask >> (i * (i + 1) / 2 + v)) & 1ull) << i;
    }
  }
  M.r1 = row;
  M.r2 = col;
}

// non-register tile visits of warp v, pass-2 tiles first (they sit on the
// dataflow critical path), then pass 1; at most `budget` of them.  Bit masks
// over the tile index: row v's tiles (pass 1) and column v's (pass 2); the
// register tiles (rt_cand's order) are the pass-2 tile (T-1, v) and then the
// lowest tiles of row v.
__device__ __forceinline__ unsigned low_bits(unsigned m, int k) {  // the k lowest set bits of m
  unsigned r = 0u;
  for (int t = 0; t < k && m; ++t) {
    const unsigned b = m & (0u - m);
    r |= b;
    m ^= b;
  }
  return r;
}
__device__ __forceinline__ void tm_visits(int v, int T, unsigned long long xmask, int budget, unsigned& m1,
                                          unsigned& m2, int& need) {
  m1 = m2 = 0u;
  need = 0;
  if (v >= T) return;
  unsigned row, col = 0u;
  if (xmask == ~0ull) {
    row = (2u << v) - 1u;
    col = ((1u << T) - 1u) & ~((1u << v) - 1u);
  } else {
    row = (unsigned)(xmask >> (v * (v + 1) / 2)) & ((2u << v) - 1u);
    for (int i = v; i < T; ++i) col |= (unsigned)((xmask >> (i * (i + 1) / 2 + v)) & 1ull) << i;
  }
  int nreg = DF_NC;
  if (nreg > 0 && v < T - 1 && ((col >> (T - 1)) & 1u)) {
    col &= ~(1u << (T - 1));
    --nreg;
  }
  row &= ~low_bits(row, nreg);
  need = __popc(col) + __popc(row);
  m2 = low_bits(col, budget);
  m1 = low_bits(row, budget - __popc(m2));
}

__device__ __forceinline__ void tm_st8(uint32_t taddr, const double (&d)[8]) {
  uint32_t r[16];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    r[2 * k] = (uint32_t)__double2loint(d[k]);
    r[2 * k + 1] = (uint32_t)__double2hiint(d[k]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
// 8 doubles of this lane's row from TMEM (load and wait in one statement, so
// no use of the registers can be scheduled before the data arrives)
__device__ __forceinline__ void tm_ld8(uint32_t taddr, double (&d)[8]) {
  uint32_t r[16];
  asm volatile(
      "{\n tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      " tcgen05.wait::ld.sync.aligned;\n}"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int k = 0; k < 8; ++k) d[k] = __hiloint2double((int)r[2 * k + 1], (int)r[2 * k]);
}

// 16 doubles of this lane's row (one tcgen05.ld.32x32b.x32, then the wait)
__device__ __forceinline__ void tm_ld16(uint32_t taddr, double (&d)[16]) {
  uint32_t r[32];
  asm volatile(
      "{\n tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      " tcgen05.wait::ld.sync.aligned;\n}"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int k = 0; k < 16; ++k) d[k] = __hiloint2double((int)r[2 * k + 1], (int)r[2 * k]);
}
// a whole 32-double row (one tcgen05.ld.32x32b.x64, then the wait)
__device__ __forceinline__ void tm_ld32(uint32_t taddr, double (&d)[32]) {
  uint32_t r[64];
  asm volatile(
      "{\n tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n"
      " tcgen05.wait::ld.sync.aligned;\n}"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]),
        "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]),
        "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
        "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]),
        "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
#pragma unroll
  for (int k = 0; k < 32; ++k) d[k] = __hiloint2double((int)r[2 * k + 1], (int)r[2 * k]);
}
#ifndef KD_TM_CH
#define KD_TM_CH 16  // doubles per TMEM load-and-wait (8, 16 or 32)
#endif
template <int CH>
__device__ __forceinline__ void tm_ldc(uint32_t taddr, double (&d)[CH]) {
  if constexpr (CH == 32) tm_ld32(taddr, d);
  else if constexpr (CH == 16) tm_ld16(taddr, d);
  else tm_ld8(taddr, d);
}

// the same 4-accumulator (off-diagonal) / 2-accumulator (diagonal) orders as rt_dot_*
__device__ __forceinline__ void tm_dot_off(uint32_t taddr, const double* v, double& a0, double& a1, double& a2,
                                           double& a3) {
  const double2* v2 = reinterpret_cast<const double2*>(v);
#pragma unroll
  for (int c0 = 0; c0 < 32; c0 += KD_TM_CH) {
    double t[KD_TM_CH];
    tm_ldc<KD_TM_CH>(taddr + 2 * c0, t);
#pragma unroll
    for (int c = 0; c < KD_TM_CH; c += 4) {
      const double2 p = v2[(c0 + c) / 2], q = v2[(c0 + c) / 2 + 1];
      a0 += t[c] * p.x;
      a1 += t[c + 1] * p.y;
      a2 += t[c + 2] * q.x;
      a3 += t[c + 3] * q.y;
    }
  }
}
__device__ __forceinline__ void tm_dot_diag(uint32_t taddr, const double* v, double& a0, double& a1) {
  const double2* v2 = reinterpret_cast<const double2*>(v);
#pragma unroll
  for (int c0 = 0; c0 < 32; c0 += KD_TM_CH) {
    double t[KD_TM_CH];
    tm_ldc<KD_TM_CH>(taddr + 2 * c0, t);
#pragma unroll
    for (int c = 0; c < KD_TM_CH; c += 2) {
      const double2 p = v2[(c0 + c) / 2];
      a0 += t[c] * p.x;
      a1 += t[c + 1] * p.y;
    }
  }
}

// plan warp wid's TMEM tiles and copy them from X (final, in shared memory)
// into its lane quarter; tbase = the CTA's allocation (512 columns)
__device__ void tm_load(TmTiles& M, uint32_t tbase, const double* X, int n, int T, unsigned long long xmask) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int lo = wid & 3, hi = lo + 4;
  unsigned a1, a2, b1, b2;
  int need_lo, need_hi;
  tm_visits(lo, T, xmask, 8, a1, a2, need_lo);
  tm_visits(hi, T, xmask, 8, b1, b2, need_hi);
  const int bud_lo = min(need_lo, max(4, 8 - need_hi));
  const int bud_hi = min(need_hi, 8 - bud_lo);
  int need;
  tm_visits(wid, T, xmask, wid < 4 ? bud_lo : bud_hi, M.m1, M.m2, need);
  const uint32_t q = tbase + ((uint32_t)(32 * lo) << 16) + (wid < 4 ? 0u : 64u * bud_lo);
  M.c1 = q;
  M.c2 = q + 64u * __popc(M.m1);
  // lane = row (pass 1) / column (pass 2); zeros outside the tile.  All 32
  // values are loaded before the four stores (one shared-memory round trip).
  auto put = [&](uint32_t taddr, int pass, int i, int j) {
    const int ri = tile_rows(i, n);
    double d[4][8];
    if (i == j) {
      const double* D = X + diag_tile(i, n);
      if (pass == 1) {
        const double* row = D + tri(lane);
#pragma unroll
        for (int e = 0; e < 32; ++e) d[e >> 3][e & 7] = (lane < ri && e <= lane) ? row[e] : 0.0;
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) d[e >> 3][e & 7] = (e >= lane && e < ri) ? D[tri(e) + lane] : 0.0;
      }
    } else {
      const double* A = X + off_tile(i, j, n);
      if (pass == 1) {
        const double* row = A + lane * LDT;
#pragma unroll
        for (int e = 0; e < 32; ++e) d[e >> 3][e & 7] = lane < ri ? row[e] : 0.0;
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) d[e >> 3][e & 7] = e < ri ? A[e * LDT + lane] : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) tm_st8(taddr + 16 * q, d[q]);
  };
  int k = 0;
  for (int j = 0; j < T; ++j)
    if ((M.m1 >> j) & 1u) put(M.c1 + 64u * k++, 1, wid, j);
  k = 0;
  for (int i = 0; i < T; ++i)
    if ((M.m2 >> i) & 1u) put(M.c2 + 64u * k++, 2, i, wid);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t tm_addr(uint32_t base, unsigned m, int t) {
  return base + 64u * __popc(m & ((1u << t) - 1u));
}


// unroll of the shared-memory tile walks in the dataflow solve (columns per
// step / 4): fewer loads in flight per warp leave registers for register tiles
#ifndef KD_DF_UNROLL
#define KD_DF_UNROLL 16
#endif
#define KD_PRAGMA_(x) _Pragma(#x)
#define KD_PRAGMA(x) KD_PRAGMA_(x)
#define DF_UNROLL KD_PRAGMA(unroll KD_DF_UNROLL)

// Tile-row readiness of the dataflow solve: a release/acquire flag word per
// tile row, polled by the consumer's lane 0 with a __nanosleep(KD_DF_WAIT)
// backoff (each poll is a shared-memory load competing with the solve passes
// for the pipe; 32 ns measured best of 0/32/200 on DR-Legs, +1 %).
#ifndef KD_DF_WAIT
#define KD_DF_WAIT 32
#endif
__device__ __forceinline__ void df_publish(int* rdy, int i, int epoch) {
  __threadfence_block();
  flag_release(rdy + i, epoch);
}
#ifndef KD_DF_BATCH
#define KD_DF_BATCH 1
#endif
// KD_DF_UNITS: each thread takes the cone unit whose first row sits at its own
// solve position, so a warp's units read the x segment its own pass-2 column
// produced (contacts spanning segments wait on the other columns' flags) and
// the barrier between the solve and the units goes away
#ifndef KD_DF_UNITS
#define KD_DF_UNITS 1
#endif
__device__ __forceinline__ void df_wait(const int* rdy, int i, int epoch) {
  while (flag_acquire(rdy + i) != epoch) {
#if KD_DF_WAIT > 0
    __nanosleep(KD_DF_WAIT);
#endif
  }
}

// inv_solve for T <= NT/32 tile rows with the barrier between the two passes
// replaced by per-tile-row dataflow flags.  Warp i computes tile row i of
// w = X b (pass 1), publishes it (rdy[i] = epoch, release), then runs tile
// column i of x = X^T w (pass 2), consuming w_k for k = i, i+1, ... as each
// is published (acquire).  The passes overlap: warp i's column work starts at
// ~(i+1) tile times instead of after the slowest row (T tile times), so the
// critical path drops from ~2T to ~T+1 tile times.  Every dot product runs in
// the same order as inv_solve's, so the result is bitwise the same; x goes to
// xo (pass 1 may still be reading b when early columns finish).  Tiles in R
// are read from registers.
template <int NT>
__device__ void inv_solve_df(const double* X, const double* b, double* w, double* xo, int n, int T,
                             unsigned long long xmask, int* rdy, int epoch, const RegTiles& R,
                             const TmTiles& M, long long* prof = nullptr) {
  int* crdy = rdy + 8;  // tile-column flags: x segment j final (KD_DF_UNITS)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();  // b complete
  if (wid >= T) return;  // (the caller's barrier after the solve is outside)
#ifdef KD_PROF_WARP
  const long long qd0 = clock64();
  long long qwait = 0;
#endif
  {  // pass 1: tile row wid
    const int i = wid;
    const int ri = tile_rows(i, n), r = lane;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (unsigned mj = M.r1; mj; mj &= mj - 1u) {
      const int j = __ffs(mj) - 1;
      const int k = rt_slot(R, 1, i, j);
      if (k >= 0) {
        RtDispatch<DF_NC>::off(R, k, b + 32 * j, a0, a1, a2, a3);
        continue;
      }
      if (KD_TMEM && ((M.m1 >> j) & 1u)) {
        tm_dot_off(tm_addr(M.c1, M.m1, j), b + 32 * j, a0, a1, a2, a3);
        continue;
      }
      if (r < ri) {
        const double* row = X + off_tile(i, j, n) + r * LDT;
        const double2* bj = reinterpret_cast<const double2*>(b + 32 * j);
DF_UNROLL
        for (int c = 0; c < 32; c += 4) {
          const double2 b01 = bj[c / 2], b23 = bj[c / 2 + 1];
          a0 += row[c] * b01.x;
          a1 += row[c + 1] * b01.y;
          a2 += row[c + 2] * b23.x;
          a3 += row[c + 3] * b23.y;
        }
      }
    }
    {
      const int k = rt_slot(R, 1, i, i);
      if (k >= 0) {
        RtDispatch<DF_NC>::diag(R, k, b + 32 * i, a0, a1);
      } else if (KD_TMEM && ((M.m1 >> i) & 1u)) {
        tm_dot_diag(tm_addr(M.c1, M.m1, i), b + 32 * i, a0, a1);
      } else if (r < ri) {
        const double* drow = X + diag_tile(i, n) + tri(r);
        const double2* bi = reinterpret_cast<const double2*>(b + 32 * i);
DF_UNROLL
        for (int c = 0; c < 32; c += 2) {
          const double2 bb = bi[c / 2];
          if (c <= r) a0 += drow[c] * bb.x;
          if (c + 1 <= r) a1 += drow[c + 1] * bb.y;
        }
      }
    }
    if (r < ri) w[32 * i + r] = (a0 + a1) + (a2 + a3);
    __syncwarp();
    if (lane == 0) df_publish(rdy, i, epoch);
#ifdef KD_PROF_WARP
    if (prof && KD_PROF_WARP == 5) prof[4 + wid] += clock64() - qd0;
#endif
  }
  {  // pass 2: tile column wid, rows consumed as they are published
    const int j = wid;
    const int c = lane, rj = tile_rows(j, n);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    // the diagonal tile needs w_j, which this warp published itself
    {
      const int k = rt_slot(R, 2, j, j);
      if (k >= 0) {
        RtDispatch<DF_NC>::diag(R, k, w + 32 * j, a0, a1);
      } else if (KD_TMEM && ((M.m2 >> j) & 1u)) {
        tm_dot_diag(tm_addr(M.c2, M.m2, j), w + 32 * j, a0, a1);
      } else if (c < rj) {
        const double* D = X + diag_tile(j, n);
        const double2* wj = reinterpret_cast<const double2*>(w + 32 * j);
DF_UNROLL
        for (int r = 0; r < 32; r += 2) {
          const double2 ww = wj[r / 2];
          if (r >= c && r < rj) a0 += D[tri(r) + c] * ww.x;
          if (r + 1 >= c && r + 1 < rj) a1 += D[tri(r + 1) + c] * ww.y;
        }
      }
    }
    unsigned ready = 0u;  // KD_DF_BATCH: bit i = row i seen published (this epoch)
    for (unsigned mi = M.r2; mi; mi &= mi - 1u) {
      const int i = __ffs(mi) - 1;
#ifdef KD_PROF_WARP
      const long long qa = clock64();
#endif
      if (KD_DF_BATCH) {
        // one acquire per lane (lane k polls row k): every row published by
        // now is seen at once, so later rows of the column need no poll
        while (!((ready >> i) & 1u)) {
          const int f = lane < T ? flag_acquire(rdy + lane) : epoch;
          ready = __ballot_sync(0xffffffffu, f == epoch);
          if (!((ready >> i) & 1u)) {
#if KD_DF_WAIT > 0
            __nanosleep(KD_DF_WAIT);
#endif
          }
        }
      } else if (lane == 0) {
        df_wait(rdy, i, epoch);
      }
      __syncwarp();
#ifdef KD_PROF_WARP
      qwait += clock64() - qa;
#endif
      const int k = rt_slot(R, 2, i, j);
      if (k >= 0) {
        RtDispatch<DF_NC>::off(R, k, w + 32 * i, a0, a1, a2, a3);
        continue;
      }
      if (KD_TMEM && ((M.m2 >> i) & 1u)) {
        tm_dot_off(tm_addr(M.c2, M.m2, i), w + 32 * i, a0, a1, a2, a3);
        continue;
      }
      if (c < rj) {
        const int ri = tile_rows(i, n);
        const double* A = X + off_tile(i, j, n) + c;
        const double2* wi = reinterpret_cast<const double2*>(w + 32 * i);
        if (ri == 32) {
DF_UNROLL
          for (int r = 0; r < 32; r += 4) {
            const double2 w01 = wi[r / 2], w23 = wi[r / 2 + 1];
            a0 += A[r * LDT] * w01.x;
            a1 += A[(r + 1) * LDT] * w01.y;
            a2 += A[(r + 2) * LDT] * w23.x;
            a3 += A[(r + 3) * LDT] * w23.y;
          }
        } else {
DF_UNROLL
          for (int r = 0; r < 32; r += 4) {
            const double2 w01 = wi[r / 2], w23 = wi[r / 2 + 1];
            if (r < ri) a0 += A[r * LDT] * w01.x;
            if (r + 1 < ri) a1 += A[(r + 1) * LDT] * w01.y;
            if (r + 2 < ri) a2 += A[(r + 2) * LDT] * w23.x;
            if (r + 3 < ri) a3 += A[(r + 3) * LDT] * w23.y;
          }
        }
      }
    }
    if (c < rj) xo[32 * j + c] = (a0 + a1) + (a2 + a3);
    if (KD_DF_UNITS) {
      __syncwarp();
      if (lane == 0) df_publish(crdy, j, epoch);
    }
  }
#ifdef KD_PROF_WARP
  if (prof && KD_PROF_WARP == 3) prof[4 + wid] += clock64() - qd0;
  if (prof && KD_PROF_WARP == 4) prof[4 + wid] += qwait;
#endif
}

// PADMM loop of the dense kernel for GLOBAL_L worlds (any n): the same
// arithmetic as the register-resident loop of dense_kernel, with every thread
// looping over its cone units (u = tid, tid + NT, ...).  Per-unit state y, z,
// y_hat, z_hat is kept in the world's slab after the factor (4 npad doubles);
// the residual maxima are exact (max is associative), so the loop's results do
// not depend on how units map to threads.
template <int NT>
__device__ void padmm_units_global(const BatchView& bv, const StepParams& sp, int w, WorldStep& ws, const double* L,
                                   double* xv, double* wv_s, double* red, int n, int T, int nlen) {
  const int tid = threadIdx.x;
  const DevWorld W = bv.worlds[w];
  const int64_t R0 = W.row_off;
  const int npad = 32 * T;
  double* ys = const_cast<double*>(L) + ((nlen + 1) & ~1);
  double* zs = ys + npad;
  double* yhs = zs + npad;
  double* zhs = yhs + npad;
  const int n_jd = ws.n_rows - ws.n_limits - 3 * ws.n_contacts;
  const int first_contact = n_jd + ws.n_limits;
  const int n_units = first_contact + ws.n_contacts;
  const double eta = sp.eta, rho = sp.rho, inv_rho = 1.0 / rho;
  const double* vfg = bv.vf + R0;
  const double* rmu = bv.rmu + R0;
  auto unit_rows = [&](int u, int& row0, int& kind, int& nr) {
    row0 = u < first_contact ? u : first_contact + 3 * (u - first_contact);
    kind = u < n_jd ? ROW_BILATERAL : (u < first_contact ? ROW_LIMIT : ROW_CONTACT);
    nr = kind == ROW_CONTACT ? 3 : 1;
  };
  // y = Pi_K(x0); hats; first right-hand side
  for (int u = tid; u < n_units; u += NT) {
    int row0, kind, nr;
    unit_rows(u, row0, kind, nr);
    double x[3] = {0, 0, 0}, y[3] = {0, 0, 0}, z[3] = {0, 0, 0};
    for (int d = 0; d < nr; ++d) {
      x[d] = bv.x0[R0 + row0 + d];
      z[d] = bv.z0[R0 + row0 + d];
    }
    const double mu = rmu[row0];
    if (kind == ROW_CONTACT) project_soc(x, mu, 1.0 / (1.0 + mu * mu), y);
    else y[0] = kind == ROW_LIMIT ? fmax(0.0, x[0]) : x[0];
    const double s0 = kind == ROW_CONTACT ? mu * fast_sqrt(z[1] * z[1] + z[2] * z[2]) : 0.0;
    for (int d = 0; d < nr; ++d) {
      ys[row0 + d] = yhs[row0 + d] = y[d];
      zs[row0 + d] = zhs[row0 + d] = z[d];
      xv[row0 + d] = -((((vfg[row0 + d] + (d == 0 ? s0 : 0.0)) - eta * x[d]) - rho * y[d]) - z[d]);
    }
  }
  double prev = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  double rp = 0.0, dmax = 0.0, rc = 0.0;
  int restarts = 0, it = 1, m = 0;
  bool converged = false;
  const int hcap = bv.hist_cap;
  const unsigned long long xm = ~0ull;
  for (it = 1; it <= sp.max_iters; ++it) {
    inv_solve<NT>(L, xv, wv_s, n, T, xm);  // barriers on entry and exit
    const double beta = sp.acceleration ? sp.nest_beta[m] : 0.0;
    rp = dmax = rc = 0.0;
    for (int u = tid; u < n_units; u += NT) {
      int row0, kind, nr;
      unit_rows(u, row0, kind, nr);
      const double mu = rmu[row0];
      double x[3] = {0, 0, 0}, wv[3] = {0, 0, 0}, yn[3] = {0, 0, 0};
      for (int d = 0; d < nr; ++d) {
        x[d] = xv[row0 + d];
        wv[d] = x[d] - zhs[row0 + d] * inv_rho;
      }
      if (kind == ROW_CONTACT) project_soc(wv, mu, 1.0 / (1.0 + mu * mu), yn);
      else yn[0] = kind == ROW_LIMIT ? fmax(0.0, wv[0]) : wv[0];
      double ymax = 0.0, zmax = 0.0;
      for (int d = 0; d < nr; ++d) {
        const double zn = zhs[row0 + d] - rho * (x[d] - yn[d]);
        rp = fmax(rp, fabs(x[d] - yn[d]));
        dmax = fmax(dmax, fabs(yn[d] - ys[row0 + d]));
        ymax = fmax(ymax, fabs(yn[d]));
        zmax = fmax(zmax, fabs(zn));
        // y_prev / z_prev parked in the hat slots until the Nesterov step
        yhs[row0 + d] = ys[row0 + d];
        zhs[row0 + d] = zs[row0 + d];
        ys[row0 + d] = yn[d];
        zs[row0 + d] = zn;
      }
      if (kind != ROW_BILATERAL) rc = fmax(rc, fmin(ymax, zmax));
    }
    const double combined = block_max_nonneg<NT>(fmax(rp, fmax(rho * dmax, rc)), red);
    if (tid == 0 && it <= hcap) bv.hist[(int64_t)w * hcap + it - 1] = combined;
    if (!sp.fixed_mode && combined < sp.eps) {
      converged = true;
      break;
    }
    bool restart = false;
    if (sp.acceleration) {
      restart = sp.restart && combined > prev;
      if (restart) {
        m = 0;
        ++restarts;
      } else {
        ++m;
      }
    }
    prev = combined;
    for (int u = tid; u < n_units; u += NT) {
      int row0, kind, nr;
      unit_rows(u, row0, kind, nr);
      double zh[3] = {0, 0, 0};
      for (int d = 0; d < nr; ++d) {
        const double yv = ys[row0 + d], zv = zs[row0 + d];
        double yh = yv, zhd = zv;  // restart, or no acceleration
        if (sp.acceleration && !restart) {
          yh = yv + beta * (yv - yhs[row0 + d]);
          zhd = zv + beta * (zv - zhs[row0 + d]);
        }
        yhs[row0 + d] = yh;
        zhs[row0 + d] = zhd;
        zh[d] = zhd;
      }
      const double mu = rmu[row0];
      const double s0 = kind == ROW_CONTACT ? mu * fast_sqrt(zh[1] * zh[1] + zh[2] * zh[2]) : 0.0;
      for (int d = 0; d < nr; ++d)
        xv[row0 + d] = -((((vfg[row0 + d] + (d == 0 ? s0 : 0.0)) - eta * xv[row0 + d]) - rho * yhs[row0 + d]) - zh[d]);
    }
  }
  __syncthreads();  // red is still being read by the last reduction
  block_max3<NT>(rp, dmax, rc, red);
  const double r_p = rp, r_d = rho * dmax, r_c = rc;
  for (int r = tid; r < n; r += NT) {
    bv.lam[R0 + r] = ys[r];
    bv.zo[R0 + r] = zs[r];
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

}  // namespace

// small bins (<= 128 rows, little shared memory) would be register-limited to
// four CTAs per SM at 255 registers: cap them so more worlds stay resident
#ifndef KD_DENSE_MINB64
#define KD_DENSE_MINB64 8
#endif
#ifndef KD_DENSE_MINB128
#define KD_DENSE_MINB128 4
#endif
template <int NT>
constexpr int dense_min_blocks() { return NT <= 64 ? KD_DENSE_MINB64 : (NT <= 128 ? KD_DENSE_MINB128 : 1); }

// One world on one CTA (the body of the dense kernels below).
template <int NT, bool GLOBAL_L>
__device__ __forceinline__ void dense_world(const BatchView& bv, const StepParams& sp, const int w) {
  extern __shared__ __align__(16) double smem[];
  WorldStep& ws = bv.wstep[w];
  // BE_DENSE_SN: the supernodal kernel already factored D in its plan's order
  // (kd_sparse.cu); this CTA forms L^-1 in that order and runs the solves
  const bool handoff = !GLOBAL_L && ws.backend == BE_DENSE_SN;
  if (!handoff && ws.backend != (GLOBAL_L ? BE_DENSE_GLOBAL : BE_DENSE_SMEM)) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = NT / 32;
  const DevWorld W = bv.worlds[w];
  const int n = handoff ? bv.snplan[W.model].S : ws.n_rows;  // hand-off: every planned slot
  const int T = (n + 31) >> 5;
  const int nlen = tile_row_base(T - 1) + (T - 1) * LDT * tile_rows(T - 1, n) + tri(tile_rows(T - 1, n));
  const int npad = 32 * T;
  double* L = GLOBAL_L ? bv.lslab + W.lslab_off : smem;
  double* xv = smem + (GLOBAL_L ? 0 : ((nlen + 1) & ~1));
  double* P = xv + npad;
  double* wv_s = P + npad;         // intermediate w = L^{-1} b
  double* red = wv_s + npad;       // 3 * NW
  int* rbs = reinterpret_cast<int*>(red + 3 * NW + 1);  // 2n body ids
  double* chain = reinterpret_cast<double*>(rbs + 2 * npad);  // 32 doubles: pivot-column broadcast
  int* rdy = reinterpret_cast<int*>(chain + 32);                // 8 tile-row flags of inv_solve_df
  // the dataflow solve (T <= warps) writes x to the P buffer, which is free
  // after the Gram phase (and unused by the hand-off)
  const bool df = !GLOBAL_L && T <= NW && !sp.no_df;
  double* xsol = df ? P : xv;
  __shared__ int fail;
  __shared__ uint32_t tmem_base;  // TMEM allocation of the dataflow solve's tiles
  // TMEM tiles only where one CTA owns the SM (255 registers x 256 threads):
  // a second CTA's tcgen05.alloc would wait for the first one's dealloc
  constexpr bool kTm = KD_TMEM && NT == 256 && !GLOBAL_L;
  const bool tm_on = !sp.no_tmem;  // KD_TMEM=0 at batch creation: tiles from shared memory (same results)
  const int64_t R0 = W.row_off;
  const RowJ* rj = bv.rowj + R0;
  const int32_t* rb = bv.rbody + 2 * R0;
  const double* regg = bv.reg + R0;
  const double eta_rho = sp.eta_rho;

  long long t_prev = clock64();
  auto stamp = [&](int k) {
    if (tid == 0) {
      const long long t = clock64();
      ws.phase_cycles[k] = t - t_prev;
      t_prev = t;
    }
  };
  if (tid == 0) fail = 0;
  if (tid < 16) rdy[tid] = 0;  // 8 tile-row + 8 tile-column flags
  if (handoff) {  // rbs holds the row -> plan position map; b is zero at unused positions
    for (int r = tid; r < ws.n_rows; r += NT) rbs[r] = bv.sn_r2p[W.snr2p_off + r];
    for (int r = tid; r < npad; r += NT) xv[r] = 0.0;
  } else {
    for (int r = tid; r < n; r += NT) {
      P[r] = bv.scale[R0 + r];
      rbs[2 * r] = rb[2 * r];
      rbs[2 * r + 1] = rb[2 * r + 1];
    }
  }
  for (int e = tid; e < nlen; e += NT) L[e] = 0.0;
  __syncthreads();
#ifdef KD_PROF_HO
  const long long h0 = clock64();
#endif
  if (handoff) {
    // scatter the supernode panels into the tile layout (the plan's flat list
    // of (Lv index, tile index) pairs), then invert the diagonal tiles
    const DevSnPlan SP = bv.snplan[W.model];
    const double* lv = bv.sn_lv + W.snlv_off;
    const uint32_t* sc = bv.sn_scat + SP.scat_off;
    // eight entries per thread and pass: all index loads, then all value loads,
    // then the stores (the two dependent L2 round trips overlap across entries)
    for (int e0 = tid; e0 < SP.n_scat; e0 += 8 * NT) {
      uint32_t q[8];
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) q[k] = e0 + k * NT < SP.n_scat ? __ldg(sc + e0 + k * NT) : 0xffffffffu;
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = q[k] != 0xffffffffu ? lv[q[k] & 0xffff] : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (q[k] != 0xffffffffu) L[q[k] >> 16] = v[k];
    }
    __syncthreads();
#ifdef KD_PROF_HO
    const long long h1 = clock64();
#endif
    for (int k = wid; k < T; k += NW) diag_invert_rinv(L + diag_tile(k, n), tile_rows(k, n), lane);
    __syncthreads();
#ifdef KD_PROF_HO
    if (tid == 0) {
      ws.phase_cycles[5] = h0 - t_prev;  // kernel start -> zero fill done
      ws.phase_cycles[6] = h1 - h0;      // scatter
      ws.phase_cycles[7] = clock64() - h1;  // diagonal inverses
    }
#endif
    stamp(0);
    stamp(2);
  } else {

  // ---- 1. D = P (J M^-1 J^T + R) P + (eta+rho) I  (assemble_dense, delassus.cpp:67-104)
  // One warp per body b walks the Gram block of the rows touching b
  // (ascending row order).  Element (i, j) is produced once, by the warp of
  // its smallest shared body: g_b1 (registers/shuffles) + g_b2 (the other
  // shared body's blocks, from L1) in ascending body order, then + R on the
  // diagonal, P-scaled and + (eta+rho) on the diagonal.  No atomics, no second
  // pass; elements without a shared body keep the zero fill.
  {
    const int nb = W.nb;
    const int32_t* cptr = bv.csr_ptr + W.body_off + w;
    const int32_t* clist = bv.csr + 2 * R0;
    for (int b = wid; b < nb; b += NW) {
      const int beg = cptr[b], end = cptr[b + 1];
      for (int pc = beg; pc < end; pc += 32) {
        const int p = pc + lane;
        double gm[6];
        int ip = -1, sp_ = 0, a0 = -1, a1 = -1;
        if (p < end) {
          const int e = clist[p];
          ip = e >> 1;
          sp_ = e & 1;
          const double* jm = rj[ip].JM + 6 * sp_;
#pragma unroll
          for (int k = 0; k < 6; ++k) gm[k] = jm[k];
          a0 = rbs[2 * ip];
          a1 = rbs[2 * ip + 1];
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
          const int qn = min(32, end - qc);
          for (int qq = 0; qq < qn; ++qq) {
            const int jrow = __shfl_sync(FULL, iq, qq);
            double gq[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) gq[k] = __shfl_sync(FULL, g[k], qq);
            if (ip < 0 || jrow > ip) continue;  // lower triangle, rows ascending
            const int c0 = rbs[2 * jrow], c1 = rbs[2 * jrow + 1];
            const int other = sp_ == 0 ? a1 : a0;  // row ip's other body (b is this side)
            const bool two = other >= 0 && (other == c0 || other == c1);
            if (two && other < b) continue;  // the smaller shared body's warp owns (i, j)
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) s += gm[k] * gq[k];
            if (two) {
              const double* jm2 = rj[ip].JM + 6 * (1 - sp_);
              const double* jj2 = rj[jrow].J + 6 * (c0 == other ? 0 : 1);
              double s2 = 0.0;
#pragma unroll
              for (int k = 0; k < 6; ++k) s2 += jm2[k] * jj2[k];
              s += s2;
            }
            if (ip == jrow) s += regg[ip];
            double d = (P[ip] * s) * P[jrow];
            if (ip == jrow) d += eta_rho;
            L[lidx(ip, jrow, n)] = d;
          }
        }
      }
    }
  }
  __syncthreads();
  stamp(0);
  // ---- 2. blocked right-looking Cholesky with look-ahead; diagonal tiles
  // become L_kk^{-1}.  While warps 1.. run the trailing update of step k,
  // warp 0 updates and factors diagonal tile k+1 (the critical path).
  long long c_panel = 0, c_syrk = 0, c_diag = 0;
  for (int k = -1; k < T; ++k) {
    long long q0 = clock64();
    if (k >= 0) {
      for (int i = k + 1 + wid; i < T; i += NW) panel_tile(L, i, k, n);
      __syncthreads();
    }
    long long q1 = clock64();
    c_panel += q1 - q0;
    if (k + 1 < T) {
      const int m = T - k - 1;
      const int units = k >= 0 ? m * (m + 1) / 2 : 0;
      if (wid == 0) {
        if (k >= 0) {
          syrk_tile(L, k + 1, k + 1, k, n, lane);
          __syncwarp();
        }
        diag_factor_invert(L + diag_tile(k + 1, n), tile_rows(k + 1, n), lane, &fail, chain);
        c_diag += clock64() - q1;
      } else {
        for (int u = wid; u < units; u += NW - 1) {  // unit 0, tile (k+1, k+1), is warp 0's
          int ii = 0;
          while ((ii + 1) * (ii + 2) / 2 <= u) ++ii;
          const int jj = u - ii * (ii + 1) / 2;
          syrk_tile(L, k + 1 + ii, k + 1 + jj, k, n, lane);
        }
      }
      __syncthreads();
      c_syrk += clock64() - q1;
    }
  }
  if (tid == 0) {
    ws.phase_cycles[5] = c_panel;
    ws.phase_cycles[6] = c_syrk;
    ws.phase_cycles[7] = c_diag;
  }
  if (fail) {
    if (tid == 0) {
      ws.fail = 1;
      atomicAdd(bv.error_count, 1);
    }
  }
  stamp(2);
  }  // !handoff
  // ---- 2b. X = L^{-1}: every PADMM solve becomes two parallel mat-vecs
  unsigned long long xm = ~0ull;
  {
    unsigned long long lm = ~0ull;
    if (handoff) {
      const DevSnPlan& SP = bv.snplan[W.model];
      lm = ((unsigned long long)(uint32_t)SP.lmask_hi << 32) | (uint32_t)SP.lmask_lo;
      xm = ((unsigned long long)(uint32_t)SP.xmask_hi << 32) | (uint32_t)SP.xmask_lo;
    }
#ifdef KD_PROF_INV
    tri_inverse<NT>(L, n, T, lm, xm, handoff ? bv.sn_kmask + bv.snplan[W.model].kmask_off : nullptr,
                    reinterpret_cast<long long*>(ws.phase_cycles));
#else
    tri_inverse<NT>(L, n, T, lm, xm, handoff ? bv.sn_kmask + bv.snplan[W.model].kmask_off : nullptr);
#endif
  }
  stamp(3);

  if constexpr (!GLOBAL_L) {
    if (handoff && W.xslab_off >= 0) {
      // K2c (kd_dense_cl.cu) runs this world's PADMM on a CTA pair: X's
      // nonzero tiles go to the world's slab in row-major tile order
      // (off-diagonal tiles 32 x LDT, diagonal tiles packed, 528 doubles each)
      double* dst = bv.xslab + W.xslab_off;
      int64_t off = 0;
      for (int i = 0; i < T; ++i)
        for (int j = 0; j <= i; ++j) {
          if (!mtile(xm, i, j)) continue;
          const int ri = tile_rows(i, n);
          const double* src = L + (i == j ? diag_tile(i, n) : off_tile(i, j, n));
          const int len = i == j ? tri(ri) : ri * LDT;
          for (int e = tid; e < len; e += NT) dst[off + e] = src[e];
          off += i == j ? 528 : 32 * LDT;
        }
      stamp(4);
      return;
    }
  }

  if constexpr (GLOBAL_L) {
    // ---- 3'. PADMM (padmm.cpp:87-159) for worlds of any size: thread t owns
    // cone units t, t + NT, ...; y, z, y_hat, z_hat live in the world's HBM
    // slab after the factor (L2-resident), the solve vector in shared memory.
    padmm_units_global<NT>(bv, sp, w, ws, L, xv, wv_s, red, n, T, nlen);
    stamp(4);
    return;
  } else {
  // ---- 3. PADMM (padmm.cpp:87-159), one cone unit per thread
  const int n_jd = ws.n_rows - ws.n_limits - 3 * ws.n_contacts;
  const int first_contact = n_jd + ws.n_limits;
  const int n_units = first_contact + ws.n_contacts;
  // this thread's cone unit: unit tid, or (KD_DF_UNITS, dataflow solve) the
  // unit whose first row sits at solve position tid (npad <= NT); the units'
  // arithmetic does not depend on the assignment
  int uix = tid;
  if (KD_DF_UNITS && df) {
    int* uat = reinterpret_cast<int*>(wv_s);  // npad ints; wv_s is free before the first solve
    for (int p = tid; p < npad; p += NT) uat[p] = -1;
    __syncthreads();
    for (int u = tid; u < n_units; u += NT) {
      const int r0 = u < first_contact ? u : first_contact + 3 * (u - first_contact);
      uat[handoff ? rbs[r0] : r0] = u;
    }
    __syncthreads();
    uix = tid < npad ? uat[tid] : -1;
    __syncthreads();
  }
  const bool has_unit = uix >= 0 && uix < n_units;
  const int row0 = !has_unit ? 0 : (uix < first_contact ? uix : first_contact + 3 * (uix - first_contact));
  const int kind = !has_unit ? ROW_BILATERAL : (uix < n_jd ? ROW_BILATERAL : (uix < first_contact ? ROW_LIMIT : ROW_CONTACT));
  const int nr = !has_unit ? 0 : (kind == ROW_CONTACT ? 3 : 1);
  const double mu = has_unit ? bv.rmu[R0 + row0] : 0.0;
  int pos[3] = {row0, row0 + 1, row0 + 2};  // the unit's rows in the solve's order
  if (handoff) {
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d < nr) pos[d] = rbs[row0 + d];
  }
  const double inv_1pmu2 = 1.0 / (1.0 + mu * mu);
  const double eta = sp.eta, rho = sp.rho;
  const double inv_rho = 1.0 / rho;  // w = x - z_hat / rho as x - z_hat * (1/rho): no division in the loop
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
  if (kind == ROW_CONTACT) project_soc(x, mu, inv_1pmu2, y);
  else if (kind == ROW_LIMIT) y[0] = fmax(0.0, x[0]);
  else y[0] = x[0];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    yh[d] = y[d];
    zh[d] = z[d];
  }
  double prev = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  double rp = 0.0, dmax = 0.0, rc = 0.0;  // this thread's last-iteration residual terms
  int restarts = 0, it = 1, m = 0;          // m: Nesterov updates since the last restart (a = a_m)
  bool converged = false;
  const int hcap = bv.hist_cap;
  // rhs = -(v_f + s - eta x - rho y_hat - z_hat)   (padmm.cpp:116-117)
  auto write_rhs = [&]() {
    const double s0 = kind == ROW_CONTACT ? mu * fast_sqrt(zh[1] * zh[1] + zh[2] * zh[2]) : 0.0;  // desaxce_shift (padmm.cpp:44-52)
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d < nr) xv[pos[d]] = -((((v[d] + (d == 0 ? s0 : 0.0)) - eta * x[d]) - rho * yh[d]) - zh[d]);
  };
  write_rhs();
  RegTiles rtiles;
  TmTiles mtiles{0u, 0u, 0u, 0u, 0u, 0u};
#ifdef KD_PROF_PADMM
  const long long q_setup = clock64();
#endif
  if (df) {
    rt_load(rtiles, L, n, T, xm);
    df_masks(mtiles, T, xm);
    if (kTm && tm_on) {
      if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#ifdef KD_PROF_TM
      const long long q_alloc = clock64();
#endif
      tm_load(mtiles, tmem_base, L, n, T, xm);
#ifdef KD_PROF_TM
      if (lane == 0) ws.phase_cycles[wid] = clock64() - q_alloc;
#endif
    }
#if defined(KD_PROF_PADMM) && !defined(KD_PROF_TM)
    __syncthreads();
    if (tid == 0) ws.phase_cycles[2] = clock64() - q_setup;
#endif
    // register tiles multiply whole 32-entry vector segments (zeros in the
    // tile beyond row/column n): the padding of b and w must hold finite values
    for (int r = n + tid; r < npad; r += NT) xv[r] = wv_s[r] = 0.0;
  }
#ifdef KD_PROF_WARP
  long long prof[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#else
  long long prof[4] = {0, 0, 0, 0};
#endif
  for (it = 1; it <= sp.max_iters; ++it) {
#ifdef KD_PROF_PADMM
    const long long p0 = clock64();
#endif
#ifdef KD_PROF_WARP
    long long qu0 = clock64();
#endif
    if (df) {
      inv_solve_df<NT>(L, xv, wv_s, xsol, n, T, xm, rdy, it, rtiles, mtiles, prof);
      if (KD_DF_UNITS) {
        // the x segments this warp's units read: its own column (published by
        // this warp) and, for contacts spanning segments, other columns
        unsigned need = 0u;
#pragma unroll
        for (int d = 0; d < 3; ++d)
          if (d < nr) need |= 1u << (pos[d] >> 5);
        need = __reduce_or_sync(0xffffffffu, need) & ~(1u << wid);
        unsigned ready = 0u;
        while ((ready & need) != need) {
          const int f = lane < T ? flag_acquire(rdy + 8 + lane) : it;
          ready = __ballot_sync(0xffffffffu, f == it);
#if KD_DF_WAIT > 0
          if ((ready & need) != need) __nanosleep(KD_DF_WAIT);
#endif
        }
        __syncwarp();
      } else {
        __syncthreads();  // x complete
      }
#ifdef KD_PROF_WARP
      qu0 = clock64();
#endif
    } else {
      inv_solve<NT>(L, xv, wv_s, n, T, xm, prof);
    }
#ifdef KD_PROF_PADMM
    const long long p1 = clock64();
#endif
    // beta_m of the Nesterov sequence (host table), fetched before the reduction
    const double beta = sp.acceleration ? sp.nest_beta[m] : 0.0;
    double yp[3], zp[3], wv[3], yn[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (d < nr) x[d] = xsol[pos[d]];
      wv[d] = x[d] - zh[d] * inv_rho;
      yp[d] = y[d];
      zp[d] = z[d];
    }
    if (kind == ROW_CONTACT) project_soc(wv, mu, inv_1pmu2, yn);
    else {
      yn[0] = kind == ROW_LIMIT ? fmax(0.0, wv[0]) : wv[0];
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
    // max(r_p, r_d, r_c) (padmm.cpp:128-131) in one reduction: rho > 0, so
    // max(rho * dmax_i) = rho * max(dmax_i) exactly
#ifdef KD_PROF_WARP
    const long long qu1 = clock64();
    if (KD_PROF_WARP == 6) prof[4 + wid] += qu1 - qu0;
#endif
    const double combined = block_max_nonneg<NT>(fmax(rp, fmax(rho * dmax, rc)), red);
#ifdef KD_PROF_WARP
    if (KD_PROF_WARP == 7) prof[4 + wid] += clock64() - qu1;
#endif
#ifdef KD_PROF_PADMM
    const long long p2 = clock64();
    prof[2] += p2 - p1;
    prof[3] += p1 - p0;  // whole solve incl. entry barrier
#endif
    if (tid == 0 && it <= hcap) bv.hist[(int64_t)w * hcap + it - 1] = combined;
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
    write_rhs();
  }
  // the last iteration's r_p, r_d, r_c (padmm.cpp:147-157)
  if (kTm && tm_on && df) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();  // red is still being read by the last reduction (and TMEM reads are done)
  if (kTm && tm_on && df && wid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
  block_max3<NT>(rp, dmax, rc, red);
  const double r_p = rp, r_d = rho * dmax, r_c = rc;
  stamp(4);
#ifdef KD_PROF_WARP
  if (lane == 0) ws.phase_cycles[wid] = prof[4 + wid];
#endif
#ifdef KD_PROF_PADMM
  if (tid == 0) {
    ws.phase_cycles[5] = prof[0];
    ws.phase_cycles[6] = prof[1];
    ws.phase_cycles[7] = prof[2];
    ws.phase_cycles[1] = prof[3];
  }
#endif
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
  }  // !GLOBAL_L
}

template <int NT, bool GLOBAL_L>
__global__ void __launch_bounds__(NT, dense_min_blocks<NT>()) dense_kernel(BatchView bv, StepParams sp, const int32_t* bin_worlds) {
  dense_world<NT, GLOBAL_L>(bv, sp, bin_worlds[blockIdx.x]);
}

// The HBM-slab bin of planned models is a rare fallback (K1 sends a world
// there only when an active contact has no planned slot): instead of one
// mostly empty CTA per world (one CTA per SM at 255 registers, ~15 us per
// part and step), each CTA tests 256 worlds' backends at once and runs the
// few that chose the slab one after another.
__global__ void __launch_bounds__(256, 1) dense_global_sweep(BatchView bv, StepParams sp, const int32_t* bin_worlds,
                                                             int count) {
  __shared__ int hits[256];
  __shared__ int nhit;
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (threadIdx.x == 0) nhit = 0;
  __syncthreads();
  if (i < count) {
    const int w = bin_worlds[i];
    if (bv.wstep[w].backend == BE_DENSE_GLOBAL) hits[atomicAdd(&nhit, 1)] = w;
  }
  __syncthreads();
  const int m = nhit;
  for (int k = 0; k < m; ++k) {
    dense_world<256, true>(bv, sp, hits[k]);
    __syncthreads();  // the world's shared memory is reused by the next one
  }
}

// Shared-memory bytes the dense kernel needs for n rows with NT threads.
size_t dense_factor_doubles(int n) {
  const int T = (n + 31) / 32;
  const int rl = n - 32 * (T - 1);
  return (size_t)528 * (T - 1) * (T - 1) + (size_t)(T - 1) * 33 * rl + (size_t)rl * (rl + 1) / 2;
}

size_t dense_smem_bytes(int n, int nt, bool global_l) {
  const int T = (n + 31) / 32;
  const int rl = n - 32 * (T - 1);
  const size_t nl = (size_t)528 * (T - 1) * (T - 1) + (size_t)(T - 1) * 33 * rl + (size_t)rl * (rl + 1) / 2;
  const size_t nlen = global_l ? 0 : ((nl + 1) & ~(size_t)1);
  const size_t npad = 32 * (size_t)T;
  return 8 * (nlen + 3 * npad + 3 * (nt / 32) + 1) + 4 * 2 * npad + 8 * 32 + 64 + 64;  // + 16 flag words
}

template <int NT, bool G>
static cudaError_t launch_t(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, int cap,
                            cudaStream_t s) {
  const size_t smem = dense_smem_bytes(cap, NT, G);
  static SmemAttrCache attr;
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(dense_kernel<NT, G>), smem, attr);
    if (e != cudaSuccess) return e;
  }
  dense_kernel<NT, G><<<count, NT, smem, s>>>(bv, sp, worlds);
  return cudaGetLastError();
}

cudaError_t launch_dense_global_sweep(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count,
                                     int cap, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const size_t smem = dense_smem_bytes(cap, 256, true);
  static SmemAttrCache attr;
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(dense_global_sweep), smem, attr);
    if (e != cudaSuccess) return e;
  }
  dense_global_sweep<<<(count + 255) / 256, 256, smem, s>>>(bv, sp, worlds, count);
  return cudaGetLastError();
}

cudaError_t launch_dense(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, int cap, int nt,
                         bool global_l, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  if (global_l) return launch_t<256, true>(bv, sp, worlds, count, cap, s);
  switch (nt) {
    case 64: return launch_t<64, false>(bv, sp, worlds, count, cap, s);
    case 128: return launch_t<128, false>(bv, sp, worlds, count, cap, s);
    case 256: return launch_t<256, false>(bv, sp, worlds, count, cap, s);
    default: return launch_t<256, false>(bv, sp, worlds, count, cap, s);
  }
}

}  // namespace kd
