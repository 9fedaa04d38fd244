// kd_fk.cu — batched forward kinematics on the device (
// environment resets with randomised joint targets, PAPER §5.3).
//
// Restates fk_solve (fk.cpp:64-106) per world, one CTA per world:
//   r = [bilateral f; coordinate - target]  (fk_residual, fk.cpp:9-24; revolute
//       differences wrapped with remainder(d, 2 pi));
//   J = bilateral rows + coordinate-rate rows with the angular blocks
//       post-multiplied by R_b (local chart, fk_jacobian, fk.cpp:28-52);
//   (J^T J + lm I) delta = -J^T r;  candidate q <- q exp(delta/2) normalised
//       (apply_update, fk.cpp:54-62); accept if |r| decreases (lm / 10,
//       floored at 1e-12), else lm x 10 and stop above 1e10.
// The normal matrix (6 nb)^2 is assembled block by block from the rows that
// couple two bodies (ascending row order) and factored by a right-looking
// Cholesky in shared memory; the reference uses Eigen's LDLT, so agreement is
// to rounding (the oracle, oracle/oracle.cpp fk_solve, uses an LLT too).
// Poses are read from and written back to the batch's device state.
#include "kd_device.cuh"
#include "kd_joint.cuh"

namespace kd {

namespace {

constexpr int kFkThreads = 256;

template <int NT>
__device__ __forceinline__ double block_reduce(double v, double* red, bool is_max) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = is_max ? warp_max(v) : warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  const double x = lane < NT / 32 ? red[lane] : 0.0;
  return is_max ? warp_max(x) : warp_sum(x);
}

struct FkRows {
  double* J;    // 12 per row (world frame; angular blocks converted to the local chart)
  int32_t* rb;  // 2 per row
  double* r;    // residual per row
};

}  // namespace

__global__ void __launch_bounds__(kFkThreads, 1) fk_kernel(BatchView bv, const int32_t* tj, const double* tv, int nt,
                                                           double tol, int max_iters, double lm0, int32_t* out_iters,
                                                           double* out_res, uint8_t* out_conv, double* gscratch,
                                                           int64_t scratch_doubles) {
  extern __shared__ __align__(16) double smem_[];
  // models whose normal matrix does not fit one CTA's shared memory work in a
  // per-world HBM scratch slab instead (same layout, same arithmetic)
  double* smem = gscratch ? gscratch + (int64_t)blockIdx.x * scratch_doubles : smem_;
  constexpr int NT = kFkThreads;
  const int w = blockIdx.x, tid = threadIdx.x;
  if (!bv.active[w]) {
    if (tid == 0) out_iters[w] = 0, out_res[w] = 0.0, out_conv[w] = 1;
    return;
  }
  const DevWorld W = bv.worlds[w];
  const DevModel M = bv.models[W.model];
  const DevJoint* mj = bv.joints + M.joint_off;
  const int nb = M.nb, nc = 6 * nb, nf = M.n_bil, nr = nf + nt;
  double* pose = bv.poses + W.pose_off;
  BodyS* bs = bv.bs + W.body_off;  // per-step scratch, free between steps
  const int32_t* wj = tj + (int64_t)w * nt;
  const double* wv = tv + (int64_t)w * nt;
  // shared layout
  double* N = smem;                                  // nc (nc + 1) / 2, packed lower
  double* g = N + nc * (nc + 1) / 2;                 // nc (rhs, then delta)
  double* Pc = g + nc;                               // 7 nb: current poses
  double* Pn = Pc + 7 * nb;                          // 7 nb: candidate poses
  double* rows = Pn + 7 * nb;                        // 2 x (13 nr): J + r, current / candidate
  double* red = rows + 2 * 13 * nr;                  // 32
  int32_t* rbi = reinterpret_cast<int32_t*>(red + 32);  // 2 x 2 nr
  FkRows cur{rows, rbi, rows + 12 * nr}, cand{rows + 13 * nr, rbi + 2 * nr, rows + 13 * nr + 12 * nr};

  for (int e = tid; e < 7 * nb; e += NT) Pc[e] = pose[e];
  __syncthreads();

  // rows and residual at poses P (fk_residual + fk_jacobian)
  auto evaluate = [&](const double* P, FkRows& o) {
    for (int b = tid; b < nb; b += NT) {
      BodyS& B = bs[b];
      const Q4 q{P[7 * b + 3], P[7 * b + 4], P[7 * b + 5], P[7 * b + 6]};
      B.ep[0] = P[7 * b], B.ep[1] = P[7 * b + 1], B.ep[2] = P[7 * b + 2];
      B.eq[0] = q.w, B.eq[1] = q.x, B.eq[2] = q.y, B.eq[3] = q.z;
      stm(B.eR, qrot(q));
    }
    __syncthreads();
    auto local = [&](int row, int side, int body, V3 lin, V3 ang) {
      double* J = o.J + 12 * row + 6 * side;
      J[0] = lin.x, J[1] = lin.y, J[2] = lin.z;
      if (body < 0) {
        J[3] = J[4] = J[5] = 0.0;
        return;
      }
      const M3 R = ldm(bs[body].eR);  // row vector x R_b
      J[3] = ang.x * R.m[0] + ang.y * R.m[3] + ang.z * R.m[6];
      J[4] = ang.x * R.m[1] + ang.y * R.m[4] + ang.z * R.m[7];
      J[5] = ang.x * R.m[2] + ang.y * R.m[5] + ang.z * R.m[8];
    };
    for (int ji = tid; ji < M.nj; ji += NT) {
      const DevJoint j = mj[ji];
      const Frames fr = joint_frames(j, bs);
      int r = j.row_offset;
      const V3 z3{0, 0, 0};
      joint_bilateral_rows(j, fr, bs, [&](V3 al, V3 aa, V3 bl, V3 bang, double fval) {
        local(r, 0, j.child, al, aa);
        local(r, 1, j.parent, j.parent >= 0 ? bl : z3, j.parent >= 0 ? bang : z3);
        o.rb[2 * r] = j.child;
        o.rb[2 * r + 1] = j.parent;
        o.r[r] = fval;
        ++r;
      });
    }
    for (int k = tid; k < nt; k += NT) {
      const DevJoint j = mj[wj[k]];
      const Frames fr = joint_frames(j, bs);
      V3 al, aa, bl, bang;
      rate_row(j, fr, bs, al, aa, bl, bang);
      const int r = nf + k;
      local(r, 0, j.child, al, aa);
      local(r, 1, j.parent, bl, bang);
      o.rb[2 * r] = j.child;
      o.rb[2 * r + 1] = j.parent;
      double d = joint_coord(j, fr) - wv[k];
      if (j.type == J_REVOLUTE) d = remainder(d, 2.0 * 3.14159265358979323846);
      o.r[r] = d;
    }
    __syncthreads();
  };
  auto norms = [&](const FkRows& o, double& n2, double& ninf) {
    double s = 0.0, m = 0.0;
    for (int r = tid; r < nr; r += NT) {
      s += o.r[r] * o.r[r];
      m = fmax(m, fabs(o.r[r]));
    }
    n2 = sqrt(block_reduce<NT>(s, red, false));
    ninf = block_reduce<NT>(m, red, true);
  };

  evaluate(Pc, cur);
  double r_norm, r_inf;
  norms(cur, r_norm, r_inf);
  int iters = 0;
  bool conv = r_inf < tol;
  double lm = lm0;
  for (int iter = 0; iter < max_iters && !conv; ++iter) {
    iters = iter + 1;
    // ---- N = J^T J + lm I (packed lower), g = -J^T r; entry (p, q) sums the
    // rows touching both bodies in ascending row order
    for (int e = tid; e < nc * (nc + 1) / 2; e += NT) {
      int p = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while ((p + 1) * (p + 2) / 2 <= e) ++p;
      while (p * (p + 1) / 2 > e) --p;
      const int q = e - p * (p + 1) / 2;
      const int bp = p / 6, kp = p - 6 * bp, bq = q / 6, kq = q - 6 * bq;
      double s = 0.0;
      for (int r = 0; r < nr; ++r) {
        const int a = cur.rb[2 * r], b = cur.rb[2 * r + 1];
        const int sp_ = a == bp ? 0 : (b == bp ? 1 : -1);
        const int sq = a == bq ? 0 : (b == bq ? 1 : -1);
        if (sp_ < 0 || sq < 0) continue;
        s += cur.J[12 * r + 6 * sp_ + kp] * cur.J[12 * r + 6 * sq + kq];
      }
      N[e] = p == q ? s + lm : s;
    }
    for (int p = tid; p < nc; p += NT) {
      const int bp = p / 6, kp = p - 6 * bp;
      double s = 0.0;
      for (int r = 0; r < nr; ++r) {
        const int a = cur.rb[2 * r], b = cur.rb[2 * r + 1];
        const int sp_ = a == bp ? 0 : (b == bp ? 1 : -1);
        if (sp_ < 0) continue;
        s += cur.J[12 * r + 6 * sp_ + kp] * cur.r[r];
      }
      g[p] = -s;
    }
    __syncthreads();
    // ---- right-looking Cholesky of N, then L y = g, L^T delta = y
    bool spd = true;
    for (int c = 0; c < nc; ++c) {
      const int cc = c * (c + 1) / 2 + c;
      const double d = N[cc];
      if (!(d > 0.0)) spd = false;
      const double l = sqrt(d);
      __syncthreads();
      for (int i = c + 1 + tid; i < nc; i += NT) N[i * (i + 1) / 2 + c] /= l;
      if (tid == 0) N[cc] = l;
      __syncthreads();
      const int m = nc - c - 1;
      for (int e = tid; e < m * (m + 1) / 2; e += NT) {
        int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
        while ((i + 1) * (i + 2) / 2 <= e) ++i;
        while (i * (i + 1) / 2 > e) --i;
        const int j = e - i * (i + 1) / 2;
        const int I = c + 1 + i, Jc = c + 1 + j;
        N[I * (I + 1) / 2 + Jc] -= N[I * (I + 1) / 2 + c] * N[Jc * (Jc + 1) / 2 + c];
      }
      __syncthreads();
    }
    if (!spd) break;
    for (int c = 0; c < nc; ++c) {  // forward, column oriented
      const double y = g[c] / N[c * (c + 1) / 2 + c];
      __syncthreads();
      if (tid == 0) g[c] = y;
      for (int i = c + 1 + tid; i < nc; i += NT) g[i] -= N[i * (i + 1) / 2 + c] * y;
      __syncthreads();
    }
    for (int c = nc - 1; c >= 0; --c) {  // backward
      const double x = g[c] / N[c * (c + 1) / 2 + c];
      __syncthreads();
      if (tid == 0) g[c] = x;
      for (int i = tid; i < c; i += NT) g[i] -= N[c * (c + 1) / 2 + i] * x;
      __syncthreads();
    }
    // ---- candidate poses (apply_update) and their residual
    for (int b = tid; b < nb; b += NT) {
      const double* d = g + 6 * b;
      Pn[7 * b] = Pc[7 * b] + d[0];
      Pn[7 * b + 1] = Pc[7 * b + 1] + d[1];
      Pn[7 * b + 2] = Pc[7 * b + 2] + d[2];
      const Q4 q{Pc[7 * b + 3], Pc[7 * b + 4], Pc[7 * b + 5], Pc[7 * b + 6]};
      Q4 o = qmul(q, quat_exp(V3{0.5 * d[3], 0.5 * d[4], 0.5 * d[5]}));
      o = qnormalized(o);
      Pn[7 * b + 3] = o.w, Pn[7 * b + 4] = o.x, Pn[7 * b + 5] = o.y, Pn[7 * b + 6] = o.z;
    }
    __syncthreads();
    evaluate(Pn, cand);
    double cn, cinf;
    norms(cand, cn, cinf);
    if (cn < r_norm) {
      for (int e = tid; e < 7 * nb; e += NT) Pc[e] = Pn[e];
      const FkRows t = cur;
      cur = cand;
      cand = t;
      r_norm = cn;
      r_inf = cinf;
      lm = fmax(lm / 10.0, 1e-12);
      __syncthreads();
      if (r_inf < tol) conv = true;
    } else {
      lm *= 10.0;
      if (lm > 1e10) break;  // stuck; report the best iterate
    }
  }
  for (int e = tid; e < 7 * nb; e += NT) pose[e] = Pc[e];
  if (tid == 0) {
    out_iters[w] = iters;
    out_res[w] = r_inf;
    out_conv[w] = r_inf < tol ? 1 : 0;
  }
}

size_t fk_smem_bytes(int nb, int nr) {
  const size_t nc = 6 * (size_t)nb;
  return 8 * (nc * (nc + 1) / 2 + nc + 14 * (size_t)nb + 26 * (size_t)nr + 32) + 4 * 4 * (size_t)nr + 64;
}

cudaError_t launch_fk(const BatchView& bv, const int32_t* tj, const double* tv, int nt, double tol, int max_iters,
                      double lm0, int32_t* iters, double* res, uint8_t* conv, size_t smem, cudaStream_t s,
                      double* gscratch) {
  if (bv.n_worlds <= 0) return cudaSuccess;
  if (gscratch) {
    fk_kernel<<<bv.n_worlds, kFkThreads, 0, s>>>(bv, tj, tv, nt, tol, max_iters, lm0, iters, res, conv, gscratch,
                                                 (int64_t)((smem + 15) / 16 * 2));
    return cudaGetLastError();
  }
  static SmemAttrCache attr;
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(fk_kernel), smem, attr);
    if (e != cudaSuccess) return e;
  }
  fk_kernel<<<bv.n_worlds, kFkThreads, smem, s>>>(bv, tj, tv, nt, tol, max_iters, lm0, iters, res, conv, nullptr, 0);
  return cudaGetLastError();
}

}  // namespace kd
