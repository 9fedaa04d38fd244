// kd_cr.cu — K2b: fused PADMM + warm-started matrix-free Conjugate Residual,
// one CTA per world (worlds with n > 300 under Auto, or backend = sparse).
//
// Restates MatrixFreeDelassus::apply (delassus.cpp:106-122) with the baked rows
// of bake_jacobian (130-154) recomputed on the fly (ja = p J, jma = fold(ja):
// the same floating-point operations, half the bytes), cr_solve (156-187) with
// the fixed budget and breakdown guard, DelassusBackend::solve accounting
// (189-197), and the PADMM loop of padmm.cpp:87-159.
// The scatter J^T v runs per body over its ascending row list (the reference's
// accumulation order); dot products use a fixed-order block reduction, so the
// result is deterministic run to run.  All n-vectors and the per-body scratch
// live in shared memory; Jacobian rows stream from L2/HBM (the HBM-bound leg of
// the roofline).
#include "kd_device.cuh"

#include <algorithm>
#include <cstdlib>

namespace kd {

namespace {

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  // every warp reduces the NW partials with the same fixed butterfly
  return warp_sum(lane < NW ? red[lane] : 0.0);
}

template <int NT>
__device__ __forceinline__ void block_max3(double& a, double& b, double& c, double* red) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  a = warp_max(a);
  b = warp_max(b);
  c = warp_max(c);
  __syncthreads();
  if (lane == 0) {
    red[3 * wid] = a;
    red[3 * wid + 1] = b;
    red[3 * wid + 2] = c;
  }
  __syncthreads();
  a = warp_max(lane < NW ? red[3 * lane] : 0.0);  // residuals are >= 0
  b = warp_max(lane < NW ? red[3 * lane + 1] : 0.0);
  c = warp_max(lane < NW ? red[3 * lane + 2] : 0.0);
}

struct CrCtx {
  int n, nb;
  const RowJ* rj;
  const int32_t* rb;
  const int32_t* cptr;
  const int32_t* clist;
  const double* P;      // smem
  const double* dadd;   // smem: P^2 R + (eta + rho)
  const double* binv;   // smem: per body [inv_mass, Iwinv(9)]
  double* scratch;      // smem: 6 nb
  const double* ja;     // smem: P-scaled J rows (12 per row), or null (stream J from global)
  const int32_t* rbs;   // smem copies of rb / cptr / clist when staged
  const int32_t* cps;
  const int32_t* cls;
};

// out = D_{eta,rho} v   (MatrixFreeDelassus::apply).  When the world's rows
// fit, ja = P J (bake_jacobian's first product, delassus.cpp:130-154) and the
// row/body index lists are staged in shared memory once per step, so an apply
// reads no global memory; otherwise J streams from L2/HBM every apply.  Both
// paths perform the same floating-point operations.
template <int NT>
__device__ void apply_op(const CrCtx& c, const double* v, double* out) {
  const int tid = threadIdx.x;
  __syncthreads();
  if (c.ja) {
    for (int u = tid; u < 6 * c.nb; u += NT) {
      const int b = u / 6, k = u - 6 * b;
      double s = 0.0;
      const int e1 = c.cps[b + 1];
      for (int e = c.cps[b]; e < e1; ++e) {
        const int code = c.cls[e];
        const int r = code >> 1;
        s += c.ja[12 * r + 6 * (code & 1) + k] * v[r];
      }
      c.scratch[u] = s;
    }
  } else {
    for (int u = tid; u < 6 * c.nb; u += NT) {
      const int b = u / 6, k = u - 6 * b;
      double s = 0.0;
      for (int e = c.cptr[b]; e < c.cptr[b + 1]; ++e) {
        const int code = c.clist[e];
        const int r = code >> 1;
        s += (c.P[r] * c.rj[r].J[6 * (code & 1) + k]) * v[r];
      }
      c.scratch[u] = s;
    }
  }
  __syncthreads();
  for (int r = tid; r < c.n; r += NT) {
    const double p = c.P[r];
    double s = c.dadd[r] * v[r];
    for (int side = 0; side < 2; ++side) {
      const int b = c.ja ? c.rbs[2 * r + side] : c.rb[2 * r + side];
      if (b < 0) continue;
      const double* bi = c.binv + 10 * b;
      double ja[6];
      if (c.ja) {
#pragma unroll
        for (int k = 0; k < 6; ++k) ja[k] = c.ja[12 * r + 6 * side + k];
      } else {
        const double* J = c.rj[r].J + 6 * side;
#pragma unroll
        for (int k = 0; k < 6; ++k) ja[k] = p * J[k];
      }
      // jma = fold_inverse_mass(ja) (delassus.cpp:12-17)
      double jm[6];
      jm[0] = ja[0] * bi[0];
      jm[1] = ja[1] * bi[0];
      jm[2] = ja[2] * bi[0];
      const double* I = bi + 1;
      jm[3] = ja[3] * I[0] + ja[4] * I[3] + ja[5] * I[6];
      jm[4] = ja[3] * I[1] + ja[4] * I[4] + ja[5] * I[7];
      jm[5] = ja[3] * I[2] + ja[4] * I[5] + ja[5] * I[8];
      const double* sc = c.scratch + 6 * b;
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) t += jm[k] * sc[k];
      s += t;
    }
    out[r] = s;
  }
  __syncthreads();
}


}  // namespace

template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) cr_kernel(BatchView bv, StepParams sp, const int32_t* bin_worlds,
                                                  int smem_doubles, int n_reg) {
  extern __shared__ __align__(16) double smem_[];
  const int w = bin_worlds[blockIdx.x];
  // worlds beyond one CTA's shared memory: the same layout in a per-world HBM slab
  double* smem = bv.cr_scratch ? bv.cr_scratch + (int64_t)w * bv.cr_scratch_stride : smem_;
  WorldStep& ws = bv.wstep[w];
  if (ws.backend != BE_MATRIX_FREE) return;
  const int n = ws.n_rows;
  if (n_reg >= 0) {
    if (n <= n_reg) return;  // cr_op_kernel took it
  } else if (ws.cr_path == 1) {
    return;  // n_reg < 0: the incidence-owner kernel took it this step (it marks every world of the bin)
  }
  const int tid = threadIdx.x;
  if (tid == 0) ws.cr_path = 3;  // KD_CR_PATH_SHARED
  const DevWorld W = bv.worlds[w];
  const int nb = W.nb;
  const int64_t R0 = W.row_off;
  // shared layout
  double* P = smem;
  double* dadd = P + n;
  double* xs = dadd + n;   // x
  double* rr = xs + n;     // r
  double* ar = rr + n;     // A r
  double* pp = ar + n;     // p
  double* ap = pp + n;     // A p
  double* rhs = ap + n;
  double* yv = rhs + n;
  double* zv = yv + n;
  double* yh = zv + n;
  double* zh = yh + n;
  double* vf = zh + n;
  double* binv = vf + n;       // 10 nb
  double* scratch = binv + 10 * nb;  // 6 nb
  double* red = scratch + 6 * nb;    // 3 * NW
  // optional staging (runtime n): ja[12 n] | int rb[2n] | cptr[nb+1] | clist[2n]
  double* ja_s = red + 3 * (NT / 32) + 1;
  int32_t* rb_s = reinterpret_cast<int32_t*>(ja_s + 12 * n);
  int32_t* cp_s = rb_s + 2 * n;
  int32_t* cl_s = cp_s + nb + 1;
  const bool staged = (ja_s - smem) + 12 * n + (4 * n + nb + 2) / 2 + 1 <= smem_doubles;

  const double eta = sp.eta, rho = sp.rho, eta_rho = sp.eta_rho;
  const double inv_rho = 1.0 / rho;  // w = x - z_hat * (1/rho): no division in the loop
  for (int r = tid; r < n; r += NT) {
    const double p = bv.scale[R0 + r];
    P[r] = p;
    dadd[r] = p * p * bv.reg[R0 + r] + eta_rho;
    vf[r] = bv.vf[R0 + r];
    xs[r] = bv.x0[R0 + r];
    zv[r] = bv.z0[R0 + r];
  }
  for (int b = tid; b < nb; b += NT) {
    const BodyS& B = bv.bs[W.body_off + b];
    binv[10 * b] = B.inv_mass;
    for (int k = 0; k < 9; ++k) binv[10 * b + 1 + k] = B.Iwinv[k];
  }
  CrCtx c{n,       nb,      bv.rowj + R0, bv.rbody + 2 * R0, bv.csr_ptr + W.body_off + w, bv.csr + 2 * R0, P, dadd,
          binv,    scratch, nullptr,      nullptr,           nullptr,                     nullptr};
  if (staged) {
    __syncthreads();  // P
    const int32_t* cptr_g = bv.csr_ptr + W.body_off + w;
    const int32_t* cl_g = bv.csr + 2 * R0;
    for (int e = tid; e < 12 * n; e += NT) {
      const int r = e / 12, k = e - 12 * r;
      ja_s[e] = P[r] * bv.rowj[R0 + r].J[k];  // bake_jacobian: ja = P J
    }
    for (int e = tid; e < 2 * n; e += NT) rb_s[e] = bv.rbody[2 * R0 + e];
    for (int b = tid; b <= nb; b += NT) cp_s[b] = cptr_g[b];
    for (int e = tid; e < 2 * n; e += NT) cl_s[e] = cl_g[e];
    c.ja = ja_s;
    c.rbs = rb_s;
    c.cps = cp_s;
    c.cls = cl_s;
  }
  if (sp.cr_only) {
    // ---- one cr_solve(op, rhs, x, max_iters, &history) (delassus.cpp:156-187)
    // on the operator bake_jacobian(cs, inertias, precond, eta_rho) builds
    // (kd_cr_solve_batched): rhs in vf, the warm start in x0; x -> lam,
    // iterations -> cr_iterations, the raw breakdown flag -> cr_breakdown,
    // |r| -> r_p, the residual-norm history (initial |r|, then after every
    // update) -> hist.
    __syncthreads();
    const int hcap = bv.hist_cap;
    double* rhs_ = rhs;
    for (int r = tid; r < n; r += NT) rhs_[r] = vf[r];
    apply_op<NT>(c, xs, ar);
    for (int r = tid; r < n; r += NT) rr[r] = rhs_[r] - ar[r];
    apply_op<NT>(c, rr, ar);
    double loc = 0.0, loc2 = 0.0, loc3 = 0.0;
    for (int r = tid; r < n; r += NT) {
      pp[r] = rr[r];
      ap[r] = ar[r];
      loc += rr[r] * ar[r];
    }
    double rar = block_sum<NT>(loc, red);
    for (int r = tid; r < n; r += NT) loc2 += rhs_[r] * rhs_[r];
    const double rhs2 = block_sum<NT>(loc2, red);
    for (int r = tid; r < n; r += NT) loc3 += rr[r] * rr[r];
    double rn = sqrt(block_sum<NT>(loc3, red));
    int nh = 0;
    if (tid == 0 && nh < hcap) bv.hist[(int64_t)w * hcap + nh] = rn;
    ++nh;
    const double beps = 1e-30 * fmax(1.0, rhs2);
    int iters = 0;
    bool brk = false;
    for (int k = 0; k < sp.cr_iters; ++k) {
      loc = 0.0;
      for (int r = tid; r < n; r += NT) loc += ap[r] * ap[r];
      const double apap = block_sum<NT>(loc, red);
      if (!(rar > beps) || !(apap > beps)) {
        brk = true;
        break;
      }
      const double alpha = rar / apap;
      loc = 0.0;
      for (int r = tid; r < n; r += NT) {
        xs[r] += alpha * pp[r];
        rr[r] -= alpha * ap[r];
        loc += rr[r] * rr[r];
      }
      rn = sqrt(block_sum<NT>(loc, red));
      if (tid == 0 && nh < hcap) bv.hist[(int64_t)w * hcap + nh] = rn;
      ++nh;
      apply_op<NT>(c, rr, ar);
      loc = 0.0;
      for (int r = tid; r < n; r += NT) loc += rr[r] * ar[r];
      const double rar_next = block_sum<NT>(loc, red);
      const double beta = rar_next / rar;
      for (int r = tid; r < n; r += NT) {
        pp[r] = rr[r] + beta * pp[r];
        ap[r] = ar[r] + beta * ap[r];
      }
      rar = rar_next;
      ++iters;
    }
    __syncthreads();
    for (int r = tid; r < n; r += NT) bv.lam[R0 + r] = xs[r];
    if (tid == 0) {
      ws.cr_iterations = iters;
      ws.cr_breakdown = brk ? 1 : 0;
      ws.r_p = rn;
      ws.iterations = 0;
      for (int i = nh; i < hcap; ++i) bv.hist[(int64_t)w * hcap + i] = -1.0;
    }
    return;
  }
  const int n_jd = n - ws.n_limits - 3 * ws.n_contacts;
  const int first_contact = n_jd + ws.n_limits;
  const int n_units = first_contact + ws.n_contacts;
  const double* rmu = bv.rmu + R0;
  __syncthreads();

  // y = Pi_K(x0); hats
  for (int u = tid; u < n_units; u += NT) {
    if (u < n_jd) {
      yv[u] = xs[u];
    } else if (u < first_contact) {
      yv[u] = fmax(0.0, xs[u]);
    } else {
      const int r = first_contact + 3 * (u - first_contact);
      double wv[3] = {xs[r], xs[r + 1], xs[r + 2]}, yn[3];
      project_soc(wv, rmu[r], 1.0 / (1.0 + rmu[r] * rmu[r]), yn);
      for (int d = 0; d < 3; ++d) yv[r + d] = yn[d];
    }
  }
  __syncthreads();
  for (int r = tid; r < n; r += NT) {
    yh[r] = yv[r];
    zh[r] = zv[r];
  }
  double prev = __longlong_as_double(0x7ff0000000000000ll);
  int m = 0;  // Nesterov updates since the last restart (a = a_m)
  double r_p = 0, r_d = 0, r_c = 0;
  int restarts = 0, it;
  bool converged = false;
  long long cr_total = 0;
  bool cr_break = false;
  const int hcap = bv.hist_cap;
  for (it = 1; it <= sp.max_iters; ++it) {
    __syncthreads();
    // rhs = -(v_f + s - eta x - rho y_hat - z_hat)
    for (int r = tid; r < n; r += NT) {
      double s = 0.0;
      if (r >= first_contact && ((r - first_contact) % 3) == 0) s = rmu[r] * fast_sqrt(zh[r + 1] * zh[r + 1] + zh[r + 2] * zh[r + 2]);
      rhs[r] = -((((vf[r] + s) - eta * xs[r]) - rho * yh[r]) - zh[r]);
    }
    // ---- cr_solve(op, rhs, x, budget)
    apply_op<NT>(c, xs, ar);
    double loc = 0.0;
    for (int r = tid; r < n; r += NT) rr[r] = rhs[r] - ar[r];
    apply_op<NT>(c, rr, ar);
    for (int r = tid; r < n; r += NT) {
      pp[r] = rr[r];
      ap[r] = ar[r];
      loc += rr[r] * ar[r];
    }
    double rar = block_sum<NT>(loc, red);
    loc = 0.0;
    for (int r = tid; r < n; r += NT) loc += rhs[r] * rhs[r];
    const double rhs2 = block_sum<NT>(loc, red);
    const double beps = 1e-30 * fmax(1.0, rhs2);
    int iters = 0;
    bool brk = false;
    for (int k = 0; k < sp.cr_iters; ++k) {
      loc = 0.0;
      for (int r = tid; r < n; r += NT) loc += ap[r] * ap[r];
      const double apap = block_sum<NT>(loc, red);
      if (!(rar > beps) || !(apap > beps)) {
        brk = true;
        break;
      }
      const double alpha = rar / apap;
      for (int r = tid; r < n; r += NT) {
        xs[r] += alpha * pp[r];
        rr[r] -= alpha * ap[r];
      }
      apply_op<NT>(c, rr, ar);
      loc = 0.0;
      for (int r = tid; r < n; r += NT) loc += rr[r] * ar[r];
      const double rar_next = block_sum<NT>(loc, red);
      const double beta = rar_next / rar;
      for (int r = tid; r < n; r += NT) {
        pp[r] = rr[r] + beta * pp[r];
        ap[r] = ar[r] + beta * ap[r];
      }
      rar = rar_next;
      ++iters;
    }
    cr_total += iters;
    if (brk) {
      loc = 0.0;
      for (int r = tid; r < n; r += NT) loc += rr[r] * rr[r];
      const double rn = sqrt(block_sum<NT>(loc, red));
      if (rn > 1e-9 * fmax(1.0, sqrt(rhs2))) cr_break = true;
    }
    __syncthreads();
    // ---- projection, dual update, residuals (padmm.cpp:120-123)
    double rp = 0.0, dmax = 0.0, rc = 0.0;
    for (int u = tid; u < n_units; u += NT) {
      const int r = u < first_contact ? u : first_contact + 3 * (u - first_contact);
      const int nr = u < first_contact ? 1 : 3;
      double wv[3], yn[3];
      for (int d = 0; d < nr; ++d) wv[d] = xs[r + d] - zh[r + d] * inv_rho;
      if (u >= first_contact) project_soc(wv, rmu[r], 1.0 / (1.0 + rmu[r] * rmu[r]), yn);
      else if (u >= n_jd) yn[0] = fmax(0.0, wv[0]);
      else yn[0] = wv[0];
      double ymax = 0.0, zmax = 0.0;
      for (int d = 0; d < nr; ++d) {
        const double zn = zh[r + d] - rho * (xs[r + d] - yn[d]);
        rp = fmax(rp, fabs(xs[r + d] - yn[d]));
        dmax = fmax(dmax, fabs(yn[d] - yv[r + d]));
        ymax = fmax(ymax, fabs(yn[d]));
        zmax = fmax(zmax, fabs(zn));
        // y_prev, z_prev are kept in yh/zh until the Nesterov step below
        yh[r + d] = yv[r + d];
        zh[r + d] = zv[r + d];
        yv[r + d] = yn[d];
        zv[r + d] = zn;
      }
      if (u >= n_jd) rc = fmax(rc, fmin(ymax, zmax));
    }
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
    if (sp.acceleration) {
      const bool restart = sp.restart && combined > prev;
      if (restart) {
        m = 0;
        ++restarts;
        for (int r = tid; r < n; r += NT) {
          yh[r] = yv[r];
          zh[r] = zv[r];
        }
      } else {
        const double beta = sp.nest_beta[m++];  // (a_m - 1) / a_{m+1}, host table
        for (int r = tid; r < n; r += NT) {
          yh[r] = yv[r] + beta * (yv[r] - yh[r]);
          zh[r] = zv[r] + beta * (zv[r] - zh[r]);
        }
      }
    } else {
      for (int r = tid; r < n; r += NT) {
        yh[r] = yv[r];
        zh[r] = zv[r];
      }
    }
    prev = combined;
  }
  __syncthreads();
  for (int r = tid; r < n; r += NT) {
    bv.lam[R0 + r] = yv[r];
    bv.zo[R0 + r] = zv[r];
  }
  if (tid == 0) {
    const int done = min(it, sp.max_iters);
    ws.iterations = done;
    ws.r_p = r_p;
    ws.r_d = r_d;
    ws.r_c = r_c;
    ws.restarts = restarts;
    ws.converged = (converged || fmax(r_p, fmax(r_d, r_c)) < sp.eps) ? 1 : 0;
    ws.cr_iterations = cr_total;
    ws.cr_breakdown = cr_break ? 1 : 0;
    for (int i = done; i < hcap; ++i) bv.hist[(int64_t)w * hcap + i] = -1.0;
  }
}

// ---------------------------------------------------------------------------
// K2b' cr_reg_kernel<NT, RPT>: the same PADMM + warm-started CR, with the CR
// state held in registers.  Thread t owns rows t, t + NT, ... (at most RPT):
// its P-scaled Jacobian blocks ja = P J (bake_jacobian, delassus.cpp:139-146),
// diag_add and the CR vectors x, r, p, Ap stay in registers for the whole
// step.  ja is also staged once per step incidence-major: slot e of a body's
// ascending incidence list (the CSR K1 builds) holds that row side's 6 values.
// An apply is then three shared-memory passes:
//   A  row owner:  v_r -> both incidence slots of row r;
//   B  body half:  s_b = sum_e ja_e^T v_{r(e)} in ascending row order (the
//                  reference scatter order, delassus.cpp:108-113),
//                  w_b = M_b^-1 s_b;
//   C  row owner:  out_r = diag_add v_r + ja_a . w_a + ja_b . w_b.
// ja . (M^-1 s) is the reference's jma . s (jma = fold_inverse_mass(ja),
// delassus.cpp:12-17, M^-1 symmetric) with the product re-associated.
// Block reductions use one barrier each (double-buffered partials, every
// thread sums the warp partials in the same fixed order).  Worlds with
// n > RPT * NT are left to cr_kernel (runtime check on both sides).
// ---------------------------------------------------------------------------
namespace {

template <int NT, int K>
__device__ __forceinline__ void bsum(double (&v)[K], double* red, int& par) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* buf = red + par * (NW * K);
  par ^= 1;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) buf[wid * K + k] = v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = buf[k];
#pragma unroll
    for (int i = 1; i < NW; ++i) s += buf[i * K + k];
    v[k] = s;
  }
}

template <int NT>
__device__ __forceinline__ void bmax3(double& a, double& b, double& c, double* red, int& par) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* buf = red + par * (NW * 3);
  par ^= 1;
  a = warp_max_nonneg(a);
  b = warp_max_nonneg(b);
  c = warp_max_nonneg(c);
  if (lane == 0) {
    buf[3 * wid] = a;
    buf[3 * wid + 1] = b;
    buf[3 * wid + 2] = c;
  }
  __syncthreads();
  a = buf[0];
  b = buf[1];
  c = buf[2];
#pragma unroll
  for (int i = 1; i < NW; ++i) {
    a = fmax(a, buf[3 * i]);
    b = fmax(b, buf[3 * i + 1]);
    c = fmax(c, buf[3 * i + 2]);
  }
}

// phase clock of thread 0 (KD_CR_REG=2 diagnostics launch)
template <bool PROF>
__device__ __forceinline__ void pstamp(long long* acc, int k, long long& t) {
  if (PROF && threadIdx.x == 0) {
    const long long c = clock64();
    acc[k] += c - t;
    t = c;
  }
}

// start residue (mod 8 incidences of 48 B) of body b's segment, by b mod 8:
// 16-byte slots {3r, 3r+2} mod 8 are distinct within each group of four
// bodies and the 8-byte slots 6r mod 16 within each group of eight
__constant__ int kBodyRes[8] = {0, 3, 4, 7, 6, 1, 2, 5};

// ---- operator 1: rows own P J in registers; J also staged incidence-major
template <int NT, int RPT, bool PROF>
struct RegOp {
  double ja[RPT][12];
  double dadd[RPT];
  int ea[RPT], eb[RPT];  // incidence slots (or -1)
  int ba[RPT], bb[RPT];  // bodies (or -1)
  double *jinc, *vinc, *wv;
  const double* binv;
  const int32_t* pseg;

  // op shared memory: jinc 6 S | vinc S | w 6 nb | binv 10 nb | int: cptr nb+1,
  // pseg 2 nb, slot 2n  (S = 2n + 7 nb + 8 incidence slots, rounded even)
  static size_t smem_bytes(int n, int nb) {
    return 8 * ((size_t)14 * n + 65 * (size_t)nb + 64) + 4 * ((size_t)3 * nb + 2 + 2 * n) + 16;
  }

  __device__ bool setup(const BatchView& bv, const DevWorld& W, int w, int n, int nb, double eta_rho, double* dsm) {
    const int tid = threadIdx.x;
    const int64_t R0 = W.row_off;
    const int nslot = (2 * n + 7 * nb + 9) & ~1;  // even: keeps w 16-byte aligned
    jinc = dsm;
    vinc = jinc + 6 * nslot;
    wv = vinc + nslot;
    double* binv_w = wv + 6 * nb;
    binv = binv_w;
    int32_t* cptr = reinterpret_cast<int32_t*>(binv_w + 10 * nb);
    int32_t* pseg_w = cptr + ((nb + 2) & ~1);
    pseg = pseg_w;
    int32_t* slot = pseg_w + 2 * nb;
    const int32_t* cptr_g = bv.csr_ptr + W.body_off + w;
    const int32_t* cl_g = bv.csr + 2 * R0;
    for (int b = tid; b <= nb; b += NT) cptr[b] = cptr_g[b];
    for (int b = tid; b < nb; b += NT) {
      const BodyS& B = bv.bs[W.body_off + b];
      binv_w[10 * b] = B.inv_mass;
      for (int k = 0; k < 9; ++k) binv_w[10 * b + 1 + k] = B.Iwinv[k];
    }
    __syncthreads();
    if (tid == 0) {
      int p = 0;
      for (int b = 0; b < nb; ++b) {
        p += (kBodyRes[b & 7] - p) & 7;
        pseg_w[2 * b] = p;
        p += cptr[b + 1] - cptr[b];
        pseg_w[2 * b + 1] = p;
      }
    }
    __syncthreads();
    for (int b = tid; b < nb; b += NT) {
      const int c0 = cptr[b], c1 = cptr[b + 1], p0 = pseg_w[2 * b];
      for (int e = c0; e < c1; ++e) slot[cl_g[e]] = p0 + (e - c0);
    }
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int r = tid + k * NT;
      dadd[k] = 0.0;
      ba[k] = bb[k] = -1;
#pragma unroll
      for (int i = 0; i < 12; ++i) ja[k][i] = 0.0;
      if (r < n) {
        const double p = bv.scale[R0 + r];
        dadd[k] = p * p * bv.reg[R0 + r] + eta_rho;
        const double* J = bv.rowj[R0 + r].J;
#pragma unroll
        for (int i = 0; i < 12; ++i) ja[k][i] = p * J[i];  // bake_jacobian: ja = P J
        ba[k] = bv.rbody[2 * (R0 + r)];
        bb[k] = bv.rbody[2 * (R0 + r) + 1];
      }
    }
    __syncthreads();  // slot
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int r = tid + k * NT;
      ea[k] = (r < n && ba[k] >= 0) ? slot[2 * r] : -1;
      eb[k] = (r < n && bb[k] >= 0) ? slot[2 * r + 1] : -1;
      if (ea[k] >= 0)
        for (int i = 0; i < 6; ++i) jinc[6 * ea[k] + i] = ja[k][i];
      if (eb[k] >= 0)
        for (int i = 0; i < 6; ++i) jinc[6 * eb[k] + i] = ja[k][6 + i];
    }
    return true;
  }

  __device__ __forceinline__ void apply(int n, int nb, const double (&v)[RPT], double (&out)[RPT], long long* acc,
                                        long long& tclk) const {
    const int tid = threadIdx.x;
    pstamp<PROF>(acc, 5, tclk);
    // A: publish v_r into both of the row's incidence slots
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      if (ea[k] >= 0) vinc[ea[k]] = v[k];
      if (eb[k] >= 0) vinc[eb[k]] = v[k];
    }
    __syncthreads();
    pstamp<PROF>(acc, 0, tclk);
    // B: body halves (linear / angular): s_b = sum over the body's incidences in
    // ascending row order of ja^T v_r, then M^-1.  Body segments start at
    // residues of 8 (kBodyRes) that keep the lanes of a warp on distinct banks
    // while they walk their lists in step; both halves run the same
    // instructions (half h reads the 16-byte pair at +4h and the word at +2+h).
    for (int u = tid; u < 2 * nb; u += NT) {
      const int b = u >> 1, h = u & 1;
      const int2 se = *reinterpret_cast<const int2*>(pseg + 2 * b);
      double sp = 0.0, sq = 0.0, sc = 0.0;  // pair .x, pair .y, single
      const double* pr = jinc + 4 * h;
      const double* pc = jinc + 2 + h;
#pragma unroll 4
      for (int e = se.x; e < se.y; ++e) {
        const double vr = vinc[e];
        const double2 a = *reinterpret_cast<const double2*>(pr + 6 * e);
        const double c = pc[6 * e];
        sp += a.x * vr;
        sq += a.y * vr;
        sc += c * vr;
      }
      // s = (s0, s1, s2) of this half: linear (sp, sq, sc), angular (sc, sp, sq)
      const double s0 = h ? sc : sp, s1 = h ? sp : sq, s2 = h ? sq : sc;
      const double* I = binv + 10 * b + 1;
      const double im = binv[10 * b];
      double* wo = wv + 6 * b + 3 * h;
      if (h == 0) {
        wo[0] = im * s0;
        wo[1] = im * s1;
        wo[2] = im * s2;
      } else {
        wo[0] = (I[0] * s0 + I[1] * s1) + I[2] * s2;
        wo[1] = (I[3] * s0 + I[4] * s1) + I[5] * s2;
        wo[2] = (I[6] * s0 + I[7] * s1) + I[8] * s2;
      }
    }
    __syncthreads();
    pstamp<PROF>(acc, 1, tclk);
    // C: gather
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      double s = dadd[k] * v[k];
      if (ba[k] >= 0) {
        const double2* wp = reinterpret_cast<const double2*>(wv + 6 * ba[k]);
        const double2 w0 = wp[0], w1 = wp[1], w2 = wp[2];
        s += ((ja[k][0] * w0.x + ja[k][1] * w0.y) + (ja[k][2] * w1.x + ja[k][3] * w1.y)) +
             (ja[k][4] * w2.x + ja[k][5] * w2.y);
      }
      if (bb[k] >= 0) {
        const double2* wp = reinterpret_cast<const double2*>(wv + 6 * bb[k]);
        const double2 w0 = wp[0], w1 = wp[1], w2 = wp[2];
        s += ((ja[k][6] * w0.x + ja[k][7] * w0.y) + (ja[k][8] * w1.x + ja[k][9] * w1.y)) +
             (ja[k][10] * w2.x + ja[k][11] * w2.y);
      }
      out[k] = s;
    }
    pstamp<PROF>(acc, 2, tclk);
  }
};

// ---- operator 2: incidence owners.  Lanes own contiguous pieces (<= P
// incidences) of one body's ascending incidence list and keep those
// incidences' P J blocks in registers; a body's pieces sit on consecutive
// lanes of one warp.  Rows only keep diag_add and their two slots.
//   A  row owner:   v_r -> both incidence slots of row r;
//   B  piece lane:  partial s = sum ja_e^T v over the piece (ascending), then a
//                   fixed tree over the body's lanes (shuffles) and w = M^-1 s;
//   C  piece lane:  q_e = ja_e . w_b per incidence -> slot e;
//      row owner:   out_r = diag_add v_r + q_a + q_b.
// Worlds whose bodies do not fit NT lanes (a body needs ceil(deg / P) lanes
// within one warp) are left to RegOp.
template <int NT, int RPT, int P, bool PROF>
struct IncOp {
  double dadd[RPT];
  int ea[RPT], eb[RPT];
  double jp[P][6];
  int e0, cnt, mb, g0, gq;
  double *vinc, *qinc;
  const double* binv;

  // op shared memory: vinc V | qinc V | binv 10 nb | int: cptr nb+1, slot 2n, lanes 4 NT, flag.
  // With an even piece bound P (the 8-incidence launch), vinc / qinc give
  // thread t's piece the slots [t PS, t PS + cnt) with the odd stride
  // PS = P + 1, so the lanes of a warp walking their pieces in step hit
  // distinct banks (contiguous pieces of length 8 put them 8 words apart:
  // 8-way conflicts, 49 % of the box pile's shared-memory wavefronts; box pile
  // +4.6 %).  With an odd P the pieces stay contiguous in CSR order, which keeps
  // the row owners' accesses consecutive (the padded layout measured 8-11 %
  // slower on the closed chain and the Stewart tower).
  static constexpr bool PAD = (P % 2) == 0;
  static constexpr int PS = P | 1;
  __host__ __device__ static int vlen(int n) { return PAD ? PS * NT : 2 * n; }
  static size_t smem_bytes(int n, int nb) {
    return 8 * ((size_t)2 * vlen(n) + 10 * (size_t)nb + 2) + 4 * ((size_t)nb + 2 + 2 * n + 4 * NT + 2) + 16;
  }

  __device__ bool setup(const BatchView& bv, const DevWorld& W, int w, int n, int nb, double eta_rho, double* dsm) {
    const int tid = threadIdx.x;
    const int64_t R0 = W.row_off;
    const int V = vlen(n);
    vinc = dsm;
    qinc = vinc + V;
    double* binv_w = qinc + V;
    binv = binv_w;
    int32_t* cptr = reinterpret_cast<int32_t*>(binv_w + 10 * nb);
    int32_t* slot = cptr + nb + 1;
    int32_t* lanes = slot + 2 * n;  // per lane: body, e0, cnt, g0 | gq << 16
    int32_t* okf = lanes + 4 * NT;
    const int32_t* cptr_g = bv.csr_ptr + W.body_off + w;
    const int32_t* cl_g = bv.csr + 2 * R0;
    for (int b = tid; b <= nb; b += NT) cptr[b] = cptr_g[b];
    for (int b = tid; b < nb; b += NT) {
      const BodyS& B = bv.bs[W.body_off + b];
      binv_w[10 * b] = B.inv_mass;
      for (int k = 0; k < 9; ++k) binv_w[10 * b + 1 + k] = B.Iwinv[k];
    }
    lanes[4 * tid] = -1;
    lanes[4 * tid + 1] = 0;
    lanes[4 * tid + 2] = 0;
    lanes[4 * tid + 3] = tid | (1 << 16);
    __syncthreads();
    if (tid == 0) {
      int L = 0, ok = 1;
      for (int b = 0; b < nb && ok; ++b) {
        const int c0 = cptr[b], d = cptr[b + 1] - c0;
        if (d == 0) continue;
        const int q = (d + P - 1) / P;
        if (q > 32) {
          ok = 0;
          break;
        }
        if ((L & 31) + q > 32) L = (L + 31) & ~31;  // a body's lanes stay in one warp
        if (L + q > NT) {
          ok = 0;
          break;
        }
        const int pl = (d + q - 1) / q;
        for (int j = 0; j < q; ++j) {
          lanes[4 * (L + j)] = b;
          lanes[4 * (L + j) + 1] = c0 + j * pl;
          lanes[4 * (L + j) + 2] = max(0, min(pl, d - j * pl));
          lanes[4 * (L + j) + 3] = L | (q << 16);
        }
        L += q;
      }
      *okf = ok;
    }
    for (int e = tid; e < 2 * n; e += NT) slot[e] = -1;
    __syncthreads();
    if (!*okf) return false;
    mb = lanes[4 * tid];
    e0 = lanes[4 * tid + 1];
    cnt = lanes[4 * tid + 2];
    for (int j = 0; j < cnt; ++j) slot[cl_g[e0 + j]] = PAD ? tid * PS + j : e0 + j;
    g0 = lanes[4 * tid + 3] & 0xffff;
    gq = lanes[4 * tid + 3] >> 16;
#pragma unroll
    for (int j = 0; j < P; ++j) {
#pragma unroll
      for (int k = 0; k < 6; ++k) jp[j][k] = 0.0;
      if (j < cnt) {
        const int code = cl_g[e0 + j];
        const int r = code >> 1;
        const double p = bv.scale[R0 + r];
        const double* J = bv.rowj[R0 + r].J + 6 * (code & 1);
#pragma unroll
        for (int k = 0; k < 6; ++k) jp[j][k] = p * J[k];  // bake_jacobian: ja = P J
      }
    }
    __syncthreads();  // slot
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int r = tid + k * NT;
      dadd[k] = 0.0;
      ea[k] = eb[k] = -1;
      if (r < n) {
        const double p = bv.scale[R0 + r];
        dadd[k] = p * p * bv.reg[R0 + r] + eta_rho;
        if (bv.rbody[2 * (R0 + r)] >= 0) ea[k] = slot[2 * r];
        if (bv.rbody[2 * (R0 + r) + 1] >= 0) eb[k] = slot[2 * r + 1];
      }
    }
    return true;
  }

  __device__ __forceinline__ void apply(int n, int nb, const double (&v)[RPT], double (&out)[RPT], long long* acc,
                                        long long& tclk) const {
    pstamp<PROF>(acc, 5, tclk);
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      if (ea[k] >= 0) vinc[ea[k]] = v[k];
      if (eb[k] >= 0) vinc[eb[k]] = v[k];
    }
    __syncthreads();
    pstamp<PROF>(acc, 0, tclk);
    double s[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < P; ++j) {
      if (j < cnt) {
        const double vv = vinc[PAD ? threadIdx.x * PS + j : e0 + j];
#pragma unroll
        for (int k = 0; k < 6; ++k) s[k] += jp[j][k] * vv;
      }
    }
    // fixed tree over the body's lanes toward its first lane, then broadcast
    const int lane = threadIdx.x & 31, gl = g0 & 31, qi = lane - gl;
    const int qmax = __reduce_max_sync(0xffffffffu, gq);
    for (int o = 1; o < qmax; o <<= 1) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double t = __shfl_down_sync(0xffffffffu, s[k], o);
        if ((qi & (2 * o - 1)) == 0 && qi + o < gq) s[k] += t;
      }
    }
    if (qmax > 1) {
#pragma unroll
      for (int k = 0; k < 6; ++k) s[k] = __shfl_sync(0xffffffffu, s[k], gl);
    }
    double wv[6];
    if (mb >= 0) {
      const double* bi = binv + 10 * mb;
      const double im = bi[0];
      const double* I = bi + 1;
      wv[0] = im * s[0];
      wv[1] = im * s[1];
      wv[2] = im * s[2];
      wv[3] = (I[0] * s[3] + I[1] * s[4]) + I[2] * s[5];
      wv[4] = (I[3] * s[3] + I[4] * s[4]) + I[5] * s[5];
      wv[5] = (I[6] * s[3] + I[7] * s[4]) + I[8] * s[5];
    }
#pragma unroll
    for (int j = 0; j < P; ++j)
      if (j < cnt)
        qinc[PAD ? threadIdx.x * PS + j : e0 + j] = ((jp[j][0] * wv[0] + jp[j][1] * wv[1]) + (jp[j][2] * wv[2] + jp[j][3] * wv[3])) +
                       (jp[j][4] * wv[4] + jp[j][5] * wv[5]);
    __syncthreads();
    pstamp<PROF>(acc, 1, tclk);
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      double t = dadd[k] * v[k];
      if (ea[k] >= 0) t += qinc[ea[k]];
      if (eb[k] >= 0) t += qinc[eb[k]];
      out[k] = t;
    }
    pstamp<PROF>(acc, 2, tclk);
  }
};
}  // namespace

// common shared memory of cr_op_kernel: 6 n vectors | 2 x 3 x NW reduction partials
static size_t cr_common_bytes(int n, int nt) { return 8 * ((size_t)6 * n + 2 * 3 * (nt / 32) + 2); }

template <class Op, int NT, int RPT, int MINB, bool PROF, bool MARK>
__global__ void __launch_bounds__(NT, MINB) cr_op_kernel(BatchView bv, StepParams sp, const int32_t* bin_worlds,
                                                         int skip_marked) {
  extern __shared__ __align__(16) double smem[];
  const int w = bin_worlds[blockIdx.x];
  WorldStep& ws = bv.wstep[w];
  if (ws.backend != BE_MATRIX_FREE) return;
  if (skip_marked && ws.cr_path == 1) return;  // the incidence-owner kernel took it
  const int n = ws.n_rows;
  const int tid = threadIdx.x;
  if (n > RPT * NT) {  // cr_kernel takes it
    if (MARK && tid == 0) ws.cr_path = 0;
    return;
  }
  const DevWorld W = bv.worlds[w];
  const int nb = W.nb;
  const int64_t R0 = W.row_off;
  double* yv = smem;
  double* zv = yv + n;
  double* yh = zv + n;
  double* zh = yh + n;
  double* vf = zh + n;
  double* xs = vf + n;
  double* red = xs + n;  // 2 buffers x 3 x NW
  double* opsm = red + ((2 * 3 * (NT / 32) + 1) & ~1);
  const double eta = sp.eta, rho = sp.rho, eta_rho = sp.eta_rho;
  const double inv_rho = 1.0 / rho;
  Op op;
  const bool ok = op.setup(bv, W, w, n, nb, eta_rho, opsm);
  if (MARK && tid == 0) ws.cr_path = ok ? 1 : 0;  // KD_CR_PATH_INCIDENCE, or left to RegOp
  if (!ok) return;
  if (!MARK && tid == 0) ws.cr_path = 2;  // KD_CR_PATH_ROWS
  double x[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int r = tid + k * NT;
    x[k] = 0.0;
    if (r < n) {
      x[k] = bv.x0[R0 + r];
      xs[r] = x[k];
      vf[r] = bv.vf[R0 + r];
      zv[r] = bv.z0[R0 + r];
    }
  }
  __syncthreads();
  const int n_jd = n - ws.n_limits - 3 * ws.n_contacts;
  const int first_contact = n_jd + ws.n_limits;
  const int n_units = first_contact + ws.n_contacts;
  const double* rmu = bv.rmu + R0;

  // y = Pi_K(x0); hats
  for (int u = tid; u < n_units; u += NT) {
    if (u < n_jd) {
      yv[u] = xs[u];
    } else if (u < first_contact) {
      yv[u] = fmax(0.0, xs[u]);
    } else {
      const int r = first_contact + 3 * (u - first_contact);
      double wv3[3] = {xs[r], xs[r + 1], xs[r + 2]}, yn[3];
      project_soc(wv3, rmu[r], 1.0 / (1.0 + rmu[r] * rmu[r]), yn);
      for (int d = 0; d < 3; ++d) yv[r + d] = yn[d];
    }
  }
  __syncthreads();
  for (int r = tid; r < n; r += NT) {
    yh[r] = yv[r];
    zh[r] = zv[r];
  }
  __syncthreads();
  int par = 0;
  double prev = __longlong_as_double(0x7ff0000000000000ll);
  int m = 0;
  double r_p = 0, r_d = 0, r_c = 0;
  int restarts = 0, it;
  bool converged = false;
  long long cr_total = 0;
  bool cr_break = false;
  const int hcap = bv.hist_cap;
  long long acc[6] = {0, 0, 0, 0, 0, 0};
  long long tclk = PROF ? clock64() : 0;
  const long long t_start = tclk;
  for (it = 1; it <= sp.max_iters; ++it) {
    // rhs = -(v_f + s - eta x - rho y_hat - z_hat)   (padmm.cpp:116-117)
    double rhs[RPT], rr[RPT], pp[RPT], ap[RPT], ar[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int r = tid + k * NT;
      rhs[k] = 0.0;
      if (r < n) {
        double s = 0.0;
        if (r >= first_contact && ((r - first_contact) % 3) == 0)
          s = rmu[r] * fast_sqrt(zh[r + 1] * zh[r + 1] + zh[r + 2] * zh[r + 2]);
        rhs[k] = -((((vf[r] + s) - eta * x[k]) - rho * yh[r]) - zh[r]);
      }
    }
    // ---- cr_solve(op, rhs, x, budget)   (delassus.cpp:156-187)
    op.apply(n, nb, x, ar, acc, tclk);
#pragma unroll
    for (int k = 0; k < RPT; ++k) rr[k] = rhs[k] - ar[k];
    op.apply(n, nb, rr, ar, acc, tclk);
    double d3[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      pp[k] = rr[k];
      ap[k] = ar[k];
      d3[0] += rr[k] * ar[k];
      d3[1] += rhs[k] * rhs[k];
      d3[2] += ar[k] * ar[k];
    }
    pstamp<PROF>(acc, 5, tclk);
    bsum<NT, 3>(d3, red, par);
    pstamp<PROF>(acc, 3, tclk);
    double rar = d3[0];
    const double rhs2 = d3[1];
    double apap = d3[2];
    const double beps = 1e-30 * fmax(1.0, rhs2);
    int iters = 0;
    bool brk = false;
    for (int kk = 0; kk < sp.cr_iters; ++kk) {
      if (kk > 0) {
        double a1[1] = {0.0};
#pragma unroll
        for (int k = 0; k < RPT; ++k) a1[0] += ap[k] * ap[k];
        pstamp<PROF>(acc, 5, tclk);
        bsum<NT, 1>(a1, red, par);
        pstamp<PROF>(acc, 3, tclk);
        apap = a1[0];
      }
      if (!(rar > beps) || !(apap > beps)) {
        brk = true;
        break;
      }
      const double alpha = fast_div(rar, apap);
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        x[k] += alpha * pp[k];
        rr[k] -= alpha * ap[k];
      }
      op.apply(n, nb, rr, ar, acc, tclk);
      double a1[1] = {0.0};
#pragma unroll
      for (int k = 0; k < RPT; ++k) a1[0] += rr[k] * ar[k];
      pstamp<PROF>(acc, 5, tclk);
      bsum<NT, 1>(a1, red, par);
      pstamp<PROF>(acc, 3, tclk);
      const double beta = fast_div(a1[0], rar);
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        pp[k] = rr[k] + beta * pp[k];
        ap[k] = ar[k] + beta * ap[k];
      }
      rar = a1[0];
      ++iters;
    }
    cr_total += iters;
    if (brk) {
      double a1[1] = {0.0};
#pragma unroll
      for (int k = 0; k < RPT; ++k) a1[0] += rr[k] * rr[k];
      bsum<NT, 1>(a1, red, par);
      if (sqrt(a1[0]) > 1e-9 * fmax(1.0, sqrt(rhs2))) cr_break = true;
    }
#pragma unroll
    for (int k = 0; k < RPT; ++k)
      if (tid + k * NT < n) xs[tid + k * NT] = x[k];
    __syncthreads();
    // ---- projection, dual update, residuals (padmm.cpp:120-123)
    double rp = 0.0, dmax = 0.0, rc = 0.0;
    for (int u = tid; u < n_units; u += NT) {
      const int r = u < first_contact ? u : first_contact + 3 * (u - first_contact);
      const int nr = u < first_contact ? 1 : 3;
      double wv3[3], yn[3];
      for (int d = 0; d < nr; ++d) wv3[d] = xs[r + d] - zh[r + d] * inv_rho;
      if (u >= first_contact) project_soc(wv3, rmu[r], fast_rcp(1.0 + rmu[r] * rmu[r]), yn);
      else if (u >= n_jd) yn[0] = fmax(0.0, wv3[0]);
      else yn[0] = wv3[0];
      double ymax = 0.0, zmax = 0.0;
      for (int d = 0; d < nr; ++d) {
        const double zn = zh[r + d] - rho * (xs[r + d] - yn[d]);
        rp = fmax(rp, fabs(xs[r + d] - yn[d]));
        dmax = fmax(dmax, fabs(yn[d] - yv[r + d]));
        ymax = fmax(ymax, fabs(yn[d]));
        zmax = fmax(zmax, fabs(zn));
        yh[r + d] = yv[r + d];  // y_prev, z_prev until the Nesterov step
        zh[r + d] = zv[r + d];
        yv[r + d] = yn[d];
        zv[r + d] = zn;
      }
      if (u >= n_jd) rc = fmax(rc, fmin(ymax, zmax));
    }
    pstamp<PROF>(acc, 5, tclk);
    bmax3<NT>(rp, dmax, rc, red, par);
    pstamp<PROF>(acc, 4, tclk);
    r_p = rp;
    r_d = rho * dmax;
    r_c = rc;
    const double combined = fmax(r_p, fmax(r_d, r_c));
    if (tid == 0 && it <= hcap) bv.hist[(int64_t)w * hcap + it - 1] = combined;
    if (!sp.fixed_mode && combined < sp.eps) {
      converged = true;
      break;
    }
    // Nesterov step on the rows of this thread's own units (no barrier needed
    // between the projection and this update)
    const bool restart = sp.acceleration && sp.restart && combined > prev;
    if (restart) {
      m = 0;
      ++restarts;
    }
    const bool nest = sp.acceleration && !restart;
    const double beta = nest ? sp.nest_beta[m] : 0.0;  // (a_m - 1) / a_{m+1}, host table
    if (nest) ++m;
    for (int u = tid; u < n_units; u += NT) {
      const int r = u < first_contact ? u : first_contact + 3 * (u - first_contact);
      const int nr = u < first_contact ? 1 : 3;
      for (int d = 0; d < nr; ++d) {
        if (nest) {
          yh[r + d] = yv[r + d] + beta * (yv[r + d] - yh[r + d]);
          zh[r + d] = zv[r + d] + beta * (zv[r + d] - zh[r + d]);
        } else {
          yh[r + d] = yv[r + d];
          zh[r + d] = zv[r + d];
        }
      }
    }
    prev = combined;
    __syncthreads();
  }
  __syncthreads();
  for (int r = tid; r < n; r += NT) {
    bv.lam[R0 + r] = yv[r];
    bv.zo[R0 + r] = zv[r];
  }
  if (tid == 0) {
    const int done = min(it, sp.max_iters);
    ws.iterations = done;
    ws.r_p = r_p;
    ws.r_d = r_d;
    ws.r_c = r_c;
    ws.restarts = restarts;
    ws.converged = (converged || fmax(r_p, fmax(r_d, r_c)) < sp.eps) ? 1 : 0;
    ws.cr_iterations = cr_total;
    ws.cr_breakdown = cr_break ? 1 : 0;
    for (int i = done; i < hcap; ++i) bv.hist[(int64_t)w * hcap + i] = -1.0;
    if (PROF) {
      // [0] publish v + barrier, [1] body sums + barrier, [2] gather, [3] CR
      // reductions, [4] PADMM residual reduction, [5] the rest, [6] total
      for (int k = 0; k < 6; ++k) ws.phase_cycles[k] = acc[k];
      ws.phase_cycles[6] = clock64() - t_start;
    }
  }
}

size_t cr_smem_bytes(int n, int nb, int nt) { return 8 * ((size_t)13 * n + 16 * (size_t)nb + 3 * (nt / 32) + 8); }
// with the optional per-step staging of P J and the index lists
size_t cr_staged_bytes(int n, int nb, int nt) {
  return 8 * ((size_t)25 * n + 16 * (size_t)nb + 3 * (nt / 32) + 8 + ((size_t)4 * n + nb + 2) / 2 + 2);
}

template <int NT, int MINB>
static cudaError_t launch_cr_t(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, int ncap,
                               int nbcap, int n_reg, cudaStream_t s) {
  if (bv.cr_scratch) {
    cr_kernel<NT, MINB><<<count, NT, 0, s>>>(bv, sp, worlds, (int)std::min<int64_t>(bv.cr_scratch_stride, 1 << 30),
                                              n_reg);
    return cudaGetLastError();
  }
  const size_t smem = std::max(cr_smem_bytes(ncap, nbcap, NT),
                               std::min<size_t>(232448 / MINB, cr_staged_bytes(ncap, nbcap, NT)));
  static SmemAttrCache attr;
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(cr_kernel<NT, MINB>), smem, attr);
    if (e != cudaSuccess) return e;
  }
  cr_kernel<NT, MINB><<<count, NT, smem, s>>>(bv, sp, worlds, (int)(smem / 8), n_reg);
  return cudaGetLastError();
}

// The shared-memory CR kernel over every listed world (any n that fits one
// CTA's shared memory), e.g. for the cr_only mode of kd_cr_solve_batched.
cudaError_t launch_cr_shared(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, int ncap,
                             int nbcap, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  return launch_cr_t<256, 1>(bv, sp, worlds, count, ncap, nbcap, 0, s);
}

template <class Op, int NT, int RPT, int MINB, bool PROF, bool MARK>
static cudaError_t launch_cr_op_p(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count,
                                  int ncap, int nbcap, int skip_marked, cudaStream_t s) {
  const int nc = std::min(ncap, RPT * NT);
  const size_t smem = cr_common_bytes(nc, NT) + Op::smem_bytes(nc, nbcap);
  static SmemAttrCache attr;
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(cr_op_kernel<Op, NT, RPT, MINB, PROF, MARK>), smem, attr);
    if (e != cudaSuccess) return e;
  }
  cr_op_kernel<Op, NT, RPT, MINB, PROF, MARK><<<count, NT, smem, s>>>(bv, sp, worlds, skip_marked);
  return cudaGetLastError();
}

static int cr_reg_mode();
#ifndef KD_INC512_P
#define KD_INC512_P 5
#endif

// KD_CR_REG: 0 = shared-memory kernel only, 1 (default) = incidence-owner then
// register-row kernels, 2 = the same with phase clocks, 3 = register-row only,
// 4 = the 512-thread incidence-owner launch for 513..1024-row bins
template <int NT, int RPT, int MINB>
static cudaError_t launch_cr_reg_t(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count,
                                   int ncap, int nbcap, cudaStream_t s) {
  const int mode = cr_reg_mode();
  const bool prof = mode == 2;
  const bool inc = mode != 3 && cr_common_bytes(std::min(ncap, RPT * NT), NT) +
                                         IncOp<NT, RPT, 5, false>::smem_bytes(std::min(ncap, RPT * NT), nbcap) <=
                                     232448 / MINB;
  cudaError_t e = cudaSuccess;
  if (inc) {
    e = prof ? launch_cr_op_p<IncOp<NT, RPT, 5, true>, NT, RPT, MINB, true, true>(bv, sp, worlds, count, ncap, nbcap, 0, s)
             : launch_cr_op_p<IncOp<NT, RPT, 5, false>, NT, RPT, MINB, false, true>(bv, sp, worlds, count, ncap, nbcap, 0, s);
    if (e != cudaSuccess) return e;
  }
  return prof ? launch_cr_op_p<RegOp<NT, RPT, true>, NT, RPT, MINB, true, false>(bv, sp, worlds, count, ncap, nbcap, inc, s)
              : launch_cr_op_p<RegOp<NT, RPT, false>, NT, RPT, MINB, false, false>(bv, sp, worlds, count, ncap, nbcap, inc, s);
}

static int cr_reg_mode() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("KD_CR_REG");
    m = e ? atoi(e) : 1;
  }
  return m;
}

cudaError_t launch_cr(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, int ncap, int nbcap,
                      int nt, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  // register-resident CR for worlds with n <= 2 NT rows (runtime n), the
  // shared-memory kernel for the rest (both launched over the bin; each skips
  // the other's worlds)
  int n_reg = 0;
  if (cr_reg_mode() && cr_common_bytes(std::min(ncap, 1024), 512) + RegOp<256, 4, false>::smem_bytes(std::min(ncap, 1024), nbcap) <= 232448) {
    cudaError_t e;
    if (ncap <= 256) {
      n_reg = 256;
      e = launch_cr_reg_t<128, 2, 4>(bv, sp, worlds, count, ncap, nbcap, s);
    } else if (ncap <= 512) {
      n_reg = 512;
      e = launch_cr_reg_t<256, 2, 2>(bv, sp, worlds, count, ncap, nbcap, s);
    } else {
      // 513..1024 rows: 256 threads with four rows each, one CTA per SM:
      // incidence owners with pieces of <= 8 incidences (254 registers, no
      // spills), row owners for the worlds whose bodies do not fit the lanes.
      // Measured against the 512-thread incidence-owner launch: sphere pile
      // 25.5k -> 33.4k, box pile 173k -> 217k world-steps/s (226k with row
      // owners alone, KD_CR_REG=3); KD_CR_REG=4 restores the 512-thread launch.
      n_reg = 1024;
      if (cr_reg_mode() == 4) e = launch_cr_reg_t<512, 2, 1>(bv, sp, worlds, count, ncap, nbcap, s);
      else if (cr_reg_mode() == 2)
        e = launch_cr_op_p<RegOp<256, 4, true>, 256, 4, 1, true, false>(bv, sp, worlds, count, ncap, nbcap, 0, s);
      else if (cr_reg_mode() == 3)
        e = launch_cr_op_p<RegOp<256, 4, false>, 256, 4, 1, false, false>(bv, sp, worlds, count, ncap, nbcap, 0, s);
      else {
        e = launch_cr_op_p<IncOp<256, 4, 8, false>, 256, 4, 1, false, true>(bv, sp, worlds, count, ncap, nbcap, 0, s);
        if (e == cudaSuccess)
          e = launch_cr_op_p<RegOp<256, 4, false>, 256, 4, 1, false, false>(bv, sp, worlds, count, ncap, nbcap, 1, s);
      }
    }
    if (e != cudaSuccess) return e;
    if (ncap <= n_reg) return cudaSuccess;
  } else if (cr_reg_mode() && ncap > 512 && ncap <= 1024 &&
             cr_common_bytes(ncap, 256) + IncOp<256, 4, 8, false>::smem_bytes(ncap, nbcap) <= 232448) {
    // many bodies (the row owners' per-body staging does not fit, e.g. the
    // 156-body Stewart tower): incidence owners, and the shared-memory kernel
    // for the worlds whose bodies do not fit the lanes (n_reg = -1: it skips
    // the worlds the incidence-owner kernel marked)
    cudaError_t e =
        launch_cr_op_p<IncOp<256, 4, 8, false>, 256, 4, 1, false, true>(bv, sp, worlds, count, ncap, nbcap, 0, s);
    if (e != cudaSuccess) return e;
    // more body pieces than 256 lanes: 512 lanes with pieces of <= 5
    if (cr_common_bytes(ncap, 512) + IncOp<512, 2, KD_INC512_P, false>::smem_bytes(ncap, nbcap) <= 232448) {
      e = launch_cr_op_p<IncOp<512, 2, KD_INC512_P, false>, 512, 2, 1, false, true>(bv, sp, worlds, count, ncap, nbcap, 1, s);
      if (e != cudaSuccess) return e;
    }
    n_reg = -1;
  }
  // two resident CTAs per SM whenever their (staged) shared memory fits: the
  // kernel is synchronisation/latency bound, so a second world hides it
  if (cr_staged_bytes(ncap, nbcap, 256) <= 232448 / 2) {
    if (nt <= 128) return launch_cr_t<128, 2>(bv, sp, worlds, count, ncap, nbcap, n_reg, s);
    return launch_cr_t<256, 2>(bv, sp, worlds, count, ncap, nbcap, n_reg, s);
  }
  if (nt <= 128) return launch_cr_t<128, 1>(bv, sp, worlds, count, ncap, nbcap, n_reg, s);
  if (nt <= 256) return launch_cr_t<256, 1>(bv, sp, worlds, count, ncap, nbcap, n_reg, s);
  return launch_cr_t<512, 1>(bv, sp, worlds, count, ncap, nbcap, n_reg, s);
}

}  // namespace kd
