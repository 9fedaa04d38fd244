// kd_solve.cu — solver-level entry points on pre-assembled systems:
// kd_padmm_solve_batched (build_backend + padmm_solve, delassus.hpp:103-105,
// padmm.hpp:64-67) and kd_cr_solve_batched (bake_jacobian + cr_solve,
// delassus.hpp:82-83).
//
// A set of problems is laid out exactly like the step path's per-world row
// slabs (kd_layout.h), so the solve runs through the same device kernels as a
// batch step: the fused dense kernel (shared-memory classes, or the HBM-slab
// variant above 232 rows) and the matrix-free CR kernels.  A prep kernel (one
// warp per problem) folds M^-1 into the rows (JM, fold_inverse_mass,
// delassus.cpp:12-17) and builds the per-body incidence lists that fix the
// reference's accumulation order.
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "kd_device.cuh"
#include "kd_host.h"

namespace kd {

__global__ void __launch_bounds__(256) solve_prep_kernel(BatchView bv) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= bv.n_worlds) return;
  const DevWorld W = bv.worlds[w];
  const int n = bv.wstep[w].n_rows;
  const int64_t R0 = W.row_off;
  RowJ* rj = bv.rowj + R0;
  const int32_t* rb = bv.rbody + 2 * R0;
  const BodyS* bs = bv.bs + W.body_off;
  for (int r = lane; r < n; r += 32) {
    RowJ& R = rj[r];
    for (int side = 0; side < 2; ++side) {
      const int b = rb[2 * r + side];
      double* jm = R.JM + 6 * side;
      const double* J = R.J + 6 * side;
      if (b < 0) {
        for (int k = 0; k < 6; ++k) jm[k] = 0.0;
        continue;
      }
      const double im = bs[b].inv_mass;
      const V3 t = vmat(V3{J[3], J[4], J[5]}, ldm(bs[b].Iwinv));
      jm[0] = J[0] * im;
      jm[1] = J[1] * im;
      jm[2] = J[2] * im;
      jm[3] = t.x;
      jm[4] = t.y;
      jm[5] = t.z;
    }
  }
  __syncwarp();
  int32_t* cptr = bv.csr_ptr + W.body_off + w;
  const int run = warp_incidence_lists(rb, n, W.nb, cptr, bv.csr + 2 * R0, lane);
  if (lane == 0) cptr[W.nb] = run;
}

namespace {

constexpr int kClasses[4][2] = {{32, 64}, {64, 64}, {128, 128}, {232, 256}};

struct Dev {
  std::vector<void*> ptrs;
  ~Dev() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class U, class T>
  cudaError_t up(U*& dst, const std::vector<T>& v) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(1, v.size()) * sizeof(T));
    if (e != cudaSuccess) return e;
    ptrs.push_back(p);
    dst = static_cast<U*>(p);
    if (!v.empty()) e = cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
    return e;
  }
  template <class T>
  cudaError_t zeros(T*& dst, size_t n) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T));
    if (e != cudaSuccess) return e;
    ptrs.push_back(p);
    dst = static_cast<T*>(p);
    return cudaMemset(p, 0, std::max<size_t>(1, n) * sizeof(T));
  }
};

#define KS_CK(x)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) return set_last_error(KD_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Problems laid out as worlds of a BatchView (rows, bodies, incidence lists).
struct SolveSet {
  Dev dev;
  BatchView v{};
  std::vector<int64_t> row_off;
  std::vector<WorldStep> ws;
  std::vector<DevWorld> worlds;
  int64_t R = 0;
  int nbmax = 0, nmax = 0;
  double* d_hist = nullptr;
  int32_t* d_err = nullptr;
  double* d_nest = nullptr;
};

int validate(const kd_solve_problem* P, int np) {
  if (np < 0 || (np > 0 && !P)) return set_last_error(KD_ERR_INVALID_ARGUMENT, "invalid problem list");
  for (int p = 0; p < np; ++p) {
    const kd_solve_problem& q = P[p];
    const std::string at = "problem " + std::to_string(p) + ": ";
    if (q.n_rows < 0 || q.n_bodies < 0 || q.n_bilateral < 0 || q.n_limits < 0 || q.n_contacts < 0 ||
        q.n_bilateral + q.n_limits + 3 * q.n_contacts != q.n_rows)
      return set_last_error(KD_ERR_INVALID_ARGUMENT, at + "n_bilateral + n_limits + 3 n_contacts != n_rows");
    if (q.n_rows > 0 && (!q.body || !q.jacobian || !q.reg || !q.scale || !q.rhs))
      return set_last_error(KD_ERR_INVALID_ARGUMENT, at + "null row array");
    if (q.n_bodies > 0 && (!q.inv_mass || !q.inv_inertia))
      return set_last_error(KD_ERR_INVALID_ARGUMENT, at + "null inertia array");
    if (q.n_contacts > 0 && !q.mu) return set_last_error(KD_ERR_INVALID_ARGUMENT, at + "null mu");
    for (int r = 0; r < 2 * q.n_rows; ++r)
      if (q.body[r] < -1 || q.body[r] >= q.n_bodies)
        return set_last_error(KD_ERR_INVALID_ARGUMENT, at + "body index out of range");
  }
  return KD_OK;
}

// Upload the problems; backend[p] is the Backend each world takes.
int build_set(SolveSet& S, const kd_solve_problem* P, int np, const std::vector<int>& backend, int hist_cap,
              const std::vector<double>& nest) {
  S.row_off.assign(np + 1, 0);
  int64_t nbod = 0;
  std::vector<RowJ> rowj;
  std::vector<int32_t> rbody, rkind;
  std::vector<double> rmu, reg, scale, vf, x0, z0;
  std::vector<BodyS> bs;
  int64_t total_slab = 0;
  for (int p = 0; p < np; ++p) {
    const kd_solve_problem& q = P[p];
    const int n = q.n_rows;
    S.row_off[p + 1] = S.row_off[p] + n;
    DevWorld W{};
    W.model = 0;
    W.nb = q.n_bodies;
    W.row_off = S.row_off[p];
    W.body_off = (int)nbod;
    W.lslab_off = -1;
    W.snlv_off = -1;
    W.xslab_off = -1;
    W.snr2p_off = -1;
    W.smem_cap = 0;
    for (int c = 0; c < 4; ++c)
      if (n <= kClasses[c][0]) {
        W.bin = c;
        W.smem_cap = kClasses[c][0];
        break;
      }
    if (backend[p] == BE_DENSE_GLOBAL) {
      W.slab_cap = n;
      W.lslab_off = total_slab;
      const int64_t t = (n + 31) / 32;
      total_slab += (((int64_t)dense_factor_doubles(n) + 1) & ~(int64_t)1) + 4 * 32 * t + 2;
    }
    S.worlds.push_back(W);
    WorldStep s{};
    s.n_rows = n;
    s.n_limits = q.n_limits;
    s.n_contacts = q.n_contacts;
    s.backend = n > 0 ? backend[p] : BE_NONE;
    S.ws.push_back(s);
    nbod += q.n_bodies;
    S.nbmax = std::max(S.nbmax, q.n_bodies);
    S.nmax = std::max(S.nmax, n);
    const int fc = q.n_bilateral + q.n_limits;
    for (int r = 0; r < n; ++r) {
      RowJ J{};
      for (int k = 0; k < 12; ++k) J.J[k] = q.jacobian[12 * (size_t)r + k];
      rowj.push_back(J);
      rbody.push_back(q.body[2 * r]);
      rbody.push_back(q.body[2 * r + 1]);
      rkind.push_back(r < q.n_bilateral ? ROW_BILATERAL : (r < fc ? ROW_LIMIT : ROW_CONTACT));
      rmu.push_back(r < fc ? 0.0 : q.mu[(r - fc) / 3]);
      reg.push_back(q.reg[r]);
      scale.push_back(q.scale[r]);
      vf.push_back(q.rhs[r]);
      x0.push_back(q.x0 ? q.x0[r] : 0.0);
      z0.push_back(q.z0 ? q.z0[r] : 0.0);
    }
    for (int b = 0; b < q.n_bodies; ++b) {
      BodyS B{};
      B.inv_mass = q.inv_mass[b];
      B.mass = B.inv_mass != 0.0 ? 1.0 / B.inv_mass : 0.0;
      for (int k = 0; k < 9; ++k) B.Iwinv[k] = q.inv_inertia[9 * (size_t)b + k];
      bs.push_back(B);
    }
  }
  S.R = S.row_off[np];
  BatchView& v = S.v;
  v.n_worlds = np;
  v.hist_cap = hist_cap;
  KS_CK(S.dev.up(v.worlds, S.worlds));
  KS_CK(S.dev.up(v.wstep, S.ws));
  KS_CK(S.dev.up(v.rowj, rowj));
  KS_CK(S.dev.up(v.rbody, rbody));
  KS_CK(S.dev.up(v.rkind, rkind));
  KS_CK(S.dev.up(v.rmu, rmu));
  KS_CK(S.dev.up(v.reg, reg));
  KS_CK(S.dev.up(v.scale, scale));
  KS_CK(S.dev.up(v.vf, vf));
  KS_CK(S.dev.up(v.x0, x0));
  KS_CK(S.dev.up(v.z0, z0));
  KS_CK(S.dev.up(v.bs, bs));
  KS_CK(S.dev.zeros(v.lam, S.R));
  KS_CK(S.dev.zeros(v.zo, S.R));
  KS_CK(S.dev.zeros(v.imp, S.R));
  KS_CK(S.dev.zeros(v.csr_ptr, nbod + np));
  KS_CK(S.dev.zeros(v.csr, 2 * S.R));
  KS_CK(S.dev.zeros(v.lslab, total_slab));
  KS_CK(S.dev.zeros(S.d_hist, (size_t)std::max(1, hist_cap) * std::max(1, np)));
  KS_CK(S.dev.zeros(S.d_err, 4));
  KS_CK(S.dev.up(S.d_nest, nest));
  v.hist = S.d_hist;
  v.error_count = S.d_err;
  if (np > 0) solve_prep_kernel<<<(np + 7) / 8, 256>>>(v);
  KS_CK(cudaGetLastError());
  return KD_OK;
}

// Nesterov beta table (padmm.cpp:54-71), as ensure_nest_table in kd_capi.cu.
std::vector<double> nest_table(int max_iters) {
  const int cap = std::max(256, max_iters);
  std::vector<double> t(cap);
  double a = 1.0;
  for (int m = 0; m < cap; ++m) {
    volatile double q = 4.0 * a * a;
    const double a_next = 0.5 * (1.0 + std::sqrt(1.0 + q));
    t[m] = (a - 1.0) / a_next;
    a = a_next;
  }
  return t;
}

StepParams params(const kd_step_config* c, double eta_rho, int cr_iters, const double* nest) {
  StepParams sp{};
  sp.dt = c->dt;
  sp.eta = c->eta;
  sp.rho = c->rho;
  sp.eps = c->eps;
  sp.max_iters = c->max_iters;
  sp.acceleration = c->acceleration;
  sp.restart = c->restart;
  sp.fixed_mode = c->fixed_iteration_mode;
  sp.cr_iters = cr_iters;
  sp.backend = KD_BACKEND_AUTO;
  sp.eta_rho = eta_rho;
  sp.nest_beta = nest;
  return sp;
}

}  // namespace
}  // namespace kd

using namespace kd;

extern "C" {

int kd_padmm_solve_batched(int32_t device, const kd_solve_problem* P, int32_t np, double eta_rho, int32_t backend,
                           int32_t cr_budget, const kd_step_config* cfg, double* lambda, double* z,
                           kd_step_diag* diags, double* history, int32_t hcap) {
  if (!cfg || (np > 0 && (!lambda || !z || !diags)) || hcap < 0 || cr_budget < 0 ||
      backend < KD_BACKEND_DENSE || backend > KD_BACKEND_AUTO || !(eta_rho > 0.0) || cfg->max_iters < 0)
    return set_last_error(KD_ERR_INVALID_ARGUMENT, "invalid arguments");
  int rc = validate(P, np);
  if (rc != KD_OK) return rc;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_last_error(KD_ERR_NO_DEVICE, "no CUDA device visible: the B200 solver has no CPU fallback");
  if (device < 0 || device >= ndev) return set_last_error(KD_ERR_INVALID_ARGUMENT, "device index out of range");
  KS_CK(cudaSetDevice(device));
  // build_backend's choice (delassus.cpp:199-206) per problem
  std::vector<int> be(np);
  std::vector<int32_t> cls[4], glob, cr;
  for (int p = 0; p < np; ++p) {
    const int n = P[p].n_rows;
    const bool dense = backend == KD_BACKEND_DENSE || (backend == KD_BACKEND_AUTO && n <= KD_DENSE_ROW_CROSSOVER);
    be[p] = !dense ? BE_MATRIX_FREE : (n <= 232 ? BE_DENSE_SMEM : BE_DENSE_GLOBAL);
    if (n == 0) continue;
    if (be[p] == BE_MATRIX_FREE) cr.push_back(p);
    else if (be[p] == BE_DENSE_GLOBAL) glob.push_back(p);
    else
      for (int c = 0; c < 4; ++c)
        if (n <= kClasses[c][0]) {
          cls[c].push_back(p);
          break;
        }
  }
  SolveSet S;
  rc = build_set(S, P, np, be, hcap, nest_table(cfg->max_iters));
  if (rc != KD_OK) return rc;
  const StepParams sp = params(cfg, eta_rho, cr_budget, S.d_nest);
  int32_t* lists = nullptr;
  std::vector<int32_t> all;
  for (int c = 0; c < 4; ++c) all.insert(all.end(), cls[c].begin(), cls[c].end());
  all.insert(all.end(), glob.begin(), glob.end());
  all.insert(all.end(), cr.begin(), cr.end());
  KS_CK(S.dev.up(lists, all));
  int off = 0;
  for (int c = 0; c < 4; ++c) {
    KS_CK(launch_dense(S.v, sp, lists + off, (int)cls[c].size(), kClasses[c][0], kClasses[c][1], false, 0));
    off += (int)cls[c].size();
  }
  if (!glob.empty()) {
    int cap = 0;
    for (int p : glob) cap = std::max(cap, P[p].n_rows);
    KS_CK(launch_dense(S.v, sp, lists + off, (int)glob.size(), cap, 256, true, 0));
  }
  off += (int)glob.size();
  if (!cr.empty()) {
    int ncap = 0, nbcap = 0;
    for (int p : cr) ncap = std::max(ncap, P[p].n_rows), nbcap = std::max(nbcap, P[p].n_bodies);
    if (cr_smem_bytes(ncap, nbcap, 512) > 232448)
      return set_last_error(KD_ERR_CAPACITY, "matrix-free path: system too large for one CTA's shared memory");
    KS_CK(launch_cr(S.v, sp, lists + off, (int)cr.size(), ncap, nbcap,
                    ncap > 256 ? 512 : (ncap > 128 ? 256 : 128), 0));
  }
  KS_CK(cudaStreamSynchronize(0));  // the launches above are on the legacy stream
  int32_t err[4];
  KS_CK(cudaMemcpy(err, S.d_err, 16, cudaMemcpyDeviceToHost));
  if (err[0])
    return set_last_error(KD_ERR_SPD_FAILURE, "Delassus factorization failed on an SPD system (" +
                                                  std::to_string(err[0]) + " problems)");
  if (S.R) {
    KS_CK(cudaMemcpy(lambda, S.v.lam, 8 * (size_t)S.R, cudaMemcpyDeviceToHost));
    KS_CK(cudaMemcpy(z, S.v.zo, 8 * (size_t)S.R, cudaMemcpyDeviceToHost));
  }
  std::vector<WorldStep> ws(np);
  if (np) KS_CK(cudaMemcpy(ws.data(), S.v.wstep, sizeof(WorldStep) * np, cudaMemcpyDeviceToHost));
  for (int p = 0; p < np; ++p) {
    kd_step_diag& o = diags[p];
    o = kd_step_diag{};
    o.n_rows = P[p].n_rows;
    o.n_limits = P[p].n_limits;
    o.contact_count = P[p].n_contacts;
    o.first_contact_row = P[p].n_bilateral + P[p].n_limits;
    if (P[p].n_rows == 0) {  // padmm_solve's early return (padmm.cpp:89-93)
      o.converged = 1;
      continue;
    }
    o.iterations = ws[p].iterations;
    o.restarts = ws[p].restarts;
    o.converged = ws[p].converged;
    o.cr_breakdown = ws[p].cr_breakdown;
    o.cr_iterations = ws[p].cr_iterations;
    o.r_p = ws[p].r_p;
    o.r_d = ws[p].r_d;
    o.r_c = ws[p].r_c;
  }
  if (history && hcap && np) {
    KS_CK(cudaMemcpy(history, S.d_hist, 8 * (size_t)hcap * np, cudaMemcpyDeviceToHost));
    for (int p = 0; p < np; ++p)
      if (P[p].n_rows == 0)
        for (int i = 0; i < hcap; ++i) history[(size_t)p * hcap + i] = -1.0;
  }
  return KD_OK;
}

int kd_cr_solve_batched(int32_t device, const kd_solve_problem* P, int32_t np, double eta_rho, int32_t max_iters,
                        double* x, int32_t* iterations, uint8_t* breakdown, double* residual_norm, double* history,
                        int32_t hcap) {
  if ((np > 0 && !x) || max_iters < 0 || hcap < 0 || eta_rho < 0.0)
    return set_last_error(KD_ERR_INVALID_ARGUMENT, "invalid arguments");
  int rc = validate(P, np);
  if (rc != KD_OK) return rc;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_last_error(KD_ERR_NO_DEVICE, "no CUDA device visible: the B200 solver has no CPU fallback");
  if (device < 0 || device >= ndev) return set_last_error(KD_ERR_INVALID_ARGUMENT, "device index out of range");
  KS_CK(cudaSetDevice(device));
  std::vector<int> be(np, BE_MATRIX_FREE);
  std::vector<int32_t> todo;
  int ncap = 0, nbcap = 0;
  for (int p = 0; p < np; ++p) {
    if (P[p].n_rows == 0) continue;
    todo.push_back(p);
    ncap = std::max(ncap, P[p].n_rows);
    nbcap = std::max(nbcap, P[p].n_bodies);
  }
  if (cr_smem_bytes(ncap, nbcap, 256) > 232448)
    return set_last_error(KD_ERR_CAPACITY, "cr_solve: system too large for one CTA's shared memory");
  SolveSet S;
  kd_step_config c;
  kd_step_config_default(&c);
  rc = build_set(S, P, np, be, hcap, nest_table(1));
  if (rc != KD_OK) return rc;
  StepParams sp = params(&c, eta_rho, max_iters, S.d_nest);
  sp.cr_only = 1;
  int32_t* list = nullptr;
  KS_CK(S.dev.up(list, todo));
  KS_CK(launch_cr_shared(S.v, sp, list, (int)todo.size(), ncap, nbcap, 0));
  KS_CK(cudaStreamSynchronize(0));  // the launches above are on the legacy stream
  if (S.R) KS_CK(cudaMemcpy(x, S.v.lam, 8 * (size_t)S.R, cudaMemcpyDeviceToHost));
  std::vector<WorldStep> ws(np);
  if (np) KS_CK(cudaMemcpy(ws.data(), S.v.wstep, sizeof(WorldStep) * np, cudaMemcpyDeviceToHost));
  if (history && hcap && np) KS_CK(cudaMemcpy(history, S.d_hist, 8 * (size_t)hcap * np, cudaMemcpyDeviceToHost));
  for (int p = 0; p < np; ++p) {
    const bool empty = P[p].n_rows == 0;
    if (iterations) iterations[p] = empty ? 0 : (int32_t)ws[p].cr_iterations;
    if (breakdown) breakdown[p] = empty ? (max_iters > 0 ? 1 : 0) : (uint8_t)ws[p].cr_breakdown;
    if (residual_norm) residual_norm[p] = empty ? 0.0 : ws[p].r_p;
    if (empty && history)
      for (int i = 0; i < hcap; ++i) history[(size_t)p * hcap + i] = i == 0 ? 0.0 : -1.0;
  }
  return KD_OK;
}

}  // extern "C"
