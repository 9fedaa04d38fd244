// kd_recover.cu — K3: impulse recovery, warm-start caches, KKT diagnostics and
// pose integration, one warp per world.
//
// Restates step() after the solve (stepper.cpp:185-235): lambda = P y,
// z_phys = z / P, store_caches (stepper.cpp:48-70), u+ = u_free + M^-1 J^T lambda
// with J^T lambda accumulated per body in ascending row order
// (apply_jacobian_transpose, constraints.cpp:121-129), the bilateral velocity
// and momentum KKT diagnostics, and the explicit pose update (semi-implicit
// Euler: u+; Moreau-Jean: midpoint 1/2(u- + u+)) with quat_integrate.
#include "kd_device.cuh"

namespace kd {

__global__ void __launch_bounds__(256) recover_kernel(BatchView bv, StepParams sp, int w0, int w1) {
  const int lane = threadIdx.x & 31;
  const int w = w0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= w1) return;
  if (!bv.active[w]) return;
  WorldStep& ws = bv.wstep[w];
  // a world whose solve was skipped this step (contact or slab capacity
  // overflow, fail = 2) or failed (non-SPD factor, fail = 1) keeps its state
  // and caches untouched; the step reports the error (kd_batch_sync)
  if (ws.fail != 0 || (ws.n_rows > 0 && ws.backend == BE_NONE)) return;
  const DevWorld W = bv.worlds[w];
  const DevModel M = bv.models[W.model];
  const int n = ws.n_rows;
  const int n_jd = M.n_bil + M.n_dyn;
  const int first_contact = n_jd + ws.n_limits;
  const int nc = ws.n_contacts;
  const int64_t R0 = W.row_off;
  const RowJ* rj = bv.rowj + R0;
  const int32_t* rb = bv.rbody + 2 * R0;
  const double* scale = bv.scale + R0;
  double* imp = bv.imp + R0;
  BodyS* bs = bv.bs + W.body_off;
  double* pose = bv.poses + W.pose_off;
  double* tw = bv.twists + W.twist_off;
  const double dt = sp.dt;

  // ---- lambda = P y; caches (only when the set is non-empty, stepper.cpp:173-187)
  for (int r = lane; r < n; r += 32) imp[r] = scale[r] * bv.lam[R0 + r];
  if (n > 0) {
    for (int r = lane; r < n_jd; r += 32) {
      bv.jc_lam[W.jcache_off + r] = imp[r];
      bv.jc_z[W.jcache_off + r] = bv.zo[R0 + r] / scale[r];
    }
    for (int s = lane; s < 2 * M.n_limited; s += 32) bv.ls_valid[W.lslot_off + s] = 0;
    __syncwarp();
    for (int r = n_jd + lane; r < first_contact; r += 32) {
      const int ji = bv.lkey[2 * (R0 + r)], bound = bv.lkey[2 * (R0 + r) + 1];
      const int slot = W.lslot_off + 2 * bv.joints[M.joint_off + ji].limit_slot + bound;
      bv.ls_lam[slot] = imp[r];
      bv.ls_z[slot] = bv.zo[R0 + r] / scale[r];
      bv.ls_valid[slot] = 1;
    }
    for (int c = lane; c < nc; c += 32) {
      const Contact& cp = bv.contacts[W.contact_off + c];
      CacheEntry& e = bv.ccache[W.contact_off + c];
      const int r = first_contact + 3 * c;
      e.ga = cp.ga;
      e.gb = cp.gb;
      e.pair = cp.pair;  // the cache stays sorted by pair (contact order): K1 finds a pair's entries by bisection
      for (int d = 0; d < 3; ++d) {
        e.pos[d] = cp.pos[d];
        e.imp[d] = imp[r + d];
        e.dual[d] = bv.zo[R0 + r + d] / scale[r + d];
      }
    }
    if (lane == 0) {
      ws.jcache_valid = 1;
      ws.ccache_count = nc;
    }
  }
  __syncwarp();

  // ---- per body: J^T lambda, u+, KKT momentum, integration
  const int32_t* cptr = bv.csr_ptr + W.body_off + w;
  const int32_t* clist = bv.csr + 2 * R0;
  double kkt = 0.0;
  for (int b = lane; b < M.nb; b += 32) {
    BodyS& B = bs[b];
    double wr[6] = {0, 0, 0, 0, 0, 0};
    for (int e = cptr[b]; e < cptr[b + 1]; ++e) {
      const int code = clist[e];
      const int r = code >> 1;
      const double* J = rj[r].J + 6 * (code & 1);
      const double l = imp[r];
#pragma unroll
      for (int k = 0; k < 6; ++k) wr[k] += J[k] * l;
    }
    double up[6], um[6];
    for (int k = 0; k < 6; ++k) {
      um[k] = tw[6 * b + k];
      up[k] = B.uf[k];
    }
    if (n > 0) {
      const M3 Iwinv = ldm(B.Iwinv);
      const V3 da = mvec(Iwinv, V3{wr[3], wr[4], wr[5]});
      for (int k = 0; k < 3; ++k) up[k] += B.inv_mass * wr[k];
      up[3] += da.x;
      up[4] += da.y;
      up[5] += da.z;
    }
    // M (u+ - u-) = dt h + J^T lambda   (stepper.cpp:207-216)
    const V3 ml = scl(B.mass, V3{up[0] - um[0], up[1] - um[1], up[2] - um[2]});
    const V3 ma = mvec(ldm(B.Iw), V3{up[3] - um[3], up[4] - um[4], up[5] - um[5]});
    for (int k = 0; k < 3; ++k) {
      kkt = fmax(kkt, fabs((-dt * B.h[k] - wr[k]) + comp(ml, k)));
      kkt = fmax(kkt, fabs((-dt * B.h[3 + k] - wr[3 + k]) + comp(ma, k)));
    }
    for (int k = 0; k < 6; ++k) B.up[k] = up[k];
    // integrate from the start-of-step pose (stepper.cpp:218-233)
    V3 vi{up[0], up[1], up[2]}, wi{up[3], up[4], up[5]};
    if (sp.moreau) {
      vi = scl(0.5, V3{um[0] + up[0], um[1] + up[1], um[2] + up[2]});
      wi = scl(0.5, V3{um[3] + up[3], um[4] + up[4], um[5] + up[5]});
    }
    double* p = pose + 7 * b;
    const V3 x = add(V3{p[0], p[1], p[2]}, scl(dt, vi));
    const Q4 q{p[3], p[4], p[5], p[6]};
    const Q4 qn = quat_integrate(q, mtvec(qrot(q), wi), dt);
    p[0] = x.x;
    p[1] = x.y;
    p[2] = x.z;
    p[3] = qn.w;
    p[4] = qn.x;
    p[5] = qn.y;
    p[6] = qn.z;
    for (int k = 0; k < 6; ++k) tw[6 * b + k] = up[k];
  }
  kkt = warp_max(kkt);
  __syncwarp();

  // ---- bilateral KKT row: |P (J u+ + R lambda - v*)| over n_jd rows (stepper.cpp:195-203)
  double bv_inf = 0.0;
  if (n > 0) {
    for (int r = lane; r < n_jd; r += 32) {
      const int ba = rb[2 * r], bb = rb[2 * r + 1];
      double s = 0.0;
      if (ba >= 0) {
        double t = 0.0;
        for (int k = 0; k < 6; ++k) t += rj[r].J[k] * bs[ba].up[k];
        s += t;
      }
      if (bb >= 0) {
        double t = 0.0;
        for (int k = 0; k < 6; ++k) t += rj[r].J[6 + k] * bs[bb].up[k];
        s += t;
      }
      bv_inf = fmax(bv_inf, scale[r] * fabs(s + bv.reg[R0 + r] * imp[r] - bv.bias[R0 + r]));
    }
  }
  bv_inf = warp_max(bv_inf);
  if (lane == 0) {
    ws.kkt = kkt;
    ws.bil_vel = bv_inf;
    bv.time[w] += dt;
  }
}

void launch_recover(const BatchView& bv, const StepParams& sp, cudaStream_t s, int w0, int w1) {
  const int wpb = 8;
  if (w1 < 0) w1 = bv.n_worlds;
  const int grid = (w1 - w0 + wpb - 1) / wpb;
  if (grid > 0) recover_kernel<<<grid, 32 * wpb, 0, s>>>(bv, sp, w0, w1);
}

}  // namespace kd
