// kd_sparse.cu — K2s: supernodal sparse-LLT path, one warp per world.
//
// Same mathematics as K2 (kd_dense.cu) — the reference's Dense backend:
//   assemble_dense  D = P (J M^-1 J^T + R) P + (eta+rho) I   (delassus.cpp:67-104)
//   DenseDelassus   D = L L^T once per step, two triangular solves per PADMM
//                   iteration                              (delassus.cpp:59-65)
//   padmm_solve     De Saxce shift, solve, cone projection, dual update,
//                   residual triple, Nesterov with restart (padmm.cpp:87-159)
// but D is factored in the fill-reducing order of the model's static plan
// (kd_snplan.h): for DR-Legs nnz(L) = 3.6k instead of n^2/2 = 24.6k and the
// factor costs ~40k FMA instead of 1.8M.  Everything a world needs (panels,
// X blocks, PADMM vectors) fits in ~55 KB of shared memory, so one warp owns
// one world for the whole solve and a CTA holds several worlds of one model
// plus one shared copy of the model's solve program.  After the program copy
// (one __syncthreads) all synchronisation is __syncwarp.
//
// Shared memory: [solve program blob] then per warp (doubles):
//   Lv[nLv] | v[S] | t[S] | vf y z yh zh [S each] (Gram: row-block staging + P) | part[max_slots]
//   | int16 row2pos[S] | int16 slot2row[S]
#include "kd_device.cuh"

namespace kd {

namespace {

constexpr unsigned FULL = 0xffffffffu;


__device__ __forceinline__ int pad2(int x) { return (x + 1) & ~1; }

}  // namespace

__global__ void __launch_bounds__(256, 3) sparse_kernel(BatchView bv, StepParams sp, const int32_t* worlds, int count,
                                                        int per_warp, int prog_words) {
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int slot_idx = blockIdx.x * (blockDim.x >> 5) + wid;
  // the CTA's worlds share one model: stage its solve program once
  uint32_t* prog = reinterpret_cast<uint32_t*>(smem);
  {
    const int w0 = worlds[blockIdx.x * (blockDim.x >> 5)];
    const DevSnPlan P0 = bv.snplan[bv.worlds[w0].model];
    const uint4* src = reinterpret_cast<const uint4*>(bv.sn_prog + P0.prog_off);
    uint4* dst = reinterpret_cast<uint4*>(prog);
    for (int i = threadIdx.x; i < (prog_words + 3) / 4; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  if (slot_idx >= count) return;
  const int w = worlds[slot_idx];
  WorldStep& ws = bv.wstep[w];
  if (ws.backend != BE_SPARSE) return;
  const DevWorld W = bv.worlds[w];
  const DevSnPlan P = bv.snplan[W.model];
  const DevModel M = bv.models[W.model];
  const int S = P.S, Sp = pad2(S);
  double* Lv = smem + ((prog_words + 3) / 4) * 2 + (size_t)wid * per_warp;
  double* v = Lv + pad2(P.nLv);
  double* t = v + Sp;
  double* vf_s = t + Sp;
  double* y_s = vf_s + Sp;
  double* z_s = y_s + Sp;
  double* yh_s = z_s + Sp;
  double* zh_s = yh_s + Sp;
  const int vreg = P.vreg;
  double* part = v + vreg;
  int16_t* row2pos = reinterpret_cast<int16_t*>(part + P.max_slots);
  int16_t* slot2row = row2pos + Sp;

  const int64_t R0 = W.row_off;
  const int n = ws.n_rows;
  const int n_lim = ws.n_limits, nc = ws.n_contacts;
  const int n_jd = P.n_jd;
  const int first_contact = n_jd + n_lim;
  const uint16_t* slot_pos = bv.sn_slot_pos + P.slotpos_off;
  long long t_prev = clock64();
  auto stamp = [&](int k) {
    if (lane == 0) {
      const long long tc = clock64();
      ws.phase_cycles[k] = tc - t_prev;
      t_prev = tc;
    }
  };

  // ---- 0. zero the factor array, map compact rows <-> planned slots
  for (int e = lane; e < P.nLv; e += 32) Lv[e] = 0.0;
  for (int s = lane; s < S; s += 32) slot2row[s] = s < n_jd ? (int16_t)s : (int16_t)-1;
  for (int r = lane; r < n_jd; r += 32) row2pos[r] = (int16_t)slot_pos[r];
  __syncwarp();
  {
    const int32_t* lk = bv.lkey + 2 * R0;
    const DevJoint* mj = bv.joints + M.joint_off;
    for (int r = n_jd + lane; r < first_contact; r += 32) {  // limit rows: (joint, bound) -> slot
      const int slot = P.lim_base + 2 * mj[lk[2 * r]].limit_slot + lk[2 * r + 1];
      slot2row[slot] = (int16_t)r;
      row2pos[r] = (int16_t)slot_pos[slot];
    }
    const Contact* ct = bv.contacts + W.contact_off;
    const int32_t* pslot = bv.sn_pair_slot + P.pair_off;
    for (int c = lane; c < nc; c += 32) {  // contacts: (pair, index within the pair) -> slot
      const int pr = ct[c].pair;
      int k = 0;
      while (c - k - 1 >= 0 && ct[c - k - 1].pair == pr) ++k;
      const int slot = pslot[pr] + 3 * k;
      for (int d = 0; d < 3; ++d) {
        slot2row[slot + d] = (int16_t)(first_contact + 3 * c + d);
        row2pos[first_contact + 3 * c + d] = (int16_t)slot_pos[slot + d];
      }
    }
  }
  __syncwarp();

  // ---- 1. Gram D = P (J M^-1 J^T + R) P + (eta+rho) I (delassus.cpp:67-104),
  // body by body in ascending order: stage the body's row blocks (JM and J of
  // the side touching it; inactive slots stage zeros), then every planned pair
  // of its rows is written (first shared body) or added (second).
  {
    const RowJ* rj = bv.rowj + R0;
    double* stJM = v;                      // scratch: the PADMM vectors are not live yet
    double* stJ = v + 6 * P.kmax;
    double* Ps = v + vreg - Sp;            // P per compact row
    for (int r = lane; r < n; r += 32) Ps[r] = bv.scale[R0 + r];
    const SnGBody* gbl = bv.sn_gbody + P.gbody_off;
    for (int b = 0; b < P.n_gbody; ++b) {
      const SnGBody gb = gbl[b];
      for (int l = lane; l < gb.k; l += 32) {
        const uint32_t e = bv.sn_gslot[gb.slot_off + l];
        const int r = slot2row[e & 0xffff];
        const int off = (e >> 16) ? 6 : 0;
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          stJM[6 * l + k] = r >= 0 ? rj[r].JM[off + k] : 0.0;
          stJ[6 * l + k] = r >= 0 ? rj[r].J[off + k] : 0.0;
        }
      }
      __syncwarp();
      const uint32_t* pw = bv.sn_gpair + gb.pair_off;
      for (int e = lane; e < gb.n_store + gb.n_acc; e += 32) {
        const uint32_t q = pw[e];
        const double* a = stJM + 6 * ((q >> 16) & 0xff);
        const double* c = stJ + 6 * (q >> 24);
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 6; ++k) s += a[k] * c[k];
        if (e < gb.n_store) Lv[q & 0xffff] = s;
        else Lv[q & 0xffff] += s;
      }
      __syncwarp();
    }
    // + R on the diagonal, P scaling, + (eta+rho) I; inactive slots -> identity
    const double* reg = bv.reg + R0;
    const double eta_rho = sp.eta_rho;
    const SnGram* gl = bv.sn_gram + P.gram_off;
    for (int e = lane; e < P.n_gram; e += 32) {
      const SnGram g = gl[e];
      const int rs = slot2row[g.s], rt = slot2row[g.t];
      const bool diag = g.flags & SG_DIAG;
      if (rs < 0 || rt < 0) {
        if (diag) Lv[g.dst] = 1.0;
        continue;
      }
      double s = Lv[g.dst];
      if (diag) s += reg[rs];
      double d = (Ps[rs] * s) * Ps[rt];
      if (diag) d += eta_rho;
      Lv[g.dst] = d;
    }
    __syncwarp();
    for (int s = lane; s < S; s += 32) v[s] = 0.0;  // inactive positions stay zero through every solve
  }
  __syncwarp();
  stamp(0);

  // ---- 2. supernodal right-looking Cholesky (postorder; one warp, so every
  // entry accumulates its updates in one fixed order) + X = L_SS^-1 per block
  {
    bool bad = false;
    const SnSuper* sup = bv.sn_sup + P.sup_off;
    for (int k = 0; k < P.n_sup; ++k) {
      const SnSuper u = sup[k];
      double* Pn = Lv + u.pb;
      double* X = Lv + u.xb;
      const int rows = u.w + u.m;
      for (int c = 0; c < u.w; ++c) {
        double* col = Pn + c * u.ld;
        const double d = col[c];
        if (!(d > 0.0)) bad = true;
        const double r = fast_rsqrt(d);
        for (int q = c + 1 + lane; q < rows; q += 32) col[q] *= r;
        __syncwarp();
        if (lane == 0) X[c * u.ws + c] = r;  // X (= L_SS^-1, transposed into the upper triangle) keeps 1/L_cc
        // trailing update of the panel's remaining columns
        for (int q = c + 1 + lane; q < rows; q += 32) {
          const double lq = col[q];
          const int jmax = min(q, u.w - 1);
          int j = c + 1;
          for (; j + 3 <= jmax; j += 4) {  // loads first: the stores cannot alias them
            const double c0 = col[j], c1 = col[j + 1], c2 = col[j + 2], c3 = col[j + 3];
            double* p0 = Pn + j * u.ld + q;
            const double p00 = p0[0], p01 = p0[u.ld], p02 = p0[2 * u.ld], p03 = p0[3 * u.ld];
            p0[0] = p00 - lq * c0;
            p0[u.ld] = p01 - lq * c1;
            p0[2 * u.ld] = p02 - lq * c2;
            p0[3 * u.ld] = p03 - lq * c3;
          }
          for (; j <= jmax; ++j) Pn[j * u.ld + q] -= lq * col[j];
        }
        __syncwarp();
      }
      // X = L_SS^-1, lane j owns column j (X_ij = -(sum_{q=j}^{i-1} L_iq X_qj) / L_ii)
      if (lane < u.w) {
        const int j = lane;
        for (int i = j + 1; i < u.w; ++i) {
          double s0 = 0.0, s1 = 0.0;
          int q = j;
          for (; q + 1 < i; q += 2) {
            s0 += Pn[q * u.ld + i] * X[q * u.ws + j];
            s1 += Pn[(q + 1) * u.ld + i] * X[(q + 1) * u.ws + j];
          }
          if (q < i) s0 += Pn[q * u.ld + i] * X[q * u.ws + j];
          X[i * u.ws + j] = -(s0 + s1) * X[i * u.ws + i];
        }
      }
      // ancestors: A_ij -= sum_c L_ic L_jc for i >= j in the row structure
      const int T = u.m * (u.m + 1) / 2;
      const uint32_t* tm = bv.sn_tmap + u.tmap_off;
      for (int e = lane; e < T; e += 32) {
        const uint32_t te = tm[e];
        const double* a = Pn + u.w + ((te >> 16) & 0xff);
        const double* b = Pn + u.w + (te >> 24);
        double s0 = 0.0, s1 = 0.0;
        int c = 0;
        for (; c + 1 < u.w; c += 2) {
          s0 += a[c * u.ld] * b[c * u.ld];
          s1 += a[(c + 1) * u.ld] * b[(c + 1) * u.ld];
        }
        if (c < u.w) s0 += a[c * u.ld] * b[c * u.ld];
        Lv[te & 0xffff] -= s0 + s1;
      }
      __syncwarp();
    }
    if (__any_sync(FULL, bad) && lane == 0) {
      ws.fail = 1;
      atomicAdd(bv.error_count, 1);
    }
  }
  stamp(2);

  // ---- 3. PADMM (padmm.cpp:87-159); units = bilateral/limit rows and contact triples.
  // The solve result x stays in v (at the row's position) until the same lane
  // overwrites it with the next right-hand side.  Nesterov's extrapolation is
  // formed in the projection pass with the no-restart coefficient and undone
  // in the rhs pass on a restart, so no previous-iterate vectors are kept.
  const int n_units = first_contact + nc;
  const double eta = sp.eta, rho = sp.rho;
  const double inv_rho = 1.0 / rho;  // w = x - z_hat * (1/rho): no division in the loop
  const double* rmu = bv.rmu + R0;
  for (int u = lane; u < n_units; u += 32) {
    const bool con = u >= first_contact;
    const int r0 = con ? first_contact + 3 * (u - first_contact) : u;
    const int nr = con ? 3 : 1;
    double x[3] = {0, 0, 0}, y[3] = {0, 0, 0}, zz[3] = {0, 0, 0};
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d < nr) {
        x[d] = bv.x0[R0 + r0 + d];
        vf_s[r0 + d] = bv.vf[R0 + r0 + d];
        zz[d] = bv.z0[R0 + r0 + d];
        z_s[r0 + d] = zz[d];
        zh_s[r0 + d] = zz[d];
      }
    if (con) project_soc(x, rmu[r0], 1.0 / (1.0 + rmu[r0] * rmu[r0]), y);  // y = Pi_K(x0)
    else y[0] = u >= n_jd ? fmax(0.0, x[0]) : x[0];
    // rhs = -(v_f + s - eta x - rho y_hat - z_hat)   (padmm.cpp:116-117)
    const double s0 = con ? rmu[r0] * fast_sqrt(zz[1] * zz[1] + zz[2] * zz[2]) : 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d < nr) {
        y_s[r0 + d] = y[d];
        yh_s[r0 + d] = y[d];
        v[row2pos[r0 + d]] = -((((vf_s[r0 + d] + (d == 0 ? s0 : 0.0)) - eta * x[d]) - rho * y[d]) - zz[d]);
      }
  }
  __syncwarp();
  double prev = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  int m = 0;  // Nesterov updates since the last restart (a = a_m)
  double rp = 0.0, dmax = 0.0, rc = 0.0;
  double r_p = 0, r_d = 0, r_c = 0;
  int restarts = 0, it = 1;
  bool converged = false;
  const int hcap = bv.hist_cap;
  for (it = 1; it <= sp.max_iters; ++it) {
    // x = D^-1 rhs: forward then backward substitution, two phases per level
    for (int l = 0; l < P.n_sph; ++l) {
      const uint4 ph = reinterpret_cast<const uint4*>(prog)[l];  // rec0, steps, mode, split
      const bool modeA = ph.z == 0;
      const double* src = modeA ? v : t;
      for (uint32_t st = 0; st < ph.y; ++st) {
        const int slot = 32 * st + lane;
        const uint2 rc = reinterpret_cast<const uint2*>(prog + ph.x)[slot];
        if (!(rc.y >> 31)) continue;
        const int dst = rc.x & 0xffff, nt = rc.x >> 16;
        const uint32_t* tm = prog + (rc.y & 0xffffff);
        // all index words, then all operand loads, then a fixed-order tree:
        // two shared-memory round trips per chunk instead of one per term
        uint32_t tw[kSnChunk];
#pragma unroll
        for (int k = 0; k < kSnChunk; ++k) tw[k] = k < nt ? tm[k] : 0u;
        double pr[kSnChunk];
#pragma unroll
        for (int k = 0; k < kSnChunk; ++k) pr[k] = k < nt ? Lv[tw[k] & 0xffff] * src[tw[k] >> 16] : 0.0;
        const double a0 = ((pr[0] + pr[1]) + (pr[2] + pr[3]));
        const double a1 = ((pr[4] + pr[5]) + (pr[6] + pr[7]));
        const double sum = a0 + a1;
        if (((rc.y >> 30) & 1) && ((rc.y >> 24) & 63) == 0) {
          if (modeA) t[dst] = v[dst] - sum;
          else v[dst] = sum;
        } else {
          part[slot] = sum;
        }
      }
      if (ph.w) {  // owners add their rows' other chunks in slot order
        __syncwarp();
        for (uint32_t st = 0; st < ph.y; ++st) {
          const int slot = 32 * st + lane;
          const uint2 rc = reinterpret_cast<const uint2*>(prog + ph.x)[slot];
          const int npart = (rc.y >> 24) & 63;
          if (!(rc.y >> 31) || !((rc.y >> 30) & 1) || npart == 0) continue;
          double sum = part[slot];
          for (int q = 1; q <= npart; ++q) sum += part[slot + q];
          const int dst = rc.x & 0xffff;
          if (modeA) t[dst] = v[dst] - sum;
          else v[dst] = sum;
        }
      }
      __syncwarp();
    }
    // projection, dual update, residual partials; candidate extrapolation
    const double beta = sp.acceleration ? sp.nest_beta[m] : 0.0;  // (a_m - 1) / a_{m+1}, host table
    rp = dmax = rc = 0.0;
    for (int u = lane; u < n_units; u += 32) {
      const bool con = u >= first_contact;
      const int r0 = con ? first_contact + 3 * (u - first_contact) : u;
      const int nr = con ? 3 : 1;
      double x[3] = {0, 0, 0}, wv[3] = {0, 0, 0}, yn[3] = {0, 0, 0};
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (d < nr) {
          x[d] = v[row2pos[r0 + d]];
          wv[d] = x[d] - zh_s[r0 + d] * inv_rho;
        }
      if (con) project_soc(wv, rmu[r0], 1.0 / (1.0 + rmu[r0] * rmu[r0]), yn);
      else yn[0] = u >= n_jd ? fmax(0.0, wv[0]) : wv[0];
      double ymax = 0.0, zmax = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (d < nr) {
          const double zn = zh_s[r0 + d] - rho * (x[d] - yn[d]);
          const double yo = y_s[r0 + d], zo = z_s[r0 + d];
          rp = fmax(rp, fabs(x[d] - yn[d]));
          dmax = fmax(dmax, fabs(yn[d] - yo));
          ymax = fmax(ymax, fabs(yn[d]));
          zmax = fmax(zmax, fabs(zn));
          y_s[r0 + d] = yn[d];
          z_s[r0 + d] = zn;
          yh_s[r0 + d] = sp.acceleration ? yn[d] + beta * (yn[d] - yo) : yn[d];
          zh_s[r0 + d] = sp.acceleration ? zn + beta * (zn - zo) : zn;
        }
      if (u >= n_jd) rc = fmax(rc, fmin(ymax, zmax));
    }
    // max(r_p, r_d, r_c) in one reduction (rho > 0: max(rho dmax_i) = rho max(dmax_i))
    const double combined = warp_max_nonneg(fmax(rp, fmax(rho * dmax, rc)));
    if (lane == 0 && it <= hcap) bv.hist[(int64_t)w * hcap + it - 1] = combined;
    if (!sp.fixed_mode && combined < sp.eps) {
      converged = true;
      break;
    }
    // nesterov_update (padmm.cpp:58-71)
    const bool restart = sp.acceleration && sp.restart && combined > prev;
    if (restart) {
      m = 0;
      ++restarts;
    } else if (sp.acceleration) {
      ++m;
    }
    for (int u = lane; u < n_units; u += 32) {
      const bool con = u >= first_contact;
      const int r0 = con ? first_contact + 3 * (u - first_contact) : u;
      const int nr = con ? 3 : 1;
      double zz[3] = {0, 0, 0};
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (d < nr) {
          if (restart) {
            yh_s[r0 + d] = y_s[r0 + d];
            zh_s[r0 + d] = z_s[r0 + d];
          }
          zz[d] = zh_s[r0 + d];
        }
      const double s0 = con ? rmu[r0] * fast_sqrt(zz[1] * zz[1] + zz[2] * zz[2]) : 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (d < nr) {
          const int pos = row2pos[r0 + d];
          v[pos] = -((((vf_s[r0 + d] + (d == 0 ? s0 : 0.0)) - eta * v[pos]) - rho * yh_s[r0 + d]) - zz[d]);
        }
    }
    prev = combined;
    __syncwarp();
  }
  stamp(4);
  // the last iteration's r_p, r_d, r_c (padmm.cpp:147-157)
  r_p = warp_max(rp);
  r_d = rho * warp_max(dmax);
  r_c = warp_max(rc);
  // outputs
  for (int r = lane; r < n; r += 32) {
    bv.lam[R0 + r] = y_s[r];
    bv.zo[R0 + r] = z_s[r];
  }
  if (lane == 0) {
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

cudaError_t launch_sparse(const BatchView& bv, const StepParams& sp, const int32_t* worlds, int count, int per_warp,
                          int wpc, int prog_words, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const size_t smem = ((size_t)prog_words + 3) / 4 * 16 + (size_t)per_warp * wpc * sizeof(double);
  static SmemAttrCache attr;
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(sparse_kernel), smem, attr);
    if (e != cudaSuccess) return e;
  }
  sparse_kernel<<<(count + wpc - 1) / wpc, 32 * wpc, smem, s>>>(bv, sp, worlds, count, per_warp, prog_words);
  return cudaGetLastError();
}

}  // namespace kd
