// kd_assemble.cu — K1: per-world constraint assembly, one warp per world.
//
// Restates, on the device and in the reference order:
//   step() prologue (stepper.cpp:139-176): Moreau-Jean eval poses, world
//     inertias (delassus.cpp:21-34), free forces at start-of-step poses
//     (stepper.cpp:108-121), u_free;
//   collide (contacts.cpp:119-145) with sphere-plane / sphere-sphere /
//     box-plane narrow phases;
//   assemble_constraints (constraints.cpp:189-329) incl. build_joint_rows
//     (20-109), coordinate_rate_row (160-187), limit and contact rows;
//   jacobi_preconditioner (delassus.cpp:36-57), v_f = J u_free - v* and its
//     preconditioned form, fold_inverse_mass (JM rows);
//   gather_warmstart (stepper.cpp:19-46) with match_warmstart
//     (contacts.cpp:147-182).
// Lanes own bodies / pairs / joints / rows; ordered outputs (contacts, limit
// rows, per-body row lists) use warp prefix sums so indexing is bit-exact with
// the reference.  Work per world is small (~10^4 flops), so 8 worlds share a
// 256-thread CTA and the grid covers the batch once.
#include "kd_device.cuh"
#include "kd_joint.cuh"

namespace kd {

namespace {

// One contact of the narrow phase.
struct CP {
  V3 pos, nrm;
  double depth;
};

// box_box: EXTENSION (KD_EXT_BOX_BOX), not in the reference, which rejects
// box-box pairs (model.cpp:56-62); parity is against the oracle's restatement
// of the same algorithm (oracle.cpp box_box): SAT over 15 axes, then either one
// edge-edge contact or the incident face clipped against the reference face's
// side planes (up to 8 points, at most 4 kept, in clip order).  Normal from
// b to a, contact at the midpoint between the incident point and the reference
// face; more than 4 clipped points -> the deepest plus three farthest-point
// picks.  Same operation order as the oracle.
__device__ __noinline__ int box_box_dev(V3 ca, const M3& Ra, const double* ha, V3 cb, const M3& Rb, const double* hb,
                                        double margin, CP* cps) {
  const V3 d = sub(ca, cb);
  auto radius = [](const M3& R, const double* h, V3 L) {
    return (h[0] * fabs(dot(mcol(R, 0), L)) + h[1] * fabs(dot(mcol(R, 1), L))) + h[2] * fabs(dot(mcol(R, 2), L));
  };
  double best_face = 1e300, best_edge = 1e300;
  int face = -1, ei = -1, ej = -1;
  for (int f = 0; f < 6; ++f) {
    const V3 L = f < 3 ? mcol(Ra, f) : mcol(Rb, f - 3);
    const double ov = (radius(Ra, ha, L) + radius(Rb, hb, L)) - fabs(dot(d, L));
    if (ov <= -margin) return 0;
    if (ov < best_face) {
      best_face = ov;
      face = f;
    }
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      V3 L = cross(mcol(Ra, i), mcol(Rb, j));
      const double l = norm(L);
      if (l < 1e-6) continue;
      L = V3{L.x / l, L.y / l, L.z / l};
      const double ov = (radius(Ra, ha, L) + radius(Rb, hb, L)) - fabs(dot(d, L));
      if (ov <= -margin) return 0;
      if (ov < best_edge) {
        best_edge = ov;
        ei = i;
        ej = j;
      }
    }
  if (ei >= 0 && best_edge < best_face - 1e-5 - 0.05 * fabs(best_face)) {
    V3 n = cross(mcol(Ra, ei), mcol(Rb, ej));
    const double ln = norm(n);
    n = V3{n.x / ln, n.y / ln, n.z / ln};
    if (dot(d, n) < 0) n = neg(n);
    V3 pa = ca, pb = cb;
    for (int k = 0; k < 3; ++k) {
      if (k != ei) pa = add(pa, scl(dot(mcol(Ra, k), n) > 0 ? -ha[k] : ha[k], mcol(Ra, k)));
      if (k != ej) pb = add(pb, scl(dot(mcol(Rb, k), n) > 0 ? hb[k] : -hb[k], mcol(Rb, k)));
    }
    const V3 da = mcol(Ra, ei), db = mcol(Rb, ej), r = sub(pa, pb);
    const double a12 = dot(da, db), b1 = dot(da, r), b2 = dot(db, r), den = 1.0 - a12 * a12;
    double s = den > 1e-12 ? (a12 * b2 - b1) / den : 0.0;
    s = fmin(fmax(s, -ha[ei]), ha[ei]);
    double t = b2 + s * a12;
    t = fmin(fmax(t, -hb[ej]), hb[ej]);
    cps[0] = CP{scl(0.5, add(add(pa, scl(s, da)), add(pb, scl(t, db)))), n, best_edge};
    return 1;
  }
  const bool refA = face < 3;
  const int fi = refA ? face : face - 3;
  const M3& RR = refA ? Ra : Rb;
  const M3& RI = refA ? Rb : Ra;
  const V3 cR = refA ? ca : cb, cI = refA ? cb : ca;
  const double* hR = refA ? ha : hb;
  const double* hI = refA ? hb : ha;
  const V3 L = mcol(RR, fi);
  const double sdl = dot(d, L);
  const V3 nf = refA ? (sdl > 0 ? neg(L) : L) : (sdl < 0 ? neg(L) : L);
  const V3 n = refA ? neg(nf) : nf;
  int k = 0;
  double best = -1.0;
  for (int q = 0; q < 3; ++q) {
    const double c = fabs(dot(mcol(RI, q), nf));
    if (c > best) {
      best = c;
      k = q;
    }
  }
  const V3 fnI = dot(mcol(RI, k), nf) > 0 ? neg(mcol(RI, k)) : mcol(RI, k);
  const int k1 = k == 0 ? 1 : 0, k2 = k == 2 ? 1 : 2;
  const V3 fc = add(cI, scl(hI[k], fnI)), u1 = scl(hI[k1], mcol(RI, k1)), u2 = scl(hI[k2], mcol(RI, k2));
  V3 poly[8], tmp[8];
  int np = 4;
  poly[0] = sub(sub(fc, u1), u2);
  poly[1] = sub(add(fc, u1), u2);
  poly[2] = add(add(fc, u1), u2);
  poly[3] = add(sub(fc, u1), u2);
  const int i1 = fi == 0 ? 1 : 0, i2 = fi == 2 ? 1 : 2;
  const V3 rc = add(cR, scl(hR[fi], nf));
  for (int pl = 0; pl < 4 && np > 0; ++pl) {
    const V3 sax = mcol(RR, pl < 2 ? i1 : i2);
    const V3 sdir = (pl & 1) ? neg(sax) : sax;
    const double ext = hR[pl < 2 ? i1 : i2];
    int nt = 0;
    V3 prev = poly[np - 1];
    double dp = dot(sub(prev, rc), sdir) - ext;
    for (int q = 0; q < np; ++q) {
      const V3 cur = poly[q];
      const double dc = dot(sub(cur, rc), sdir) - ext;
      if (dc <= 0) {
        if (dp > 0) tmp[nt++] = add(prev, scl(dp / (dp - dc), sub(cur, prev)));
        tmp[nt++] = cur;
      } else if (dp <= 0) {
        tmp[nt++] = add(prev, scl(dp / (dp - dc), sub(cur, prev)));
      }
      prev = cur;
      dp = dc;
    }
    np = nt;
    for (int q = 0; q < np; ++q) poly[q] = tmp[q];
  }
  double dep[8];
  int hits = 0;
  for (int q = 0; q < np; ++q) {
    dep[q] = -dot(sub(poly[q], rc), nf);
    if (dep[q] > -margin) hits |= 1 << q;
    poly[q] = add(poly[q], scl(0.5 * dep[q], nf));  // the contact position
  }
  if (__popc(hits) > 4) {  // the deepest, then farthest-point picks, clip order (as the oracle)
    int first = -1;
    for (int q = 0; q < np; ++q)
      if ((hits >> q & 1) && (first < 0 || dep[q] > dep[first])) first = q;
    int pick = 1 << first;
    // md[q]: squared distance from q to the nearest picked point, updated per
    // pick (the same minimum the oracle recomputes over the picked set)
    double md[8];
    for (int q = 0; q < np; ++q) {
      const V3 dv = sub(poly[q], poly[first]);
      md[q] = dot(dv, dv);
    }
    for (int r = 1; r < 4; ++r) {
      int bq = -1;
      double bd = -1.0;
      for (int q = 0; q < np; ++q)
        if ((hits >> q & 1) && md[q] > bd) {
          bd = md[q];
          bq = q;
        }
      pick |= 1 << bq;
      for (int q = 0; q < np; ++q) {
        const V3 dv = sub(poly[q], poly[bq]);
        md[q] = fmin(md[q], dot(dv, dv));
      }
    }
    hits = pick;
  }
  int cnt = 0;
  for (int q = 0; q < np; ++q)
    if (hits >> q & 1) cps[cnt++] = CP{poly[q], n, dep[q]};
  return cnt;
}


}  // namespace

__global__ void __launch_bounds__(256) assemble_kernel(BatchView bv, StepParams sp, int w0, int w1) {
  const int lane = threadIdx.x & 31;
  const int w = w0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= w1) return;
  WorldStep& ws = bv.wstep[w];
  if (!bv.active[w]) {
    if (lane == 0) ws.backend = BE_NONE, ws.n_rows = -1;
    return;
  }
  const DevWorld W = bv.worlds[w];
  const DevModel M = bv.models[W.model];
  const DevBody* mb = bv.bodies + M.body_off;
  const DevJoint* mj = bv.joints + M.joint_off;
  const DevGeom* mg = bv.geoms + M.geom_off;
  const DevPair* mp = bv.pairs + M.pair_off;
  const double* pose = bv.poses + W.pose_off;
  const double* tw = bv.twists + W.twist_off;
  BodyS* bs = bv.bs + W.body_off;
  const int64_t R0 = W.row_off;
  RowJ* rj = bv.rowj + R0;
  int32_t* rb = bv.rbody + 2 * R0;
  int32_t* rk = bv.rkind + R0;
  int32_t* lk = bv.lkey + 2 * R0;
  double* rmu = bv.rmu + R0;
  double* bias = bv.bias + R0;
  double* reg = bv.reg + R0;
  double* scale = bv.scale + R0;
  double* vf = bv.vf + R0;
  double* x0 = bv.x0 + R0;
  double* z0 = bv.z0 + R0;
  Contact* ct = bv.contacts + W.contact_off;
  const double dt = sp.dt;
  const double bgain = sp.beta / dt;

  // ---- 1. bodies: eval pose, inertias, free forces, u_free (stepper.cpp:139-164)
  for (int b = lane; b < M.nb; b += 32) {
    const double* p = pose + 7 * b;
    const double* t = tw + 6 * b;
    const V3 x{p[0], p[1], p[2]};
    const Q4 q{p[3], p[4], p[5], p[6]};
    const V3 vl{t[0], t[1], t[2]}, va{t[3], t[4], t[5]};
    V3 ex = x;
    Q4 eq = q;
    if (sp.moreau) {
      ex = add(x, scl(0.5 * dt, vl));
      const V3 wb = mtvec(qrot(q), va);
      eq = quat_integrate(q, wb, 0.5 * dt);
    }
    const M3 eR = qrot(eq);
    const DevBody db = mb[b];
    const M3 ib = ldm(db.ib);
    const M3 Iw = world_inertia(ib, eq);
    const M3 inv = llt_inverse3(Iw);
    const M3 Iwinv = mscl(0.5, madd(inv, mtrans(inv)));
    const M3 Iw0 = world_inertia(ib, q);  // free_forces uses the start-of-step pose
    const V3 hf = scl(db.mass, ld3(M.gravity));
    const V3 ht = neg(cross(va, mvec(Iw0, va)));
    const V3 ufl = add(vl, scl(dt * (1.0 / db.mass), hf));
    const V3 ufa = add(va, scl(dt, mvec(Iwinv, ht)));
    BodyS& o = bs[b];
    st3(o.ep, ex);
    o.eq[0] = eq.w; o.eq[1] = eq.x; o.eq[2] = eq.y; o.eq[3] = eq.z;
    stm(o.eR, eR);
    o.uf[0] = ufl.x; o.uf[1] = ufl.y; o.uf[2] = ufl.z; o.uf[3] = ufa.x; o.uf[4] = ufa.y; o.uf[5] = ufa.z;
    o.h[0] = hf.x; o.h[1] = hf.y; o.h[2] = hf.z; o.h[3] = ht.x; o.h[4] = ht.y; o.h[5] = ht.z;
    stm(o.Iw, Iw);
    stm(o.Iwinv, Iwinv);
    o.mass = db.mass;
    o.inv_mass = 1.0 / db.mass;
  }
  __syncwarp();

  // ---- 2. narrow phase (contacts.cpp:119-145), pair order then corner index
  int nc = 0;
  for (int base = 0; base < M.npairs; base += 32) {
    const int pi = base + lane;
    CP cps[4];
    int cnt = 0;
    DevPair pr{0, 0, 0, 0};
    if (pi < M.npairs) {
      pr = mp[pi];
      const DevGeom ga = mg[pr.a], gb = mg[pr.b];
      if (pr.kind == P_SPHERE_PLANE) {  // sphere_plane (contacts.cpp:26-43)
        const V3 c = ld3(bs[ga.body].ep);
        const V3 n = ld3(gb.normal);
        const double depth = ga.radius - (dot(n, c) - gb.offset);
        if (!(depth <= -sp.contact_margin)) {
          cps[0] = CP{sub(c, scl(ga.radius, n)), n, depth};
          cnt = 1;
        }
      } else if (pr.kind == P_SPHERE_SPHERE) {  // sphere_sphere (contacts.cpp:45-64)
        const V3 ca = ld3(bs[ga.body].ep), cb = ld3(bs[gb.body].ep);
        const V3 d = sub(ca, cb);
        const double dist = norm(d);
        const double depth = ga.radius + gb.radius - dist;
        if (!(depth <= -sp.contact_margin)) {
          const V3 n = dist > 1e-12 ? V3{d.x / dist, d.y / dist, d.z / dist} : V3{0, 0, 1};
          cps[0] = CP{scl(0.5, add(sub(ca, scl(ga.radius, n)), add(cb, scl(gb.radius, n)))), n, depth};
          cnt = 1;
        }
      } else if (pr.kind == P_BOX_BOX) {  // extension (box_box_dev)
        cnt = box_box_dev(ld3(bs[ga.body].ep), ldm(bs[ga.body].eR), ga.he, ld3(bs[gb.body].ep), ldm(bs[gb.body].eR),
                          gb.he, sp.contact_margin, cps);
      } else {  // box_plane (contacts.cpp:66-106)
        const V3 c = ld3(bs[ga.body].ep);
        const M3 R = ldm(bs[ga.body].eR);
        const V3 n = ld3(gb.normal);
        double dep[8];
        V3 pt[8];
        int hits = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const V3 loc{(k & 1) ? ga.he[0] : -ga.he[0], (k & 2) ? ga.he[1] : -ga.he[1], (k & 4) ? ga.he[2] : -ga.he[2]};
          pt[k] = add(c, mvec(R, loc));
          dep[k] = gb.offset - dot(n, pt[k]);
          if (dep[k] > -sp.contact_margin) hits |= 1 << k;
        }
        const int nh = __popc(hits);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (!(hits & (1 << k))) continue;
          if (nh > 4) {  // stable_sort by depth desc, keep 4 (contacts.cpp:88-92)
            int rank = 0;
            for (int j2 = 0; j2 < 8; ++j2)
              if ((hits & (1 << j2)) && (dep[j2] > dep[k] || (dep[j2] == dep[k] && j2 < k))) ++rank;
            if (rank >= 4) continue;
          }
          cps[cnt++] = CP{pt[k], n, dep[k]};
        }
      }
    }
    int excl;
    const int tot = warp_exclusive_sum(cnt, lane, excl);
    if (nc + excl + cnt > W.contact_cap) cnt = max(0, W.contact_cap - nc - excl);  // overflow: reported below
    if (cnt) {
      const DevGeom ga = mg[pr.a], gb = mg[pr.b];
      const double mu = sqrt(ga.mu * gb.mu);
      const double e = fmax(ga.restitution, gb.restitution);
      for (int k = 0; k < cnt; ++k) {
        Contact& o = ct[nc + excl + k];
        o.ga = pr.a;
        o.gb = pr.b;
        o.pair = pi;
        st3(o.pos, cps[k].pos);
        st3(o.nrm, cps[k].nrm);
        o.depth = cps[k].depth;
        o.mu = mu;
        o.e = e;
      }
    }
    nc += tot;
  }
  bool overflow = false;
  if (nc > W.contact_cap) {
    overflow = true;
    nc = W.contact_cap;
  }

  // ---- 3. joint rows, joint-dynamics rows, limit activation (constraints.cpp:20-109, 189-295)
  const int n_jd = M.n_bil + M.n_dyn;
  double f_inf = 0.0;
  int nlim = 0;
  for (int base = 0; base < M.nj; base += 32) {
    const int ji = base + lane;
    int lim_cnt = 0;
    int lo_act = 0, up_act = 0;
    double g_lo = 0, g_up = 0;
    Frames fr;
    DevJoint j;
    if (ji < M.nj) {
      j = mj[ji];
      fr = joint_frames(j, bs);
      // build_joint_rows (constraints.cpp:20-109), the sequence of
      // joint_bilateral_rows (kd_joint.cuh) kept inline for K1's register
      // allocation (measured 0.49 vs 0.75 ms per 4096-world step)
      const M3 wpt = mtrans(fr.Rp);
      const int child = j.child;
      const V3 lever_c = sub(fr.ac, ld3(bs[child].ep));
      const V3 f_pos = mvec(wpt, sub(fr.ac, fr.ap));
      const M3 c_ang = mmul(mscl(-1.0, wpt), skew(lever_c));
      M3 p_lin = mzero(), p_ang = mzero();
      if (j.parent >= 0) {
        p_lin = mscl(-1.0, wpt);
        p_ang = mmul(wpt, skew(sub(fr.ac, ld3(bs[j.parent].ep))));
      }
      const int pb = j.parent;
      V3 f_rot{0, 0, 0};
      M3 r_ang = mzero();
      if (j.type != J_SPHERICAL) {
        const M3 rel = mmul(wpt, fr.Rc);
        f_rot = so3_log(rel);
        r_ang = mmul(left_jacobian_inverse(f_rot), wpt);
      }
      const V3 z3{0, 0, 0};
      int r = j.row_offset;
      auto emit = [&](V3 al, V3 aa, V3 bl, V3 bang, double fval) {
        put_row(rj, rb, r, child, pb, al, aa, pb >= 0 ? bl : z3, pb >= 0 ? bang : z3);
        rk[r] = ROW_BILATERAL;
        rmu[r] = 0.0;
        reg[r] = 0.0;
        bias[r] = fmin(fmax(-bgain * fval, -sp.bias_clamp), sp.bias_clamp);  // clamp_abs
        f_inf = fmax(f_inf, fabs(fval));
        ++r;
      };
      auto emit_pos = [&](int k) { emit(mrow(wpt, k), mrow(c_ang, k), mrow(p_lin, k), mrow(p_ang, k), comp(f_pos, k)); };
      auto emit_rot = [&](int k) { emit(z3, mrow(r_ang, k), z3, neg(mrow(r_ang, k)), comp(f_rot, k)); };
      // push_combined (constraints.cpp:77-87): weights^T applied to a 3-row block
      auto emit_comb = [&](bool pos, const double* wv) {
        V3 al{0, 0, 0}, aa{0, 0, 0}, bl{0, 0, 0}, bang{0, 0, 0};
        for (int k = 0; k < 3; ++k) {
          const double wk = wv[k];
          if (pos) {
            al = add(al, scl(wk, mrow(wpt, k)));
            aa = add(aa, scl(wk, mrow(c_ang, k)));
            bl = add(bl, scl(wk, mrow(p_lin, k)));
            bang = add(bang, scl(wk, mrow(p_ang, k)));
          } else {
            aa = add(aa, scl(wk, mrow(r_ang, k)));
            bang = add(bang, scl(wk, neg(mrow(r_ang, k))));
          }
        }
        emit(al, aa, bl, bang, dot(ld3(wv), pos ? f_pos : f_rot));
      };
      switch (j.type) {
        case J_FIXED:
          for (int k = 0; k < 3; ++k) emit_pos(k);
          for (int k = 0; k < 3; ++k) emit_rot(k);
          break;
        case J_REVOLUTE:
          for (int k = 0; k < 3; ++k) emit_pos(k);
          emit_comb(false, j.comp0);
          emit_comb(false, j.comp1);
          break;
        case J_PRISMATIC:
          emit_comb(true, j.comp0);
          emit_comb(true, j.comp1);
          for (int k = 0; k < 3; ++k) emit_rot(k);
          break;
        default:
          for (int k = 0; k < 3; ++k) emit_pos(k);
          break;
      }
      // coordinate (limited or actuated scalar joints), dynamics rows
      const bool scalar = j.type == J_REVOLUTE || j.type == J_PRISMATIC;
      double coord = 0.0;
      if (scalar && (j.flags & (JF_LIMITS | JF_PD))) coord = joint_coord(j, fr);
      if (j.flags & (JF_PD | JF_ARMATURE | JF_DAMPING)) {
        V3 al, aa, bl, bang;
        rate_row(j, fr, bs, al, aa, bl, bang);
        int rr = M.n_bil + j.dyn_offset;
        if (j.flags & JF_PD) {
          put_row(rj, rb, rr, child, pb, al, aa, bl, bang);
          rk[rr] = ROW_BILATERAL;
          rmu[rr] = 0.0;
          reg[rr] = 1.0 / (dt * (dt * j.kp + j.kd));
          bias[rr] = (j.kp * (j.target - coord) + j.kd * j.target_rate) / (dt * j.kp + j.kd);
          ++rr;
        }
        if (j.flags & JF_ARMATURE) {
          put_row(rj, rb, rr, child, pb, al, aa, bl, bang);
          rk[rr] = ROW_BILATERAL;
          rmu[rr] = 0.0;
          reg[rr] = 1.0 / j.armature;
          bias[rr] = row_dot(rj[rr].J, child, pb, tw);
          ++rr;
        }
        if (j.flags & JF_DAMPING) {
          put_row(rj, rb, rr, child, pb, al, aa, bl, bang);
          rk[rr] = ROW_BILATERAL;
          rmu[rr] = 0.0;
          reg[rr] = 1.0 / (dt * j.damping);
          bias[rr] = 0.0;
          ++rr;
        }
      }
      if (j.flags & JF_LIMITS) {  // constraints.cpp:222-229
        const double margin = j.type == J_REVOLUTE ? sp.lim_margin_ang : sp.lim_margin_lin;
        g_lo = coord - j.lower;
        g_up = j.upper - coord;
        lo_act = g_lo < margin;
        up_act = g_up < margin;
        lim_cnt = lo_act + up_act;
      }
    }
    int excl;
    const int tot = warp_exclusive_sum(lim_cnt, lane, excl);
    if (lim_cnt) {  // limit rows (constraints.cpp:281-295), lower before upper
      V3 al, aa, bl, bang;
      rate_row(j, fr, bs, al, aa, bl, bang);
      int r = n_jd + nlim + excl;
      for (int bound = 0; bound < 2; ++bound) {
        if (!(bound == 0 ? lo_act : up_act)) continue;
        const double sgn = bound == 1 ? -1.0 : 1.0;
        put_row(rj, rb, r, j.child, j.parent, scl(sgn, al), scl(sgn, aa), scl(sgn, bl), scl(sgn, bang));
        const double gap = bound == 0 ? g_lo : g_up;
        rk[r] = ROW_LIMIT;
        rmu[r] = 0.0;
        reg[r] = 0.0;
        bias[r] = fmin(-bgain * fmin(gap, 0.0), sp.bias_clamp);
        lk[2 * r] = ji;
        lk[2 * r + 1] = bound;
        ++r;
      }
    }
    nlim += tot;
  }
  f_inf = warp_max(f_inf);
  const int first_contact = n_jd + nlim;
  const int n = first_contact + 3 * nc;
  __syncwarp();

  // ---- 4. contact rows (constraints.cpp:297-326)
  for (int c = lane; c < nc; c += 32) {
    const Contact cp = ct[c];
    const V3 nrm = ld3(cp.nrm);
    V3 t1, t2;
    orthonormal_complement(nrm, t1, t2);  // contact_frame (contacts.cpp:110-117)
    const int ba = mg[cp.ga].body;
    const int bb = mg[cp.gb].body;
    const int r = first_contact + 3 * c;
    const V3 pos = ld3(cp.pos);
    for (int d = 0; d < 3; ++d) {
      const V3 dir = d == 0 ? nrm : (d == 1 ? t1 : t2);
      const V3 aa = vmat(neg(dir), skew(sub(pos, ld3(bs[ba].ep))));
      V3 bl{0, 0, 0}, bang{0, 0, 0};
      if (bb >= 0) {
        bl = neg(dir);
        bang = vmat(dir, skew(sub(pos, ld3(bs[bb].ep))));
      }
      put_row(rj, rb, r + d, ba, bb >= 0 ? bb : -1, dir, aa, bl, bang);
      rk[r + d] = ROW_CONTACT;
      rmu[r + d] = cp.mu;
      reg[r + d] = 0.0;
      bias[r + d] = 0.0;
    }
    const double vn = row_dot(rj[r].J, ba, bb >= 0 ? bb : -1, tw);
    double bn = fmin(-bgain * fmin(-cp.depth, 0.0), sp.bias_clamp);
    if (vn < -sp.impact_thr) bn += -cp.e * vn;
    bias[r] = bn;
  }

  // ---- 5. contact warm start: match_warmstart per geom-pair group (contacts.cpp:147-182)
  const int ncache = ws.ccache_count;
  const CacheEntry* cache = bv.ccache + W.contact_off;
  for (int c = lane; c < nc; c += 32) {
    const int r = first_contact + 3 * c;
    for (int d = 0; d < 3; ++d) x0[r + d] = z0[r + d] = 0.0;
  }
  __syncwarp();
  if (sp.warm_start) {
    for (int c = lane; c < nc; c += 32) {
      const Contact cp = ct[c];
      if (c > 0 && ct[c - 1].ga == cp.ga && ct[c - 1].gb == cp.gb) continue;  // not group head
      int gsize = 1;
      while (c + gsize < nc && ct[c + gsize].ga == cp.ga && ct[c + gsize].gb == cp.gb && gsize < 4) ++gsize;
      // candidates (dist, entry, contact) within tolerance 1e-3
      double cd[16];
      int ce[16], cc[16], ncand = 0;
      // the pair's entries: the cache is sorted by pair index (K3 writes it in
      // contact order), so bisect to the first one (same candidates, same order)
      int e0 = 0, e1 = ncache;
      while (e0 < e1) {
        const int mid = (e0 + e1) >> 1;
        if (cache[mid].pair < cp.pair) e0 = mid + 1;
        else e1 = mid;
      }
      for (int e = e0; e < ncache && cache[e].pair == cp.pair; ++e) {
        for (int k = 0; k < gsize; ++k) {
          const double dd = norm(sub(ld3(cache[e].pos), ld3(ct[c + k].pos)));
          if (dd <= 1e-3 && ncand < 16) {
            cd[ncand] = dd;
            ce[ncand] = e;
            cc[ncand] = k;
            ++ncand;
          }
        }
      }
      // greedy nearest-first over the sorted candidate list
      unsigned used_e = 0, done_c = 0;  // a pair's cache entries are contiguous and <= 4
      for (int round = 0; round < ncand; ++round) {
        int best = -1;
        for (int k = 0; k < ncand; ++k) {
          if (ce[k] < 0) continue;
          if (best < 0 || cd[k] < cd[best] || (cd[k] == cd[best] && (ce[k] < ce[best] || (ce[k] == ce[best] && cc[k] < cc[best]))))
            best = k;
        }
        if (best < 0) break;
        const int e = ce[best], k = cc[best];
        ce[best] = -1;
        if ((used_e >> (e & 31)) & 1u) continue;
        if ((done_c >> k) & 1u) continue;
        used_e |= 1u << (e & 31);
        done_c |= 1u << k;
        const int r = first_contact + 3 * (c + k);
        for (int d = 0; d < 3; ++d) {
          x0[r + d] = cache[e].imp[d];
          z0[r + d] = cache[e].dual[d];
        }
      }
    }
  }
  __syncwarp();

  // ---- 6. rows: JM, preconditioner, v_f, remaining warm start (delassus.cpp:12-57; stepper.cpp:19-46, 175-176)
  const bool jvalid = sp.warm_start && ws.jcache_valid;
  for (int r = lane; r < n; r += 32) {
    // J in registers (16-byte loads), JM formed there and written with
    // 16-byte stores: the scalar read-modify-write of the row filled the
    // load/store queue (ncu: lg_throttle 25 % of K1's stalls); same
    // arithmetic in the same order
    double2* R2 = reinterpret_cast<double2*>(&rj[r]);
    double J[12], JMr[12];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const double2 v = R2[k];
      J[2 * k] = v.x;
      J[2 * k + 1] = v.y;
    }
    const int ba = rb[2 * r], bb = rb[2 * r + 1];
    double d = reg[r];
    if (ba >= 0) {
      const BodyS& B = bs[ba];
      const V3 t = vmat(V3{J[3], J[4], J[5]}, ldm(B.Iwinv));
      JMr[0] = J[0] * B.inv_mass; JMr[1] = J[1] * B.inv_mass; JMr[2] = J[2] * B.inv_mass;
      JMr[3] = t.x; JMr[4] = t.y; JMr[5] = t.z;
      double s = 0;
#pragma unroll
      for (int k = 0; k < 6; ++k) s += JMr[k] * J[k];
      d += s;
    } else {
#pragma unroll
      for (int k = 0; k < 6; ++k) JMr[k] = 0.0;
    }
    if (bb >= 0) {
      const BodyS& B = bs[bb];
      const V3 t = vmat(V3{J[9], J[10], J[11]}, ldm(B.Iwinv));
      JMr[6] = J[6] * B.inv_mass; JMr[7] = J[7] * B.inv_mass; JMr[8] = J[8] * B.inv_mass;
      JMr[9] = t.x; JMr[10] = t.y; JMr[11] = t.z;
      double s = 0;
#pragma unroll
      for (int k = 0; k < 6; ++k) s += JMr[6 + k] * J[6 + k];
      d += s;
    } else {
#pragma unroll
      for (int k = 0; k < 6; ++k) JMr[6 + k] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) R2[6 + k] = make_double2(JMr[2 * k], JMr[2 * k + 1]);
    scale[r] = 1.0 / sqrt(fmax(d, 1e-12));
  }
  __syncwarp();
  for (int r = lane; r < n; r += 32) {
    double p = scale[r];
    if (r >= first_contact) {  // SOC rows share the normal-row scale (delassus.cpp:50-55)
      p = scale[first_contact + 3 * ((r - first_contact) / 3)];
    }
    // v_f = J u_free - v*; scaled by P
    // (16-byte loads: BodyS::uf and the RowJ halves are 16-byte aligned)
    const int ba = rb[2 * r], bb = rb[2 * r + 1];
    const double2* J2 = reinterpret_cast<const double2*>(rj[r].J);
    double s = 0.0;
    if (ba >= 0) {
      const double2* u2 = reinterpret_cast<const double2*>(bs[ba].uf);
      double t = 0;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double2 j = J2[k], u = u2[k];
        t += j.x * u.x;
        t += j.y * u.y;
      }
      s += t;
    }
    if (bb >= 0) {
      const double2* u2 = reinterpret_cast<const double2*>(bs[bb].uf);
      double t = 0;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double2 j = J2[3 + k], u = u2[k];
        t += j.x * u.x;
        t += j.y * u.y;
      }
      s += t;
    }
    vf[r] = p * (s - bias[r]);
    // warm start of joint and limit rows (contacts were filled above)
    double xl = 0.0, xz = 0.0;
    if (r < n_jd) {
      if (jvalid) {
        xl = bv.jc_lam[W.jcache_off + r];
        xz = bv.jc_z[W.jcache_off + r];
      }
    } else if (r < first_contact) {
      if (sp.warm_start) {
        const int ji = lk[2 * r], bound = lk[2 * r + 1];
        const int slot = W.lslot_off + 2 * mj[ji].limit_slot + bound;
        if (bv.ls_valid[slot]) {
          xl = bv.ls_lam[slot];
          xz = bv.ls_z[slot];
        }
      }
    } else {
      xl = x0[r];
      xz = z0[r];
    }
    x0[r] = xl / p;
    z0[r] = xz * p;
    if (r >= first_contact) scale[r] = p;
  }
  __syncwarp();

  // ---- 7. per-body row lists in ascending row order (for J^T lambda and the CR scatter)
  int32_t* cptr = bv.csr_ptr + W.body_off + w;
  int32_t* clist = bv.csr + 2 * R0;
  const int run = warp_incidence_lists(rb, n, M.nb, cptr, clist, lane);
  bool sn_ok = sp.sparse && M.sn;
  if (sn_ok) {
    const int32_t* pslot = bv.sn_pair_slot + bv.snplan[W.model].pair_off;
    bool planned = true;
    for (int c = lane; c < nc; c += 32) planned = planned && pslot[ct[c].pair] >= 0;
    sn_ok = __all_sync(0xffffffffu, planned);
  }
  if (lane == 0) {
    cptr[M.nb] = run;
    ws.n_rows = n;
    ws.n_limits = nlim;
    ws.n_contacts = nc;
    ws.f_inf = M.n_bil > 0 ? f_inf : 0.0;
    int be = BE_NONE;
    ws.fail = 0;
    if (n > 0) {  // build_backend choice (delassus.cpp:204-206)
      const bool dense = sp.backend == 0 /*KD_BACKEND_DENSE*/ || (sp.backend == 2 /*AUTO*/ && n <= 300);
      be = dense ? (n <= W.smem_cap ? BE_DENSE_SMEM : BE_DENSE_GLOBAL) : BE_MATRIX_FREE;
      // the dense LLT is factored by the supernodal kernel when the model has a
      // plan and every active contact lies in a planned slot (kd_snplan.h);
      // for larger plans the factor is handed to the dense kernel (BE_DENSE_SN)
      if (dense && sn_ok && !overflow) be = M.sn == 2 ? BE_DENSE_SN : BE_SPARSE;
      if (be == BE_DENSE_GLOBAL && n > W.slab_cap) overflow = true;
    }
    if (overflow) {
      be = BE_NONE;
      ws.fail = 2;
      atomicAdd(bv.error_count + 1, 1);
    }
    ws.backend = be;
    // solver diagnostics default (SolveDiagnostics{}, padmm.hpp:19-28) for n == 0
    ws.iterations = 0;
    ws.restarts = 0;
    ws.converged = 1;
    ws.cr_breakdown = 0;
    ws.cr_iterations = 0;
    ws.r_p = ws.r_d = ws.r_c = 0.0;
  }
}

void launch_assemble(const BatchView& bv, const StepParams& sp, cudaStream_t s, int w0, int w1) {
  const int wpb = 8;
  if (w1 < 0) w1 = bv.n_worlds;
  const int grid = (w1 - w0 + wpb - 1) / wpb;
  if (grid > 0) assemble_kernel<<<grid, 32 * wpb, 0, s>>>(bv, sp, w0, w1);
}

}  // namespace kd
