// kd_joint.cuh — per-joint geometry shared by K1 (assembly) and the FK kernel:
// joint_world_frames / joint_coordinate (model.cpp:309-340), build_joint_rows
// (constraints.cpp:20-109) and coordinate_rate_row (constraints.cpp:160-187),
// over BodyS poses (ep, eq, eR).
#pragma once

#include "kd_device.cuh"

namespace kd {

struct Frames {
  V3 ap, ac;  // anchors
  M3 Rp, Rc;  // joint frames in world
};

// joint_world_frames (model.cpp:309-324)
__device__ __forceinline__ Frames joint_frames(const DevJoint& j, const BodyS* bs) {
  Frames f;
  if (j.parent < 0) {
    f.ap = ld3(j.fp_pos);
    f.Rp = ldm(j.fp_R);
  } else {
    const BodyS& p = bs[j.parent];
    f.ap = add(ld3(p.ep), qapply(ldq(p.eq), ld3(j.fp_pos)));
    f.Rp = mmul(ldm(p.eR), ldm(j.fp_R));
  }
  const BodyS& c = bs[j.child];
  f.ac = add(ld3(c.ep), qapply(ldq(c.eq), ld3(j.fc_pos)));
  f.Rc = mmul(ldm(c.eR), ldm(j.fc_R));
  return f;
}

// joint_coordinate (model.cpp:326-340)
__device__ __forceinline__ double joint_coord(const DevJoint& j, const Frames& f) {
  if (j.type == J_REVOLUTE) {
    Q4 rel = qfrom(mmul(mtrans(f.Rp), f.Rc));
    if (rel.w < 0) rel = Q4{-rel.w, -rel.x, -rel.y, -rel.z};
    return 2.0 * atan2(dot(ld3(j.axis), V3{rel.x, rel.y, rel.z}), rel.w);
  }
  return dot(ld3(j.axis), mvec(mtrans(f.Rp), sub(f.ac, f.ap)));
}

__device__ __forceinline__ void put_row(RowJ* rj, int32_t* rb, int r, int ba, int bb, V3 al, V3 aa, V3 bl, V3 ba3) {
  // six 16-byte stores (RowJ rows are 16-byte aligned: 192-byte rows in a cudaMalloc'd array)
  double2* J = reinterpret_cast<double2*>(rj[r].J);
  J[0] = make_double2(al.x, al.y);
  J[1] = make_double2(al.z, aa.x);
  J[2] = make_double2(aa.y, aa.z);
  J[3] = make_double2(bl.x, bl.y);
  J[4] = make_double2(bl.z, ba3.x);
  J[5] = make_double2(ba3.y, ba3.z);
  rb[2 * r] = ba;
  rb[2 * r + 1] = bb;
}

// JacobianRow::dot (constraints.hpp:25-30)
__device__ __forceinline__ double row_dot(const double* J, int ba, int bb, const double* u) {
  double s = 0.0;
  if (ba >= 0) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) t += J[k] * u[6 * ba + k];
    s += t;
  }
  if (bb >= 0) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) t += J[6 + k] * u[6 * bb + k];
    s += t;
  }
  return s;
}

// coordinate_rate_row (constraints.cpp:160-187): returns blocks via out params.
__device__ __forceinline__ void rate_row(const DevJoint& j, const Frames& f, const BodyS* bs, V3& al, V3& aa, V3& bl,
                                         V3& bang) {
  const V3 axis_w = mvec(f.Rp, ld3(j.axis));
  const V3 z{0, 0, 0};
  if (j.type == J_REVOLUTE) {
    al = z;
    aa = axis_w;
    bl = z;
    bang = (j.parent >= 0) ? neg(axis_w) : z;
  } else {
    const V3 lever = sub(f.ac, ld3(bs[j.child].ep));
    al = axis_w;
    aa = vmat(neg(axis_w), skew(lever));
    if (j.parent >= 0) {
      bl = neg(axis_w);
      bang = vmat(axis_w, skew(sub(f.ac, ld3(bs[j.parent].ep))));
    } else {
      bl = z;
      bang = z;
    }
  }
}


// build_joint_rows (constraints.cpp:20-109): calls emit(al, aa, bl, bang, f)
// once per bilateral row in the reference row order (child block a, parent
// block b; the caller zeroes b for a world parent).  Used by the FK kernel;
// K1 (kd_assemble.cu) keeps the same sequence inlined in its joint loop,
// where the functor form measured 0.75 vs 0.49 ms per 4096-world step.
template <class Emit>
__device__ __forceinline__ void joint_bilateral_rows(const DevJoint& j, const Frames& fr, const BodyS* bs, Emit emit) {
  const V3 z3{0, 0, 0};
  const M3 wpt = mtrans(fr.Rp);
  const V3 lever_c = sub(fr.ac, ld3(bs[j.child].ep));
  const V3 f_pos = mvec(wpt, sub(fr.ac, fr.ap));
  const M3 c_ang = mmul(mscl(-1.0, wpt), skew(lever_c));
  M3 p_lin = mzero(), p_ang = mzero();
  if (j.parent >= 0) {
    p_lin = mscl(-1.0, wpt);
    p_ang = mmul(wpt, skew(sub(fr.ac, ld3(bs[j.parent].ep))));
  }
  V3 f_rot{0, 0, 0};
  M3 r_ang = mzero();
  if (j.type != J_SPHERICAL) {
    const M3 rel = mmul(wpt, fr.Rc);
    f_rot = so3_log(rel);
    r_ang = mmul(left_jacobian_inverse(f_rot), wpt);
  }
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
}

}  // namespace kd
