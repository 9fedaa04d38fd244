// kd_model.cpp — host-side model build (the drop-in for build_model,
// model.hpp:117 / model.cpp:100-307) producing the device model format.
//
// Validation order and messages follow the reference so callers see the same
// ModelError codes and text; the output is the immutable DevModel + arrays of
// DevBody / DevJoint / DevGeom / DevPair (kd_layout.h) that every world of the
// model shares on the device.
#include "kd_host.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>

namespace kd {

namespace {

struct BuildError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw BuildError{code, msg}; }

std::string s(const char* p) { return p ? std::string(p) : std::string(); }

double frob(const double* a) {
  double t = 0;
  for (int i = 0; i < 9; ++i) t += a[i] * a[i];
  return std::sqrt(t);
}

// symmetric 3x3 eigenvalues (ascending) by cyclic Jacobi rotations
void sym_eig3(const double* in, double ev[3]) {
  M3 a{{in[0], in[1], in[2], in[3], in[4], in[5], in[6], in[7], in[8]}};
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = a.m[1] * a.m[1] + a.m[2] * a.m[2] + a.m[5] * a.m[5];
    if (off < 1e-300) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        const double apq = a.m[3 * p + q];
        if (apq == 0.0) continue;
        const double th = (a.m[4 * q] - a.m[4 * p]) / (2.0 * apq);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
        M3 j = mident();
        j.m[4 * p] = c;
        j.m[4 * q] = c;
        j.m[3 * p + q] = sn;
        j.m[3 * q + p] = -sn;
        a = mmul(mmul(mtrans(j), a), j);
      }
  }
  ev[0] = a.m[0];
  ev[1] = a.m[4];
  ev[2] = a.m[8];
  std::sort(ev, ev + 3);
}

}  // namespace

// joint_world_frames + joint_coordinate on the host (model.cpp:309-340)
double host_joint_coordinate(const HostModel& m, int joint, const double* poses7) {
  const DevJoint& j = m.joints[joint];
  auto pose = [&](int b, V3& x, Q4& q) {
    const double* p = poses7 + 7 * b;
    x = V3{p[0], p[1], p[2]};
    q = Q4{p[3], p[4], p[5], p[6]};
  };
  V3 ap, ac;
  M3 Rp, Rc;
  const M3 fpR{{j.fp_R[0], j.fp_R[1], j.fp_R[2], j.fp_R[3], j.fp_R[4], j.fp_R[5], j.fp_R[6], j.fp_R[7], j.fp_R[8]}};
  const M3 fcR{{j.fc_R[0], j.fc_R[1], j.fc_R[2], j.fc_R[3], j.fc_R[4], j.fc_R[5], j.fc_R[6], j.fc_R[7], j.fc_R[8]}};
  if (j.parent < 0) {
    ap = V3{j.fp_pos[0], j.fp_pos[1], j.fp_pos[2]};
    Rp = fpR;
  } else {
    V3 x;
    Q4 q;
    pose(j.parent, x, q);
    ap = add(x, qapply(q, V3{j.fp_pos[0], j.fp_pos[1], j.fp_pos[2]}));
    Rp = mmul(qrot(q), fpR);
  }
  V3 x;
  Q4 q;
  pose(j.child, x, q);
  ac = add(x, qapply(q, V3{j.fc_pos[0], j.fc_pos[1], j.fc_pos[2]}));
  Rc = mmul(qrot(q), fcR);
  const V3 axis{j.axis[0], j.axis[1], j.axis[2]};
  if (j.type == J_REVOLUTE) {
    Q4 rel = qfrom(mmul(mtrans(Rp), Rc));
    if (rel.w < 0) rel = Q4{-rel.w, -rel.x, -rel.y, -rel.z};
    return 2.0 * std::atan2(dot(axis, V3{rel.x, rel.y, rel.z}), rel.w);
  }
  return dot(axis, mvec(mtrans(Rp), sub(ac, ap)));
}

int build_host_model(const kd_scene_desc* d, HostModel& m, std::string& err, uint32_t extensions) {
  try {
    m.name = s(d->name);
    for (int k = 0; k < 3; ++k) m.gravity[k] = d->gravity[k];
    std::map<std::string, int> body_ids;
    // bodies (model.cpp:105-121)
    for (int i = 0; i < d->n_bodies; ++i) {
      const kd_body_desc& sb = d->bodies[i];
      const std::string name = s(sb.name);
      if (name == "world" || body_ids.count(name))
        fail(KD_ERR_MODEL_DUPLICATE_NAME, "body name '" + name + "' is reserved or duplicated");
      body_ids[name] = (int)m.bodies.size();
      DevBody b{};
      b.mass = sb.mass;
      b.inv_mass = 1.0 / sb.mass;
      for (int k = 0; k < 9; ++k) b.ib[k] = sb.inertia[k];
      Q4 q{sb.orientation[0], sb.orientation[1], sb.orientation[2], sb.orientation[3]};
      q = qnormalized(q);
      m.init_pose.insert(m.init_pose.end(), {sb.position[0], sb.position[1], sb.position[2], q.w, q.x, q.y, q.z});
      m.init_twist.insert(m.init_twist.end(), {sb.linear_velocity[0], sb.linear_velocity[1], sb.linear_velocity[2],
                                               sb.angular_velocity[0], sb.angular_velocity[1],
                                               sb.angular_velocity[2]});
      // validate_inertia (model.cpp:21-42)
      if (!(b.mass > 0)) fail(KD_ERR_MODEL_BAD_INERTIA, "body '" + name + "': mass must be positive");
      double asym[9];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) asym[3 * r + c] = b.ib[3 * r + c] - b.ib[3 * c + r];
      if (frob(asym) > 1e-9 * std::max(1.0, frob(b.ib)))
        fail(KD_ERR_MODEL_BAD_INERTIA, "body '" + name + "': inertia tensor is not symmetric");
      double ev[3];
      sym_eig3(b.ib, ev);
      if (!(ev[0] > 0))
        fail(KD_ERR_MODEL_BAD_INERTIA, "body '" + name + "': inertia tensor is not positive definite");
      if (ev[2] > ev[0] + ev[1] + 1e-9 * ev[2])
        fail(KD_ERR_MODEL_BAD_INERTIA, "body '" + name + "': principal moments violate the triangle inequality");
      m.bodies.push_back(b);
      m.body_names.push_back(name);
    }
    auto resolve = [&](const std::string& name, const std::string& ctx) -> int {
      if (name == "world") return -1;
      auto it = body_ids.find(name);
      if (it == body_ids.end()) fail(KD_ERR_MODEL_INVALID_REFERENCE, ctx + ": unknown body '" + name + "'");
      return it->second;
    };
    // joints (model.cpp:132-195)
    std::map<std::string, int> joint_names;
    std::vector<bool> has_target;
    std::vector<double> target;
    for (int i = 0; i < d->n_joints; ++i) {
      const kd_joint_desc& sj = d->joints[i];
      const std::string name = s(sj.name), type = s(sj.type);
      if (joint_names.count(name)) fail(KD_ERR_MODEL_DUPLICATE_NAME, "duplicate joint name '" + name + "'");
      joint_names[name] = (int)m.joints.size();
      DevJoint j{};
      if (type == "fixed") j.type = J_FIXED;
      else if (type == "revolute") j.type = J_REVOLUTE;
      else if (type == "prismatic") j.type = J_PRISMATIC;
      else if (type == "spherical") j.type = J_SPHERICAL;
      else fail(KD_ERR_MODEL_INVALID_REFERENCE, "joint '" + name + "': unknown type '" + type + "'");
      j.parent = resolve(s(sj.parent), "joint '" + name + "'");
      j.child = resolve(s(sj.child), "joint '" + name + "'");
      if (j.child < 0)
        fail(KD_ERR_MODEL_INVALID_REFERENCE,
             "joint '" + name + "': child must be a body (use parent=\"world\" to anchor)");
      if (j.parent == j.child)
        fail(KD_ERR_MODEL_INVALID_REFERENCE, "joint '" + name + "': parent and child must differ");
      for (int k = 0; k < 3; ++k) {
        j.fp_pos[k] = sj.parent_position[k];
        j.fc_pos[k] = sj.child_position[k];
      }
      for (int k = 0; k < 4; ++k) {
        j.fp_q[k] = sj.parent_orientation[k];
        j.fc_q[k] = sj.child_orientation[k];
      }
      const M3 fpR = qrot(Q4{j.fp_q[0], j.fp_q[1], j.fp_q[2], j.fp_q[3]});
      const M3 fcR = qrot(Q4{j.fc_q[0], j.fc_q[1], j.fc_q[2], j.fc_q[3]});
      for (int k = 0; k < 9; ++k) {
        j.fp_R[k] = fpR.m[k];
        j.fc_R[k] = fcR.m[k];
      }
      const bool has_axis = j.type == J_REVOLUTE || j.type == J_PRISMATIC;
      V3 axis{0, 0, 1};
      if (has_axis) {
        const V3 a{sj.axis[0], sj.axis[1], sj.axis[2]};
        const double n = norm(a);
        if (std::fabs(n - 1.0) > 1e-6) fail(KD_ERR_MODEL_NON_UNIT_AXIS, "joint '" + name + "': axis must be unit length");
        axis = V3{a.x / n, a.y / n, a.z / n};
      }
      j.axis[0] = axis.x;
      j.axis[1] = axis.y;
      j.axis[2] = axis.z;
      if (sj.has_limits) {
        if (!has_axis)
          fail(KD_ERR_MODEL_UNSUPPORTED_ON_JOINT_TYPE,
               "joint '" + name + "': limits are only supported on revolute/prismatic joints");
        if (!(sj.lower < sj.upper))
          fail(KD_ERR_MODEL_BAD_LIMITS, "joint '" + name + "': lower limit must be below upper limit");
        j.flags |= JF_LIMITS;
        j.lower = sj.lower;
        j.upper = sj.upper;
      }
      if (sj.kp < 0 || sj.kd < 0 || sj.armature < 0 || sj.damping < 0)
        fail(KD_ERR_MODEL_BAD_LIMITS, "joint '" + name + "': gains, armature and damping must be nonnegative");
      if ((sj.kp > 0 || sj.kd > 0 || sj.armature > 0 || sj.damping > 0) && !has_axis)
        fail(KD_ERR_MODEL_UNSUPPORTED_ON_JOINT_TYPE,
             "joint '" + name +
                 "': actuation/armature/damping need a joint coordinate (revolute or prismatic)");
      if (sj.kp > 0 || sj.kd > 0) j.flags |= JF_PD;
      if (sj.armature > 0) j.flags |= JF_ARMATURE;
      if (sj.damping > 0) j.flags |= JF_DAMPING;
      j.kp = sj.kp;
      j.kd = sj.kd;
      j.target_rate = sj.target_rate;
      j.armature = sj.armature;
      j.damping = sj.damping;
      m.joints.push_back(j);
      m.joint_names.push_back(name);
      has_target.push_back(sj.has_target != 0);
      target.push_back(sj.target);
    }
    // geoms (model.cpp:197-234)
    for (int i = 0; i < d->n_geoms; ++i) {
      const kd_geom_desc& sg = d->geoms[i];
      const std::string body = s(sg.body), shape = s(sg.shape);
      DevGeom g{};
      g.body = resolve(body, "geom on '" + body + "'");
      if (shape == "sphere") {
        g.shape = G_SPHERE;
        if (!(sg.radius > 0)) fail(KD_ERR_MODEL_BAD_GEOMETRY, "sphere geom needs a positive radius");
        g.radius = sg.radius;
      } else if (shape == "box") {
        g.shape = G_BOX;
        if (!(std::min(sg.half_extents[0], std::min(sg.half_extents[1], sg.half_extents[2])) > 0))
          fail(KD_ERR_MODEL_BAD_GEOMETRY, "box geom needs positive half extents");
        for (int k = 0; k < 3; ++k) g.he[k] = sg.half_extents[k];
      } else if (shape == "plane") {
        g.shape = G_PLANE;
        const V3 nv{sg.normal[0], sg.normal[1], sg.normal[2]};
        const double n = norm(nv);
        if (n < 1e-12) fail(KD_ERR_MODEL_BAD_GEOMETRY, "plane normal must be nonzero");
        g.normal[0] = nv.x / n;
        g.normal[1] = nv.y / n;
        g.normal[2] = nv.z / n;
        g.offset = sg.offset;
      } else {
        fail(KD_ERR_MODEL_BAD_GEOMETRY, "unknown geom shape '" + shape + "'");
      }
      if (g.shape == G_PLANE && g.body != -1) fail(KD_ERR_MODEL_BAD_GEOMETRY, "planes must be attached to the world");
      if (g.shape != G_PLANE && g.body == -1) fail(KD_ERR_MODEL_BAD_GEOMETRY, "only planes may be attached to the world");
      g.mu = sg.mu;
      g.restitution = sg.restitution;
      if (g.mu < 0) fail(KD_ERR_MODEL_BAD_GEOMETRY, "friction must be nonnegative");
      if (g.restitution < 0 || g.restitution > 1) fail(KD_ERR_MODEL_BAD_GEOMETRY, "restitution must lie in [0, 1]");
      m.geoms.push_back(g);
    }
    // collision pairs in collide() order (model.cpp:238-250, contacts.cpp:122-143)
    static const char* names[3] = {"sphere", "plane", "box"};
    int max_contacts = 0;
    for (int a = 0; a < (int)m.geoms.size(); ++a)
      for (int b = a + 1; b < (int)m.geoms.size(); ++b) {
        const DevGeom& ga = m.geoms[a];
        const DevGeom& gb = m.geoms[b];
        if (ga.body == gb.body) continue;
        if (ga.body == -1 && gb.body == -1) continue;
        DevPair p{};
        if (ga.shape == G_SPHERE && gb.shape == G_SPHERE) p = DevPair{a, b, P_SPHERE_SPHERE, 0};
        else if (ga.shape == G_SPHERE && gb.shape == G_PLANE) p = DevPair{a, b, P_SPHERE_PLANE, 0};
        else if (ga.shape == G_PLANE && gb.shape == G_SPHERE) p = DevPair{b, a, P_SPHERE_PLANE, 0};
        else if (ga.shape == G_BOX && gb.shape == G_PLANE) p = DevPair{a, b, P_BOX_PLANE, 0};
        else if (ga.shape == G_PLANE && gb.shape == G_BOX) p = DevPair{b, a, P_BOX_PLANE, 0};
        else if (ga.shape == G_BOX && gb.shape == G_BOX && (extensions & KD_EXT_BOX_BOX))
          p = DevPair{a, b, P_BOX_BOX, 0};  // extension (kd_assemble.cu box_box)
        else
          fail(KD_ERR_MODEL_UNSUPPORTED_COLLISION_PAIR,
               std::string("unsupported collision pair: ") + names[ga.shape] + "-" + names[gb.shape]);
        max_contacts += (p.kind == P_BOX_PLANE || p.kind == P_BOX_BOX) ? 4 : 1;
        m.pairs.push_back(p);
      }
    // row layout (model.cpp:254-276)
    int row = 0, limited = 0;
    for (DevJoint& j : m.joints) {
      j.row_offset = row;
      j.row_count = j.type == J_FIXED ? 6 : (j.type == J_SPHERICAL ? 3 : 5);
      row += j.row_count;
      if (j.type == J_REVOLUTE || j.type == J_PRISMATIC) {
        V3 b1, b2;
        orthonormal_complement(V3{j.axis[0], j.axis[1], j.axis[2]}, b1, b2);
        j.comp0[0] = b1.x; j.comp0[1] = b1.y; j.comp0[2] = b1.z;
        j.comp1[0] = b2.x; j.comp1[1] = b2.y; j.comp1[2] = b2.z;
      }
      j.limit_slot = (j.flags & JF_LIMITS) ? limited++ : -1;
    }
    m.n_bil = row;
    int dyn = 0;
    for (DevJoint& j : m.joints) {
      j.dyn_offset = dyn;
      dyn += ((j.flags & JF_PD) ? 1 : 0) + ((j.flags & JF_ARMATURE) ? 1 : 0) + ((j.flags & JF_DAMPING) ? 1 : 0);
    }
    m.n_dyn = dyn;
    // loops: E - V + C with the world as a vertex (model.cpp:278-291)
    const int nv = (int)m.bodies.size() + 1;
    std::vector<int> par(nv);
    std::iota(par.begin(), par.end(), 0);
    auto find = [&](int a) {
      while (par[a] != a) a = par[a] = par[par[a]];
      return a;
    };
    for (const DevJoint& j : m.joints) par[find(j.parent < 0 ? nv - 1 : j.parent)] = find(j.child);
    int comps = 0;
    for (int v = 0; v < nv; ++v)
      if (find(v) == v) ++comps;
    m.n_loops = (int)m.joints.size() - nv + comps;
    // default PD targets (model.cpp:293-305)
    for (size_t i = 0; i < m.joints.size(); ++i) {
      if (!(m.joints[i].flags & JF_PD)) continue;
      m.joints[i].target = has_target[i] ? target[i] : host_joint_coordinate(m, (int)i, m.init_pose.data());
    }
    m.info.n_bodies = (int)m.bodies.size();
    m.info.n_joints = (int)m.joints.size();
    m.info.n_geoms = (int)m.geoms.size();
    m.info.n_bilateral_rows = m.n_bil;
    m.info.n_dynamics_rows = m.n_dyn;
    m.info.n_loops = m.n_loops;
    m.info.n_limited_joints = limited;
    m.info.max_contacts = max_contacts;
    m.info.row_capacity = m.n_bil + m.n_dyn + 2 * limited + 3 * max_contacts;
    return KD_OK;
  } catch (const BuildError& e) {
    err = e.msg;
    return e.code;
  }
}

}  // namespace kd
