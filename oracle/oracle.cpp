// oracle.cpp — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
//
// Line-by-line CPU restatement of /root/reference/proj/src/{se3,model,contacts,
// constraints,delassus,padmm,stepper,batch}.cpp in fp64.  Each function cites
// the reference lines it follows.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg may load this code.
#include "oracle.hpp"

#include <algorithm>
#include <atomic>
#include <limits>
#include <numeric>
#include <thread>

namespace oracle {

// ============================================================ Eigen mirrors
// Eigen Quaternion product (Quaternion.h quat_product, generic path).
Quat operator*(const Quat& a, const Quat& b) {
  return Quat(a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z,
              a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
              a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z,
              a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x);
}

// Eigen QuaternionBase::_transformVector: uv = vec x v; uv += uv; v + w uv + vec x uv.
Vec3 operator*(const Quat& q, const Vec3& v) {
  Vec3 uv = cross(q.vec(), v);
  uv = uv + uv;
  return v + q.w * uv + cross(q.vec(), uv);
}

// Eigen QuaternionBase::toRotationMatrix.
Mat3 Quat::to_rotation_matrix() const {
  Mat3 r;
  const double tx = 2 * x, ty = 2 * y, tz = 2 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  r(0, 0) = 1 - (tyy + tzz);
  r(0, 1) = txy - twz;
  r(0, 2) = txz + twy;
  r(1, 0) = txy + twz;
  r(1, 1) = 1 - (txx + tzz);
  r(1, 2) = tyz - twx;
  r(2, 0) = txz - twy;
  r(2, 1) = tyz + twx;
  r(2, 2) = 1 - (txx + tyy);
  return r;
}

// Eigen quaternionbase_assign_impl<Matrix3>::run (Quaternion(Mat3)).
Quat Quat::from_matrix(const Mat3& m) {
  Quat q;
  double t = m(0, 0) + m(1, 1) + m(2, 2);
  if (t > 0) {
    t = std::sqrt(t + 1.0);
    q.w = 0.5 * t;
    t = 0.5 / t;
    q.x = (m(2, 1) - m(1, 2)) * t;
    q.y = (m(0, 2) - m(2, 0)) * t;
    q.z = (m(1, 0) - m(0, 1)) * t;
  } else {
    int i = 0;
    if (m(1, 1) > m(0, 0)) i = 1;
    if (m(2, 2) > m(i, i)) i = 2;
    const int j = (i + 1) % 3;
    const int k = (j + 1) % 3;
    t = std::sqrt(m(i, i) - m(j, j) - m(k, k) + 1.0);
    double c[3];
    c[i] = 0.5 * t;
    t = 0.5 / t;
    q.w = (m(k, j) - m(j, k)) * t;
    c[j] = (m(j, i) + m(i, j)) * t;
    c[k] = (m(k, i) + m(i, k)) * t;
    q.x = c[0];
    q.y = c[1];
    q.z = c[2];
  }
  return q;
}

// ============================================================ se3.cpp
// skew: se3.cpp:7-11
Mat3 skew(const Vec3& v) {
  Mat3 m;
  m(0, 1) = -v.z;
  m(0, 2) = v.y;
  m(1, 0) = v.z;
  m(1, 2) = -v.x;
  m(2, 0) = -v.y;
  m(2, 1) = v.x;
  return m;
}

// quat_exp: se3.cpp:13-25
Quat quat_exp(const Vec3& v) {
  const double angle = norm(v);
  double sinc;
  if (angle < 1e-8) {
    sinc = 1.0 - angle * angle / 6.0;
  } else {
    sinc = std::sin(angle) / angle;
  }
  Quat q;
  q.w = std::cos(angle);
  const Vec3 s = sinc * v;
  q.x = s.x;
  q.y = s.y;
  q.z = s.z;
  return q;
}

// quat_integrate: se3.cpp:27-32
Quat quat_integrate(const Quat& q, const Vec3& w, double dt) {
  const Quat dq = quat_exp((0.5 * dt) * w);
  Quat out = q * dq;
  out.normalize();
  return out;
}

// so3_exp: se3.cpp:34-46 (test-only in the reference; used by the KATs)
Mat3 so3_exp(const Vec3& phi) {
  const double angle = norm(phi);
  const Mat3 k = skew(phi);
  double a, b;
  if (angle < 1e-8) {
    a = 1.0 - angle * angle / 6.0;
    b = 0.5 - angle * angle / 24.0;
  } else {
    a = std::sin(angle) / angle;
    b = (1.0 - std::cos(angle)) / (angle * angle);
  }
  return (Mat3::identity() + a * k) + (b * k) * k;
}

// so3_log(Quat): se3.cpp:48-59
Vec3 so3_log(const Quat& q_in) {
  Quat q = q_in.normalized();
  if (q.w < 0) {
    q.w = -q.w;
    q.x = -q.x;
    q.y = -q.y;
    q.z = -q.z;
  }
  const double vn = norm(q.vec());
  const double angle = 2.0 * std::atan2(vn, q.w);
  if (vn < 1e-12) return 2.0 * q.vec();
  return (angle / vn) * q.vec();
}

// so3_log(Mat3): se3.cpp:61
Vec3 so3_log(const Mat3& r) { return so3_log(Quat::from_matrix(r)); }

// left_jacobian_inverse: se3.cpp:63-74
Mat3 left_jacobian_inverse(const Vec3& phi) {
  const double angle = norm(phi);
  const Mat3 k = skew(phi);
  double c;
  if (angle < 1e-4) {
    c = 1.0 / 12.0 + angle * angle / 720.0;
  } else {
    c = 1.0 / (angle * angle) - (1.0 + std::cos(angle)) / (2.0 * angle * std::sin(angle));
  }
  return (Mat3::identity() - 0.5 * k) + (c * k) * k;
}

// world_inertia: se3.cpp:76-80
Mat3 world_inertia(const InertiaBlock& in, const Quat& q) {
  const Mat3 r = q.to_rotation_matrix();
  const Mat3 iw = (r * in.body_inertia) * r.transpose();
  return 0.5 * (iw + iw.transpose());
}

// Mat3::llt().solve(Identity) (delassus.cpp:30): unblocked lower Cholesky then
// forward/back substitution per column.
Mat3 llt_inverse3(const Mat3& a) {
  double l[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int k = 0; k < 3; ++k) {
    double x = a(k, k);
    for (int j = 0; j < k; ++j) x -= l[k][j] * l[k][j];
    x = std::sqrt(x);
    l[k][k] = x;
    for (int i = k + 1; i < 3; ++i) {
      double s = a(i, k);
      for (int j = 0; j < k; ++j) s -= l[i][j] * l[k][j];
      l[i][k] = s / x;
    }
  }
  Mat3 inv;
  for (int c = 0; c < 3; ++c) {
    double y[3];
    for (int i = 0; i < 3; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int j = 0; j < i; ++j) s -= l[i][j] * y[j];
      y[i] = s / l[i][i];
    }
    for (int i = 2; i >= 0; --i) {
      double s = y[i];
      for (int j = i + 1; j < 3; ++j) s -= l[j][i] * inv(j, c);
      inv(i, c) = s / l[i][i];
    }
  }
  return inv;
}

// orthonormal_complement: se3.cpp:97-110
void orthonormal_complement(const Vec3& axis, Vec3& b1, Vec3& b2) {
  int least = 0;
  for (int k = 1; k < 3; ++k)
    if (std::abs(axis[k]) < std::abs(axis[least])) least = k;
  Vec3 e;
  e[least] = 1.0;
  b1 = normalized(e - dot(e, axis) * axis);
  b2 = cross(axis, b1);
}

// ============================================================ model.cpp
namespace {

JointType parse_joint_type(const std::string& s, const std::string& name) {  // model.cpp:12-19
  if (s == "fixed") return JointType::Fixed;
  if (s == "revolute") return JointType::Revolute;
  if (s == "prismatic") return JointType::Prismatic;
  if (s == "spherical") return JointType::Spherical;
  throw ModelError(InvalidReference, "joint '" + name + "': unknown type '" + s + "'");
}

double frobenius(const Mat3& a) {
  double s = 0;
  for (double v : a.m) s += v * v;
  return std::sqrt(s);
}

// Symmetric 3x3 eigenvalues, ascending (stand-in for SelfAdjointEigenSolver,
// model.cpp:31): cyclic Jacobi to machine precision.
Vec3 sym_eigenvalues(Mat3 a) {
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = a(0, 1) * a(0, 1) + a(0, 2) * a(0, 2) + a(1, 2) * a(1, 2);
    if (off < 1e-300) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a(p, q) == 0.0) continue;
        const double theta = (a(q, q) - a(p, p)) / (2.0 * a(p, q));
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        Mat3 j = Mat3::identity();
        j(p, p) = c;
        j(q, q) = c;
        j(p, q) = s;
        j(q, p) = -s;
        a = (j.transpose() * a) * j;
      }
  }
  double ev[3] = {a(0, 0), a(1, 1), a(2, 2)};
  std::sort(ev, ev + 3);
  return {ev[0], ev[1], ev[2]};
}

void validate_inertia(const BodySpec& b) {  // model.cpp:21-42
  if (!(b.inertia.mass > 0))
    throw ModelError(BadInertia, "body '" + b.name + "': mass must be positive");
  const Mat3& in = b.inertia.body_inertia;
  if (frobenius(in - in.transpose()) > 1e-9 * std::max(1.0, frobenius(in)))
    throw ModelError(BadInertia, "body '" + b.name + "': inertia tensor is not symmetric");
  const Vec3 ev = sym_eigenvalues(in);
  if (!(ev.x > 0))
    throw ModelError(BadInertia, "body '" + b.name + "': inertia tensor is not positive definite");
  if (ev.z > ev.x + ev.y + 1e-9 * ev.z)
    throw ModelError(BadInertia,
                     "body '" + b.name + "': principal moments violate the triangle inequality");
}

struct UnionFind {  // model.cpp:44-52
  std::vector<int> parent;
  explicit UnionFind(int n) : parent(n) { std::iota(parent.begin(), parent.end(), 0); }
  int find(int a) {
    while (parent[a] != a) a = parent[a] = parent[parent[a]];
    return a;
  }
  void unite(int a, int b) { parent[find(a)] = find(b); }
};

bool pair_supported(Shape a, Shape b) {  // model.cpp:56-62
  if (a == Shape::Sphere && b == Shape::Sphere) return true;
  if ((a == Shape::Sphere && b == Shape::Plane) || (a == Shape::Plane && b == Shape::Sphere)) return true;
  if ((a == Shape::Box && b == Shape::Plane) || (a == Shape::Plane && b == Shape::Box)) return true;
  return false;
}
const char* shape_name(Shape s) {
  switch (s) {
    case Shape::Sphere: return "sphere";
    case Shape::Plane: return "plane";
    case Shape::Box: return "box";
  }
  return "?";
}

}  // namespace

int joint_row_count(JointType t) {  // model.cpp:75-83
  switch (t) {
    case JointType::Fixed: return 6;
    case JointType::Revolute: return 5;
    case JointType::Prismatic: return 5;
    case JointType::Spherical: return 3;
  }
  return 0;
}

// build_model: model.cpp:100-307
MechanismModel build_model(const SceneDescription& scene) {
  MechanismModel m;
  m.name = scene.name;
  m.gravity = scene.gravity;
  m.box_box = scene.box_box;  // extension flag (see box_box in the contacts section)
  std::map<std::string, int> body_ids;
  for (const SceneBody& sb : scene.bodies) {
    if (sb.name == "world" || body_ids.count(sb.name))
      throw ModelError(DuplicateName, "body name '" + sb.name + "' is reserved or duplicated");
    body_ids[sb.name] = (int)m.bodies.size();
    BodySpec b;
    b.name = sb.name;
    b.inertia.mass = sb.mass;
    b.inertia.body_inertia = sb.inertia;
    b.initial_pose = sb.pose;
    b.initial_pose.orientation.normalize();
    b.initial_twist = sb.twist;
    validate_inertia(b);
    m.bodies.push_back(b);
  }
  auto resolve = [&](const std::string& name, const std::string& ctx) -> int {
    if (name == "world") return kWorld;
    auto it = body_ids.find(name);
    if (it == body_ids.end()) throw ModelError(InvalidReference, ctx + ": unknown body '" + name + "'");
    return it->second;
  };
  std::map<std::string, int> joint_names;
  for (const SceneJoint& sj : scene.joints) {
    if (joint_names.count(sj.name))
      throw ModelError(DuplicateName, "duplicate joint name '" + sj.name + "'");
    joint_names[sj.name] = (int)m.joints.size();
    JointSpec j;
    j.name = sj.name;
    j.type = parse_joint_type(sj.type, sj.name);
    j.parent = resolve(sj.parent, "joint '" + sj.name + "'");
    j.child = resolve(sj.child, "joint '" + sj.name + "'");
    if (j.child == kWorld)
      throw ModelError(InvalidReference, "joint '" + sj.name +
                                             "': child must be a body (use parent=\"world\" to anchor)");
    if (j.parent == j.child)
      throw ModelError(InvalidReference, "joint '" + sj.name + "': parent and child must differ");
    j.frame_in_parent = sj.frame_in_parent;
    j.frame_in_child = sj.frame_in_child;
    const bool has_axis = j.type == JointType::Revolute || j.type == JointType::Prismatic;
    if (has_axis) {
      const double n = norm(sj.axis);
      if (std::abs(n - 1.0) > 1e-6)
        throw ModelError(NonUnitAxis, "joint '" + sj.name + "': axis must be unit length");
      j.axis = sj.axis / n;
    }
    if (sj.has_limits) {
      if (!has_axis)
        throw ModelError(UnsupportedOnJointType,
                         "joint '" + sj.name + "': limits are only supported on revolute/prismatic joints");
      if (!(sj.lower < sj.upper))
        throw ModelError(BadLimits, "joint '" + sj.name + "': lower limit must be below upper limit");
      j.has_limits = true;
      j.lower = sj.lower;
      j.upper = sj.upper;
    }
    if (sj.kp < 0 || sj.kd < 0 || sj.armature < 0 || sj.damping < 0)
      throw ModelError(BadLimits,
                       "joint '" + sj.name + "': gains, armature and damping must be nonnegative");
    if ((sj.kp > 0 || sj.kd > 0 || sj.armature > 0 || sj.damping > 0) && !has_axis)
      throw ModelError(UnsupportedOnJointType,
                       "joint '" + sj.name +
                           "': actuation/armature/damping need a joint coordinate (revolute or prismatic)");
    j.has_actuation = sj.kp > 0 || sj.kd > 0;
    j.kp = sj.kp;
    j.kd = sj.kd;
    j.target_rate = sj.target_rate;
    j.armature = sj.armature;
    j.damping = sj.damping;
    m.joints.push_back(j);
  }
  for (const SceneGeom& sg : scene.geoms) {
    GeomSpec g;
    g.body = resolve(sg.body, "geom on '" + sg.body + "'");
    if (sg.shape == "sphere") {
      g.shape = Shape::Sphere;
      if (!(sg.radius > 0)) throw ModelError(BadGeometry, "sphere geom needs a positive radius");
      g.radius = sg.radius;
    } else if (sg.shape == "box") {
      g.shape = Shape::Box;
      if (!(std::min(sg.half_extents.x, std::min(sg.half_extents.y, sg.half_extents.z)) > 0))
        throw ModelError(BadGeometry, "box geom needs positive half extents");
      g.half_extents = sg.half_extents;
    } else if (sg.shape == "plane") {
      g.shape = Shape::Plane;
      const double n = norm(sg.normal);
      if (n < 1e-12) throw ModelError(BadGeometry, "plane normal must be nonzero");
      g.plane_normal = sg.normal / n;
      g.plane_offset = sg.offset;
    } else {
      throw ModelError(BadGeometry, "unknown geom shape '" + sg.shape + "'");
    }
    if (g.shape == Shape::Plane && g.body != kWorld)
      throw ModelError(BadGeometry, "planes must be attached to the world");
    if (g.shape != Shape::Plane && g.body == kWorld)
      throw ModelError(BadGeometry, "only planes may be attached to the world");
    g.mu = sg.mu;
    g.restitution = sg.restitution;
    if (g.mu < 0) throw ModelError(BadGeometry, "friction must be nonnegative");
    if (g.restitution < 0 || g.restitution > 1)
      throw ModelError(BadGeometry, "restitution must lie in [0, 1]");
    m.geoms.push_back(g);
  }
  for (size_t a = 0; a < m.geoms.size(); ++a)  // model.cpp:238-250
    for (size_t b = a + 1; b < m.geoms.size(); ++b) {
      const GeomSpec& ga = m.geoms[a];
      const GeomSpec& gb = m.geoms[b];
      if (ga.body == gb.body) continue;
      if (ga.body == kWorld && gb.body == kWorld) continue;
      if (!pair_supported(ga.shape, gb.shape) && !(scene.box_box && ga.shape == Shape::Box && gb.shape == Shape::Box))
        throw ModelError(UnsupportedCollisionPair, std::string("unsupported collision pair: ") +
                                                       shape_name(ga.shape) + "-" + shape_name(gb.shape));
    }
  // Row layout: model.cpp:254-276
  m.joint_layout.resize(m.joints.size());
  int row = 0;
  for (size_t i = 0; i < m.joints.size(); ++i) {
    JointLayout& lay = m.joint_layout[i];
    lay.row_offset = row;
    lay.row_count = joint_row_count(m.joints[i].type);
    row += lay.row_count;
    if (m.joints[i].type == JointType::Revolute || m.joints[i].type == JointType::Prismatic)
      orthonormal_complement(m.joints[i].axis, lay.comp0, lay.comp1);
  }
  m.n_bilateral_rows = row;
  int dyn = 0;
  for (size_t i = 0; i < m.joints.size(); ++i) {
    JointLayout& lay = m.joint_layout[i];
    lay.dyn_offset = dyn;
    lay.has_pd = m.joints[i].has_actuation;
    lay.has_armature = m.joints[i].armature > 0;
    lay.has_damping = m.joints[i].damping > 0;
    lay.dyn_count = (lay.has_pd ? 1 : 0) + (lay.has_armature ? 1 : 0) + (lay.has_damping ? 1 : 0);
    dyn += lay.dyn_count;
  }
  m.n_dynamics_rows = dyn;
  // Loops E - V + C with the world as a vertex: model.cpp:278-291
  const int n_vertices = m.n_bodies() + 1;
  UnionFind uf(n_vertices);
  const int world_vertex = m.n_bodies();
  for (const JointSpec& j : m.joints) uf.unite(j.parent == kWorld ? world_vertex : j.parent, j.child);
  int components = 0;
  for (int v = 0; v < n_vertices; ++v)
    if (uf.find(v) == v) ++components;
  m.n_loops = (int)m.joints.size() - n_vertices + components;
  // Default PD targets: model.cpp:293-305
  std::vector<Pose> poses;
  for (const BodySpec& b : m.bodies) poses.push_back(b.initial_pose);
  for (size_t i = 0; i < m.joints.size(); ++i) {
    if (!m.joints[i].has_actuation) continue;
    if (scene.joints[i].has_target)
      m.joints[i].target = scene.joints[i].target;
    else
      m.joints[i].target = joint_coordinate(m, (int)i, poses);
  }
  return m;
}

// joint_world_frames: model.cpp:309-324
JointFrames joint_world_frames(const MechanismModel& m, int joint, const std::vector<Pose>& poses) {
  const JointSpec& j = m.joints[joint];
  JointFrames f;
  if (j.parent == kWorld) {
    f.anchor_parent = j.frame_in_parent.position;
    f.frame_parent = j.frame_in_parent.rotation();
  } else {
    const Pose& p = poses[j.parent];
    f.anchor_parent = p.transform(j.frame_in_parent.position);
    f.frame_parent = p.rotation() * j.frame_in_parent.rotation();
  }
  const Pose& c = poses[j.child];
  f.anchor_child = c.transform(j.frame_in_child.position);
  f.frame_child = c.rotation() * j.frame_in_child.rotation();
  return f;
}

// joint_coordinate: model.cpp:326-340
double joint_coordinate(const MechanismModel& m, int joint, const std::vector<Pose>& poses) {
  const JointSpec& j = m.joints[joint];
  const JointFrames f = joint_world_frames(m, joint, poses);
  if (j.type == JointType::Revolute) {
    Quat rel = Quat::from_matrix(f.frame_parent.transpose() * f.frame_child);
    if (rel.w < 0) rel = Quat(-rel.w, -rel.x, -rel.y, -rel.z);
    return 2.0 * std::atan2(dot(j.axis, rel.vec()), rel.w);
  }
  if (j.type == JointType::Prismatic)
    return dot(j.axis, f.frame_parent.transpose() * (f.anchor_child - f.anchor_parent));
  throw ModelError(WrongJointType, "joint '" + j.name + "' has no scalar coordinate");
}

// ============================================================ contacts.cpp
namespace {
double combined_mu(const GeomSpec& a, const GeomSpec& b) { return std::sqrt(a.mu * b.mu); }  // :21
double combined_e(const GeomSpec& a, const GeomSpec& b) { return std::max(a.restitution, b.restitution); }

void sphere_plane(const MechanismModel& m, int sphere, int plane, const std::vector<Pose>& poses,
                  double margin, std::vector<ContactPoint>& out) {  // contacts.cpp:26-43
  const GeomSpec& gs = m.geoms[sphere];
  const GeomSpec& gp = m.geoms[plane];
  const Vec3 c = poses[gs.body].position;
  const double dist = dot(gp.plane_normal, c) - gp.plane_offset;
  const double depth = gs.radius - dist;
  if (depth <= -margin) return;
  ContactPoint cp;
  cp.geom_a = sphere;
  cp.geom_b = plane;
  cp.normal = gp.plane_normal;
  cp.position = c - gs.radius * gp.plane_normal;
  cp.depth = depth;
  cp.mu = combined_mu(gs, gp);
  cp.restitution = combined_e(gs, gp);
  out.push_back(cp);
}

void sphere_sphere(const MechanismModel& m, int a, int b, const std::vector<Pose>& poses,
                   double margin, std::vector<ContactPoint>& out) {  // contacts.cpp:45-64
  const GeomSpec& ga = m.geoms[a];
  const GeomSpec& gb = m.geoms[b];
  const Vec3 ca = poses[ga.body].position;
  const Vec3 cb = poses[gb.body].position;
  const Vec3 delta = ca - cb;
  const double dist = norm(delta);
  const double depth = ga.radius + gb.radius - dist;
  if (depth <= -margin) return;
  ContactPoint cp;
  cp.geom_a = a;
  cp.geom_b = b;
  cp.normal = dist > 1e-12 ? delta / dist : Vec3(0, 0, 1);
  cp.position = 0.5 * ((ca - ga.radius * cp.normal) + (cb + gb.radius * cp.normal));
  cp.depth = depth;
  cp.mu = combined_mu(ga, gb);
  cp.restitution = combined_e(ga, gb);
  out.push_back(cp);
}

void box_plane(const MechanismModel& m, int box, int plane, const std::vector<Pose>& poses,
               double margin, std::vector<ContactPoint>& out) {  // contacts.cpp:66-106
  const GeomSpec& gb = m.geoms[box];
  const GeomSpec& gp = m.geoms[plane];
  const Vec3 pos = poses[gb.body].position;
  const Mat3 rot = poses[gb.body].rotation();
  struct Corner {
    int index;
    Vec3 point;
    double depth;
  };
  std::vector<Corner> hits;
  for (int k = 0; k < 8; ++k) {
    const Vec3 local((k & 1) ? gb.half_extents.x : -gb.half_extents.x,
                     (k & 2) ? gb.half_extents.y : -gb.half_extents.y,
                     (k & 4) ? gb.half_extents.z : -gb.half_extents.z);
    const Vec3 p = pos + rot * local;
    const double depth = gp.plane_offset - dot(gp.plane_normal, p);
    if (depth > -margin) hits.push_back({k, p, depth});
  }
  if (hits.size() > 4) {
    std::stable_sort(hits.begin(), hits.end(),
                     [](const Corner& a, const Corner& b) { return a.depth > b.depth; });
    hits.resize(4);
  }
  std::sort(hits.begin(), hits.end(), [](const Corner& a, const Corner& b) { return a.index < b.index; });
  for (const Corner& c : hits) {
    ContactPoint cp;
    cp.geom_a = box;
    cp.geom_b = plane;
    cp.normal = gp.plane_normal;
    cp.position = c.point;
    cp.depth = c.depth;
    cp.mu = combined_mu(gb, gp);
    cp.restitution = combined_e(gb, gp);
    out.push_back(cp);
  }
}

// ---- box_box: EXTENSION, not in the reference (it rejects box-box pairs,
// model.cpp:56-62), so parity is unpinned: this restatement and the device
// narrow phase (kd_assemble.cu) implement the same algorithm.
//   SAT over the 15 axes (3 + 3 face normals, 9 edge cross products; edge
//   axes shorter than 1e-6 skipped); any axis with overlap <= -margin separates.
//   Face case (a face axis has the least overlap, edges preferred only below
//   best_face - 1e-5 - 0.05 |best_face|): the incident face of the other box
//   (most anti-parallel) is clipped against the reference face's four side
//   planes (Sutherland-Hodgman, order +s1 -s1 +s2 -s2); each clipped point
//   with depth = -(p - face_center) . n_face > -margin becomes a contact at the
//   midpoint of the point and its projection on the reference face; more than
//   4 -> the deepest (first on ties), then three farthest-point picks (largest
//   minimum squared distance to the picked points, first on ties), emitted in
//   clip order.
//   Edge case: one contact at the midpoint of the closest points of the two
//   supporting edges, depth = the axis overlap.
//   Normal from b to a (the sphere_sphere convention), geom_a < geom_b.
void box_box(const MechanismModel& m, int a, int b, const std::vector<Pose>& poses, double margin,
             std::vector<ContactPoint>& out) {
  const GeomSpec& ga = m.geoms[a];
  const GeomSpec& gb = m.geoms[b];
  const Vec3 ca = poses[ga.body].position, cb = poses[gb.body].position;
  const Mat3 Ra = poses[ga.body].rotation(), Rb = poses[gb.body].rotation();
  const Vec3 ha = ga.half_extents, hb = gb.half_extents;
  const Vec3 d = ca - cb;
  auto radius = [](const Mat3& R, const Vec3& h, const Vec3& L) {
    return (h.x * std::abs(dot(R.col(0), L)) + h.y * std::abs(dot(R.col(1), L))) + h.z * std::abs(dot(R.col(2), L));
  };
  double best_face = 1e300, best_edge = 1e300;
  int face = -1, ei = -1, ej = -1;
  for (int f = 0; f < 6; ++f) {
    const Vec3 L = f < 3 ? Ra.col(f) : Rb.col(f - 3);
    const double ov = (radius(Ra, ha, L) + radius(Rb, hb, L)) - std::abs(dot(d, L));
    if (ov <= -margin) return;
    if (ov < best_face) {
      best_face = ov;
      face = f;
    }
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      Vec3 L = cross(Ra.col(i), Rb.col(j));
      const double l = norm(L);
      if (l < 1e-6) continue;
      L = L / l;
      const double ov = (radius(Ra, ha, L) + radius(Rb, hb, L)) - std::abs(dot(d, L));
      if (ov <= -margin) return;
      if (ov < best_edge) {
        best_edge = ov;
        ei = i;
        ej = j;
      }
    }
  const double mu = combined_mu(ga, gb), e = combined_e(ga, gb);
  if (ei >= 0 && best_edge < best_face - 1e-5 - 0.05 * std::abs(best_face)) {
    Vec3 n = normalized(cross(Ra.col(ei), Rb.col(ej)));
    if (dot(d, n) < 0) n = -n;
    Vec3 pa = ca, pb = cb;
    for (int k = 0; k < 3; ++k) {
      if (k != ei) pa = pa + (dot(Ra.col(k), n) > 0 ? -ha[k] : ha[k]) * Ra.col(k);
      if (k != ej) pb = pb + (dot(Rb.col(k), n) > 0 ? hb[k] : -hb[k]) * Rb.col(k);
    }
    const Vec3 da = Ra.col(ei), db = Rb.col(ej), r = pa - pb;
    const double a12 = dot(da, db), b1 = dot(da, r), b2 = dot(db, r), den = 1.0 - a12 * a12;
    double s = den > 1e-12 ? (a12 * b2 - b1) / den : 0.0;
    s = std::min(std::max(s, -ha[ei]), ha[ei]);
    double t = b2 + s * a12;
    t = std::min(std::max(t, -hb[ej]), hb[ej]);
    ContactPoint cp;
    cp.geom_a = a;
    cp.geom_b = b;
    cp.normal = n;
    cp.position = 0.5 * ((pa + s * da) + (pb + t * db));
    cp.depth = best_edge;
    cp.mu = mu;
    cp.restitution = e;
    out.push_back(cp);
    return;
  }
  // face case: reference box R (owner of the face axis), incident box I
  const bool refA = face < 3;
  const int fi = refA ? face : face - 3;
  const Mat3& RR = refA ? Ra : Rb;
  const Mat3& RI = refA ? Rb : Ra;
  const Vec3 cR = refA ? ca : cb, cI = refA ? cb : ca;
  const Vec3 hR = refA ? ha : hb, hI = refA ? hb : ha;
  const Vec3 L = RR.col(fi);
  const double sdl = dot(d, L);
  // outward normal of the reference face toward the other box; contact normal b -> a
  const Vec3 nf = refA ? (sdl > 0 ? -L : L) : (sdl < 0 ? -L : L);
  const Vec3 n = refA ? -nf : nf;
  int k = 0;
  double best = -1.0;
  for (int q = 0; q < 3; ++q) {
    const double c = std::abs(dot(RI.col(q), nf));
    if (c > best) {
      best = c;
      k = q;
    }
  }
  const Vec3 fnI = dot(RI.col(k), nf) > 0 ? -RI.col(k) : RI.col(k);
  const int k1 = k == 0 ? 1 : 0, k2 = k == 2 ? 1 : 2;
  const Vec3 fc = cI + hI[k] * fnI, u1 = hI[k1] * RI.col(k1), u2 = hI[k2] * RI.col(k2);
  Vec3 poly[8], tmp[8];
  int np = 4;
  poly[0] = (fc - u1) - u2;
  poly[1] = (fc + u1) - u2;
  poly[2] = (fc + u1) + u2;
  poly[3] = (fc - u1) + u2;
  const int i1 = fi == 0 ? 1 : 0, i2 = fi == 2 ? 1 : 2;
  const Vec3 rc = cR + hR[fi] * nf;
  for (int pl = 0; pl < 4 && np > 0; ++pl) {
    const Vec3 sdir = (pl & 1) ? -RR.col(pl < 2 ? i1 : i2) : RR.col(pl < 2 ? i1 : i2);
    const double ext = hR[pl < 2 ? i1 : i2];
    int nt = 0;
    Vec3 prev = poly[np - 1];
    double dp = dot(prev - rc, sdir) - ext;
    for (int q = 0; q < np; ++q) {
      const Vec3 cur = poly[q];
      const double dc = dot(cur - rc, sdir) - ext;
      if (dc <= 0) {
        if (dp > 0) tmp[nt++] = prev + (dp / (dp - dc)) * (cur - prev);
        tmp[nt++] = cur;
      } else if (dp <= 0) {
        tmp[nt++] = prev + (dp / (dp - dc)) * (cur - prev);
      }
      prev = cur;
      dp = dc;
    }
    np = nt;
    for (int q = 0; q < np; ++q) poly[q] = tmp[q];
  }
  struct Hit {
    int index;
    Vec3 point;
    double depth;
  };
  std::vector<Hit> hits;
  for (int q = 0; q < np; ++q) {
    const double depth = -dot(poly[q] - rc, nf);
    if (depth > -margin) hits.push_back({q, poly[q] + (0.5 * depth) * nf, depth});
  }
  if (hits.size() > 4) {  // the deepest point, then farthest-point picks (spread support), clip order
    std::vector<int> pick;
    int first = 0;
    for (int q = 1; q < (int)hits.size(); ++q)
      if (hits[q].depth > hits[first].depth) first = q;
    pick.push_back(first);
    while (pick.size() < 4) {
      int bq = -1;
      double bd = -1.0;
      for (int q = 0; q < (int)hits.size(); ++q) {
        double md = 1e300;
        for (int pq : pick) md = std::min(md, squared_norm(hits[q].point - hits[pq].point));
        if (md > bd) {
          bd = md;
          bq = q;
        }
      }
      pick.push_back(bq);
    }
    std::sort(pick.begin(), pick.end());
    std::vector<Hit> kept;
    for (int q : pick) kept.push_back(hits[q]);
    hits = kept;
  }
  for (const Hit& h : hits) {
    ContactPoint cp;
    cp.geom_a = a;
    cp.geom_b = b;
    cp.normal = n;
    cp.position = h.point;
    cp.depth = h.depth;
    cp.mu = mu;
    cp.restitution = e;
    out.push_back(cp);
  }
}
}  // namespace

// contact_frame: contacts.cpp:110-117
Mat3 contact_frame(const Vec3& n) {
  Vec3 t1, t2;
  orthonormal_complement(n, t1, t2);
  Mat3 f;
  for (int r = 0; r < 3; ++r) {
    f(r, 0) = n[r];
    f(r, 1) = t1[r];
    f(r, 2) = t2[r];
  }
  return f;
}

// collide: contacts.cpp:119-145
std::vector<ContactPoint> collide(const MechanismModel& m, const std::vector<Pose>& poses, double margin) {
  std::vector<ContactPoint> out;
  const int n = (int)m.geoms.size();
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const GeomSpec& gi = m.geoms[i];
      const GeomSpec& gj = m.geoms[j];
      if (gi.body == gj.body) continue;
      if (gi.body == kWorld && gj.body == kWorld) continue;
      if (gi.shape == Shape::Sphere && gj.shape == Shape::Sphere) sphere_sphere(m, i, j, poses, margin, out);
      else if (gi.shape == Shape::Sphere && gj.shape == Shape::Plane) sphere_plane(m, i, j, poses, margin, out);
      else if (gi.shape == Shape::Plane && gj.shape == Shape::Sphere) sphere_plane(m, j, i, poses, margin, out);
      else if (gi.shape == Shape::Box && gj.shape == Shape::Plane) box_plane(m, i, j, poses, margin, out);
      else if (gi.shape == Shape::Plane && gj.shape == Shape::Box) box_plane(m, j, i, poses, margin, out);
      else if (gi.shape == Shape::Box && gj.shape == Shape::Box && m.box_box) box_box(m, i, j, poses, margin, out);
    }
  return out;
}

// match_warmstart: contacts.cpp:147-182
std::vector<ContactInit> match_warmstart(const std::vector<ReactionCacheEntry>& cache,
                                         const std::vector<ContactPoint>& contacts, double tolerance) {
  std::vector<ContactInit> init(contacts.size());
  struct Candidate {
    double dist;
    int entry, contact;
  };
  std::vector<Candidate> cand;
  for (size_t e = 0; e < cache.size(); ++e)
    for (size_t c = 0; c < contacts.size(); ++c) {
      if (cache[e].geom_a != contacts[c].geom_a || cache[e].geom_b != contacts[c].geom_b) continue;
      const double d = norm(cache[e].position - contacts[c].position);
      if (d <= tolerance) cand.push_back({d, (int)e, (int)c});
    }
  std::sort(cand.begin(), cand.end(), [](const Candidate& a, const Candidate& b) {
    if (a.dist != b.dist) return a.dist < b.dist;
    if (a.entry != b.entry) return a.entry < b.entry;
    return a.contact < b.contact;
  });
  std::vector<bool> used(cache.size(), false), done(contacts.size(), false);
  for (const Candidate& c : cand) {
    if (used[c.entry] || done[c.contact]) continue;
    used[c.entry] = true;
    done[c.contact] = true;
    init[c.contact].impulse = cache[c.entry].impulse;
    init[c.contact].dual = cache[c.entry].dual;
  }
  return init;
}

// ============================================================ constraints.cpp
double JacobianRow::dot(const Vec& u) const {  // constraints.hpp:25-30
  double s = 0;
  if (body_a >= 0) {
    double t = 0;
    for (int k = 0; k < 6; ++k) t += block_a[k] * u[6 * body_a + k];
    s += t;
  }
  if (body_b >= 0) {
    double t = 0;
    for (int k = 0; k < 6; ++k) t += block_b[k] * u[6 * body_b + k];
    s += t;
  }
  return s;
}

namespace {
void set_block(Row6& b, const Vec3& lin, const Vec3& ang) {
  b[0] = lin.x;
  b[1] = lin.y;
  b[2] = lin.z;
  b[3] = ang.x;
  b[4] = ang.y;
  b[5] = ang.z;
}

struct JointRows {
  std::vector<JacobianRow> rows;
  std::vector<double> f;
};

// build_joint_rows: constraints.cpp:20-109
JointRows build_joint_rows(const MechanismModel& m, int joint, const std::vector<Pose>& poses) {
  const JointSpec& spec = m.joints[joint];
  const JointLayout& lay = m.joint_layout[joint];
  const JointFrames fr = joint_world_frames(m, joint, poses);
  const Mat3 wpt = fr.frame_parent.transpose();
  const int child = spec.child;
  const Vec3 lever_child = fr.anchor_child - poses[child].position;

  JacobianRow pos_rows[3];
  const Vec3 f_pos = wpt * (fr.anchor_child - fr.anchor_parent);
  {
    const Mat3 child_lin = wpt;
    const Mat3 child_ang = (-wpt) * skew(lever_child);
    Mat3 parent_lin, parent_ang;
    if (spec.parent != kWorld) {
      parent_lin = -wpt;
      parent_ang = wpt * skew(fr.anchor_child - poses[spec.parent].position);
    }
    for (int r = 0; r < 3; ++r) {
      pos_rows[r].body_a = child;
      set_block(pos_rows[r].block_a, child_lin.row(r), child_ang.row(r));
      if (spec.parent != kWorld) {
        pos_rows[r].body_b = spec.parent;
        set_block(pos_rows[r].block_b, parent_lin.row(r), parent_ang.row(r));
      }
    }
  }
  JacobianRow rot_rows[3];
  Vec3 f_rot;
  if (spec.type != JointType::Spherical) {
    const Mat3 rel = wpt * fr.frame_child;
    f_rot = so3_log(rel);
    const Mat3 ljin = left_jacobian_inverse(f_rot);
    const Mat3 child_ang = ljin * wpt;
    for (int r = 0; r < 3; ++r) {
      rot_rows[r].body_a = child;
      set_block(rot_rows[r].block_a, Vec3(), child_ang.row(r));
      if (spec.parent != kWorld) {
        rot_rows[r].body_b = spec.parent;
        set_block(rot_rows[r].block_b, Vec3(), -child_ang.row(r));
      }
    }
  }
  JointRows out;
  auto push = [&](const JacobianRow& row, double fv) {
    out.rows.push_back(row);
    out.f.push_back(fv);
  };
  auto push_combined = [&](const JacobianRow base[3], const Vec3& fvec, const Vec3& w) {
    JacobianRow row;
    row.body_a = base[0].body_a;
    row.body_b = base[0].body_b;
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 6; ++k) {
        row.block_a[k] += w[r] * base[r].block_a[k];
        row.block_b[k] += w[r] * base[r].block_b[k];
      }
    push(row, dot(w, fvec));
  };
  switch (spec.type) {
    case JointType::Fixed:
      for (int r = 0; r < 3; ++r) push(pos_rows[r], f_pos[r]);
      for (int r = 0; r < 3; ++r) push(rot_rows[r], f_rot[r]);
      break;
    case JointType::Revolute:
      for (int r = 0; r < 3; ++r) push(pos_rows[r], f_pos[r]);
      push_combined(rot_rows, f_rot, lay.comp0);
      push_combined(rot_rows, f_rot, lay.comp1);
      break;
    case JointType::Prismatic:
      push_combined(pos_rows, f_pos, lay.comp0);
      push_combined(pos_rows, f_pos, lay.comp1);
      for (int r = 0; r < 3; ++r) push(rot_rows[r], f_rot[r]);
      break;
    case JointType::Spherical:
      for (int r = 0; r < 3; ++r) push(pos_rows[r], f_pos[r]);
      break;
  }
  return out;
}

double clamp_abs(double v, double cap) { return std::clamp(v, -cap, cap); }  // constraints.cpp:111
}  // namespace

// apply_jacobian / _transpose: constraints.cpp:115-129
Vec ConstraintSet::apply_jacobian(const Vec& u) const {
  Vec out(n_rows);
  for (int r = 0; r < n_rows; ++r) out[r] = rows[r].dot(u);
  return out;
}
Vec ConstraintSet::apply_jacobian_transpose(const Vec& lambda) const {
  Vec out(6 * n_bodies, 0.0);
  for (int r = 0; r < n_rows; ++r) {
    const JacobianRow& row = rows[r];
    if (row.body_a >= 0)
      for (int k = 0; k < 6; ++k) out[6 * row.body_a + k] += row.block_a[k] * lambda[r];
    if (row.body_b >= 0)
      for (int k = 0; k < 6; ++k) out[6 * row.body_b + k] += row.block_b[k] * lambda[r];
  }
  return out;
}

// build_bilateral: constraints.cpp:141-154
BilateralBlock build_bilateral(const MechanismModel& m, const std::vector<Pose>& poses) {
  BilateralBlock out;
  out.f.resize(m.n_bilateral_rows);
  int row = 0;
  for (size_t j = 0; j < m.joints.size(); ++j) {
    JointRows jr = build_joint_rows(m, (int)j, poses);
    for (size_t k = 0; k < jr.rows.size(); ++k) {
      out.rows.push_back(jr.rows[k]);
      out.f[row++] = jr.f[k];
    }
  }
  return out;
}

// coordinate_rate_row: constraints.cpp:160-187
JacobianRow coordinate_rate_row(const MechanismModel& m, int joint, const std::vector<Pose>& poses) {
  const JointSpec& spec = m.joints[joint];
  if (spec.type != JointType::Revolute && spec.type != JointType::Prismatic)
    throw ModelError(WrongJointType, "joint '" + spec.name + "' has no scalar coordinate");
  const JointFrames fr = joint_world_frames(m, joint, poses);
  const Vec3 axis_w = fr.frame_parent * spec.axis;
  JacobianRow row;
  row.body_a = spec.child;
  if (spec.type == JointType::Revolute) {
    set_block(row.block_a, Vec3(), axis_w);
    if (spec.parent != kWorld) {
      row.body_b = spec.parent;
      set_block(row.block_b, Vec3(), -axis_w);
    }
  } else {
    const Vec3 lever_child = fr.anchor_child - poses[spec.child].position;
    set_block(row.block_a, axis_w, row_times(-axis_w, skew(lever_child)));
    if (spec.parent != kWorld) {
      row.body_b = spec.parent;
      set_block(row.block_b, -axis_w, row_times(axis_w, skew(fr.anchor_child - poses[spec.parent].position)));
    }
  }
  return row;
}

// assemble_constraints: constraints.cpp:189-329
ConstraintSet assemble_constraints(const MechanismModel& m, const std::vector<Pose>& poses,
                                   const std::vector<Twist>& twists,
                                   const std::vector<ContactPoint>& contacts, const AssembleConfig& cfg) {
  ConstraintSet cs;
  cs.n_bodies = m.n_bodies();
  cs.n_bilateral = m.n_bilateral_rows;
  cs.n_dynamics = m.n_dynamics_rows;
  cs.contacts = contacts;
  const double dt = cfg.dt;
  const double bgain = cfg.beta / dt;
  Vec u(6 * cs.n_bodies);
  for (int b = 0; b < cs.n_bodies; ++b) {
    u[6 * b + 0] = twists[b].linear.x;
    u[6 * b + 1] = twists[b].linear.y;
    u[6 * b + 2] = twists[b].linear.z;
    u[6 * b + 3] = twists[b].angular.x;
    u[6 * b + 4] = twists[b].angular.y;
    u[6 * b + 5] = twists[b].angular.z;
  }
  struct LimitRow {
    int joint, bound;
    double gap;
  };
  std::vector<LimitRow> limits;
  std::vector<double> coord(m.joints.size(), 0.0);
  for (size_t j = 0; j < m.joints.size(); ++j) {
    const JointSpec& spec = m.joints[j];
    const bool scalar = spec.type == JointType::Revolute || spec.type == JointType::Prismatic;
    if (scalar && (spec.has_limits || spec.has_actuation)) coord[j] = joint_coordinate(m, (int)j, poses);
    if (!spec.has_limits) continue;
    const double margin = spec.type == JointType::Revolute ? cfg.limit_margin_angular : cfg.limit_margin_linear;
    const double g_lo = coord[j] - spec.lower;
    if (g_lo < margin) limits.push_back({(int)j, 0, g_lo});
    const double g_up = spec.upper - coord[j];
    if (g_up < margin) limits.push_back({(int)j, 1, g_up});
  }
  cs.n_limits = (int)limits.size();
  cs.n_contact_rows = 3 * (int)contacts.size();
  cs.n_rows = cs.n_bilateral + cs.n_dynamics + cs.n_limits + cs.n_contact_rows;
  cs.rows.resize(cs.n_rows);
  cs.bias.assign(cs.n_rows, 0.0);
  cs.reg.assign(cs.n_rows, 0.0);
  cs.limit_gap.resize(cs.n_limits);
  cs.cones.n_rows = cs.n_rows;

  BilateralBlock bb = build_bilateral(m, poses);
  cs.bilateral_f = bb.f;
  for (int r = 0; r < cs.n_bilateral; ++r) {
    cs.rows[r] = bb.rows[r];
    cs.bias[r] = clamp_abs(-bgain * bb.f[r], cfg.bias_clamp);
  }
  int r = cs.n_bilateral;
  for (size_t j = 0; j < m.joints.size(); ++j) {
    const JointSpec& spec = m.joints[j];
    const JointLayout& lay = m.joint_layout[j];
    if (lay.dyn_count == 0) continue;
    const JacobianRow rate = coordinate_rate_row(m, (int)j, poses);
    if (lay.has_pd) {
      cs.rows[r] = rate;
      cs.reg[r] = 1.0 / (dt * (dt * spec.kp + spec.kd));
      cs.bias[r] = (spec.kp * (spec.target - coord[j]) + spec.kd * spec.target_rate) / (dt * spec.kp + spec.kd);
      ++r;
    }
    if (lay.has_armature) {
      cs.rows[r] = rate;
      cs.reg[r] = 1.0 / spec.armature;
      cs.bias[r] = rate.dot(u);
      ++r;
    }
    if (lay.has_damping) {
      cs.rows[r] = rate;
      cs.reg[r] = 1.0 / (dt * spec.damping);
      cs.bias[r] = 0.0;
      ++r;
    }
  }
  if (cs.n_bilateral + cs.n_dynamics > 0)
    cs.cones.groups.push_back({ConeKind::Bilateral, 0, cs.n_bilateral + cs.n_dynamics, 0.0});
  for (int k = 0; k < cs.n_limits; ++k) {
    const LimitRow& lim = limits[k];
    JacobianRow rate = coordinate_rate_row(m, lim.joint, poses);
    if (lim.bound == 1)
      for (int q = 0; q < 6; ++q) {
        rate.block_a[q] = -rate.block_a[q];
        rate.block_b[q] = -rate.block_b[q];
      }
    cs.rows[r] = rate;
    cs.bias[r] = std::min(-bgain * std::min(lim.gap, 0.0), cfg.bias_clamp);
    cs.limit_gap[k] = lim.gap;
    cs.limit_keys.emplace_back(lim.joint, lim.bound);
    cs.cones.groups.push_back({ConeKind::Nonnegative, r, 1, 0.0});
    ++r;
  }
  for (size_t c = 0; c < contacts.size(); ++c) {
    const ContactPoint& cp = contacts[c];
    const Mat3 frame = contact_frame(cp.normal);
    cs.contact_frames.push_back(frame);
    const int body_a = m.geoms[cp.geom_a].body;
    const int body_b = m.geoms[cp.geom_b].body;
    for (int d = 0; d < 3; ++d) {
      const Vec3 dir = frame.col(d);
      JacobianRow row;
      row.body_a = body_a;
      set_block(row.block_a, dir, row_times(-dir, skew(cp.position - poses[body_a].position)));
      if (body_b != kWorld) {
        row.body_b = body_b;
        set_block(row.block_b, -dir, row_times(dir, skew(cp.position - poses[body_b].position)));
      }
      cs.rows[r + d] = row;
    }
    const double vn_minus = cs.rows[r].dot(u);
    double bias_n = std::min(-bgain * std::min(-cp.depth, 0.0), cfg.bias_clamp);
    if (vn_minus < -cfg.impact_velocity_threshold) bias_n += -cp.restitution * vn_minus;
    cs.bias[r] = bias_n;
    cs.cones.groups.push_back({ConeKind::SecondOrder, r, 3, cp.mu});
    r += 3;
  }
  return cs;
}

// constraint_jacobian_fd_check: constraints.cpp:331-365
double constraint_jacobian_fd_check(const MechanismModel& m, const std::vector<Pose>& poses, double step) {
  const BilateralBlock bb = build_bilateral(m, poses);
  const int n_rows = (int)bb.rows.size();
  double worst = 0.0;
  for (int b = 0; b < m.n_bodies(); ++b)
    for (int k = 0; k < 6; ++k) {
      std::vector<Pose> plus(poses), minus(poses);
      if (k < 3) {
        plus[b].position[k] += step;
        minus[b].position[k] -= step;
      } else {
        Vec3 delta;
        delta[k - 3] = 1.0;
        plus[b].orientation = quat_exp((0.5 * step) * delta) * plus[b].orientation;
        minus[b].orientation = quat_exp((-0.5 * step) * delta) * minus[b].orientation;
      }
      const Vec fp = build_bilateral(m, plus).f;
      const Vec fm = build_bilateral(m, minus).f;
      for (int row = 0; row < n_rows; ++row) {
        const double fd = (fp[row] - fm[row]) / (2.0 * step);
        double an = 0.0;
        if (bb.rows[row].body_a == b) an += bb.rows[row].block_a[k];
        if (bb.rows[row].body_b == b) an += bb.rows[row].block_b[k];
        worst = std::max(worst, std::abs(fd - an));
      }
    }
  return worst;
}

// ============================================================ delassus.cpp
namespace {
// fold_inverse_mass: delassus.cpp:12-17
Row6 fold_inverse_mass(const Row6& b, const BodyInertiaWorld& in) {
  Row6 o;
  for (int k = 0; k < 3; ++k) o[k] = b[k] * in.inv_mass;
  const Vec3 t = row_times(Vec3(b[3], b[4], b[5]), in.inv_inertia_world);
  o[3] = t.x;
  o[4] = t.y;
  o[5] = t.z;
  return o;
}
double dot6(const Row6& a, const Row6& b) {
  double s = 0;
  for (int k = 0; k < 6; ++k) s += a[k] * b[k];
  return s;
}
}  // namespace

// world_inertias: delassus.cpp:21-34
std::vector<BodyInertiaWorld> world_inertias(const MechanismModel& m, const std::vector<Pose>& poses) {
  std::vector<BodyInertiaWorld> out(m.n_bodies());
  for (int b = 0; b < m.n_bodies(); ++b) {
    const InertiaBlock& in = m.bodies[b].inertia;
    BodyInertiaWorld& w = out[b];
    w.mass = in.mass;
    w.inv_mass = 1.0 / in.mass;
    w.inertia_world = world_inertia(in, poses[b].orientation);
    const Mat3 inv = llt_inverse3(w.inertia_world);
    w.inv_inertia_world = 0.5 * (inv + inv.transpose());
  }
  return out;
}

// jacobi_preconditioner: delassus.cpp:36-57
Preconditioner jacobi_preconditioner(const ConstraintSet& cs, const std::vector<BodyInertiaWorld>& in) {
  constexpr double kFloor = 1e-12;
  Vec diag(cs.n_rows);
  for (int r = 0; r < cs.n_rows; ++r) {
    const JacobianRow& row = cs.rows[r];
    double d = cs.reg[r];
    if (row.body_a >= 0) d += dot6(fold_inverse_mass(row.block_a, in[row.body_a]), row.block_a);
    if (row.body_b >= 0) d += dot6(fold_inverse_mass(row.block_b, in[row.body_b]), row.block_b);
    diag[r] = d;
  }
  Preconditioner p;
  p.scale.resize(cs.n_rows);
  for (int r = 0; r < cs.n_rows; ++r) p.scale[r] = 1.0 / std::sqrt(std::max(diag[r], kFloor));
  for (const ConeGroup& g : cs.cones.groups)
    if (g.kind == ConeKind::SecondOrder) {
      p.scale[g.begin + 1] = p.scale[g.begin];
      p.scale[g.begin + 2] = p.scale[g.begin];
    }
  return p;
}

// DenseDelassus::factorize (Eigen LLT, delassus.cpp:59-63), unblocked lower
// algorithm (Eigen llt_inplace::unblocked).
bool DenseDelassus::factorize() {
  const int n = matrix.n;
  factor = matrix;
  for (int k = 0; k < n; ++k) {
    double x = factor(k, k);
    for (int j = 0; j < k; ++j) x -= factor(k, j) * factor(k, j);
    if (x <= 0.0) {
      factorized = false;
      return false;
    }
    x = std::sqrt(x);
    factor(k, k) = x;
    for (int i = k + 1; i < n; ++i) {
      double s = factor(i, k);
      for (int j = 0; j < k; ++j) s -= factor(i, j) * factor(k, j);
      factor(i, k) = s / x;
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) factor(i, j) = 0.0;
  factorized = true;
  return true;
}

// DenseDelassus::solve (delassus.cpp:65): L y = b, L^T x = y.
Vec DenseDelassus::solve(const Vec& rhs) const {
  const int n = factor.n;
  Vec y(n);
  for (int i = 0; i < n; ++i) {
    double s = rhs[i];
    for (int j = 0; j < i; ++j) s -= factor(i, j) * y[j];
    y[i] = s / factor(i, i);
  }
  Vec x(n);
  for (int i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int j = i + 1; j < n; ++j) s -= factor(j, i) * x[j];
    x[i] = s / factor(i, i);
  }
  return x;
}

// assemble_dense: delassus.cpp:67-104
DenseDelassus assemble_dense(const ConstraintSet& cs, const std::vector<BodyInertiaWorld>& in,
                             double eta_rho, const Preconditioner* precond) {
  DenseDelassus dd;
  const int n = cs.n_rows;
  dd.matrix.n = n;
  dd.matrix.a.assign((size_t)n * n, 0.0);
  std::vector<std::vector<std::pair<int, const Row6*>>> per_body(cs.n_bodies);
  for (int r = 0; r < n; ++r) {
    const JacobianRow& row = cs.rows[r];
    if (row.body_a >= 0) per_body[row.body_a].push_back({r, &row.block_a});
    if (row.body_b >= 0) per_body[row.body_b].push_back({r, &row.block_b});
  }
  for (int b = 0; b < cs.n_bodies; ++b) {
    const auto& t = per_body[b];
    const int k = (int)t.size();
    if (k == 0) continue;
    std::vector<Row6> gm(k);
    for (int i = 0; i < k; ++i) gm[i] = fold_inverse_mass(*t[i].second, in[b]);
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) dd.matrix(t[i].first, t[j].first) += dot6(gm[i], *t[j].second);
  }
  for (int r = 0; r < n; ++r) dd.matrix(r, r) += cs.reg[r];
  if (precond)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) dd.matrix(i, j) = precond->scale[i] * dd.matrix(i, j) * precond->scale[j];
  for (int r = 0; r < n; ++r) dd.matrix(r, r) += eta_rho;
  DenseMatrix sym = dd.matrix;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) sym(i, j) = 0.5 * (dd.matrix(i, j) + dd.matrix(j, i));
  dd.matrix = sym;
  dd.factorize();
  return dd;
}

// MatrixFreeDelassus::apply: delassus.cpp:106-122
void MatrixFreeDelassus::apply(const Vec& v, Vec& out) const {
  scratch.assign(6 * n_bodies, 0.0);
  const int n = (int)rows.size();
  for (int r = 0; r < n; ++r) {
    const BakedRow& row = rows[r];
    if (row.body_a >= 0)
      for (int k = 0; k < 6; ++k) scratch[6 * row.body_a + k] += row.ja[k] * v[r];
    if (row.body_b >= 0)
      for (int k = 0; k < 6; ++k) scratch[6 * row.body_b + k] += row.jb[k] * v[r];
  }
  out.resize(n);
  for (int r = 0; r < n; ++r) {
    const BakedRow& row = rows[r];
    double s = diag_add[r] * v[r];
    if (row.body_a >= 0) {
      double t = 0;
      for (int k = 0; k < 6; ++k) t += row.jma[k] * scratch[6 * row.body_a + k];
      s += t;
    }
    if (row.body_b >= 0) {
      double t = 0;
      for (int k = 0; k < 6; ++k) t += row.jmb[k] * scratch[6 * row.body_b + k];
      s += t;
    }
    out[r] = s;
  }
}

// bake_jacobian: delassus.cpp:130-154
MatrixFreeDelassus bake_jacobian(const ConstraintSet& cs, const std::vector<BodyInertiaWorld>& in,
                                 const Preconditioner& precond, double eta_rho) {
  MatrixFreeDelassus op;
  op.n_bodies = cs.n_bodies;
  op.rows.resize(cs.n_rows);
  op.diag_add.resize(cs.n_rows);
  for (int r = 0; r < cs.n_rows; ++r) {
    const JacobianRow& row = cs.rows[r];
    BakedRow& b = op.rows[r];
    const double p = precond.scale[r];
    b.body_a = row.body_a;
    b.body_b = row.body_b;
    if (row.body_a >= 0) {
      for (int k = 0; k < 6; ++k) b.ja[k] = p * row.block_a[k];
      b.jma = fold_inverse_mass(b.ja, in[row.body_a]);
    }
    if (row.body_b >= 0) {
      for (int k = 0; k < 6; ++k) b.jb[k] = p * row.block_b[k];
      b.jmb = fold_inverse_mass(b.jb, in[row.body_b]);
    }
    op.diag_add[r] = p * p * cs.reg[r] + eta_rho;
  }
  return op;
}

namespace {
double vdot(const Vec& a, const Vec& b) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
}  // namespace

// cr_solve: delassus.cpp:156-187
CrResult cr_solve(const MatrixFreeDelassus& op, const Vec& rhs, Vec& x, int max_iters,
                  std::vector<double>* history) {
  CrResult res;
  const size_t n = rhs.size();
  if (x.size() != n) x.assign(n, 0.0);
  Vec ax = op.apply(x);
  Vec r(n);
  for (size_t i = 0; i < n; ++i) r[i] = rhs[i] - ax[i];
  Vec ar = op.apply(r);
  Vec p = r, ap = ar;
  double rar = vdot(r, ar);
  if (history) history->push_back(std::sqrt(vdot(r, r)));
  const double breakdown_eps = 1e-30 * std::max(1.0, vdot(rhs, rhs));
  for (int k = 0; k < max_iters; ++k) {
    const double apap = vdot(ap, ap);
    if (!(rar > breakdown_eps) || !(apap > breakdown_eps)) {
      res.breakdown = true;
      break;
    }
    const double alpha = rar / apap;
    for (size_t i = 0; i < n; ++i) x[i] += alpha * p[i];
    for (size_t i = 0; i < n; ++i) r[i] -= alpha * ap[i];
    if (history) history->push_back(std::sqrt(vdot(r, r)));
    ar = op.apply(r);
    const double rar_next = vdot(r, ar);
    const double beta = rar_next / rar;
    for (size_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
    for (size_t i = 0; i < n; ++i) ap[i] = ar[i] + beta * ap[i];
    rar = rar_next;
    ++res.iterations;
  }
  res.residual_norm = std::sqrt(vdot(r, r));
  return res;
}

// DelassusBackend::solve: delassus.cpp:189-197
void DelassusBackend::solve(const Vec& rhs, Vec& x) const {
  if (dense) {
    x = dense->solve(rhs);
    return;
  }
  const CrResult r = cr_solve(*matrix_free, rhs, x, cr_budget);
  cr_iterations_total += r.iterations;
  cr_breakdown = cr_breakdown || (r.breakdown && r.residual_norm > 1e-9 * std::max(1.0, std::sqrt(vdot(rhs, rhs))));
}

// build_backend: delassus.cpp:199-220
DelassusBackend build_backend(const ConstraintSet& cs, const std::vector<BodyInertiaWorld>& in,
                              const Preconditioner& p, double eta_rho, BackendChoice choice, int cr_budget) {
  DelassusBackend be;
  be.cr_budget = cr_budget;
  const bool use_dense =
      choice == BackendChoice::Dense || (choice == BackendChoice::Auto && cs.n_rows <= kDenseRowCrossover);
  if (use_dense) {
    be.dense = std::make_unique<DenseDelassus>(assemble_dense(cs, in, eta_rho, &p));
    if (!be.dense->factorized)
      throw std::runtime_error("Delassus factorization failed on an SPD system (" + std::to_string(cs.n_rows) +
                               " rows, eta+rho = " + std::to_string(eta_rho) + ")");
  } else {
    be.matrix_free = std::make_unique<MatrixFreeDelassus>(bake_jacobian(cs, in, p, eta_rho));
  }
  return be;
}

// ============================================================ padmm.cpp
// project_cone: padmm.cpp:10-42
Vec project_cone(const Vec& w, const ConeProduct& cones) {
  Vec y = w;
  for (const ConeGroup& g : cones.groups) {
    switch (g.kind) {
      case ConeKind::Bilateral: break;
      case ConeKind::Nonnegative:
        for (int k = 0; k < g.dim; ++k) y[g.begin + k] = std::max(0.0, y[g.begin + k]);
        break;
      case ConeKind::SecondOrder: {
        const double wn = w[g.begin];
        const double t0 = w[g.begin + 1], t1 = w[g.begin + 2];
        const double tn = std::sqrt(t0 * t0 + t1 * t1);
        if (tn <= g.mu * wn) break;
        if (g.mu * tn <= -wn) {
          y[g.begin] = y[g.begin + 1] = y[g.begin + 2] = 0.0;
          break;
        }
        const double tau = (wn + g.mu * tn) / (1.0 + g.mu * g.mu);
        y[g.begin] = tau;
        if (tn > 0) {
          y[g.begin + 1] = g.mu * tau * t0 / tn;
          y[g.begin + 2] = g.mu * tau * t1 / tn;
        } else {
          y[g.begin + 1] = 0;
          y[g.begin + 2] = 0;
        }
        break;
      }
    }
  }
  return y;
}

// desaxce_shift: padmm.cpp:44-52
Vec desaxce_shift(const Vec& v, const ConeProduct& cones) {
  Vec s(v.size(), 0.0);
  for (const ConeGroup& g : cones.groups) {
    if (g.kind != ConeKind::SecondOrder) continue;
    s[g.begin] = g.mu * std::hypot(v[g.begin + 1], v[g.begin + 2]);
  }
  return s;
}

// nesterov_next_coefficient: padmm.cpp:54-56
double nesterov_next_coefficient(double a) { return 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * a * a)); }

// nesterov_update: padmm.cpp:58-71
void nesterov_update(PadmmState& st, bool restart) {
  if (restart) {
    st.a = 1.0;
    st.y_hat = st.y;
    st.z_hat = st.z;
    ++st.restarts;
    return;
  }
  const double a_next = nesterov_next_coefficient(st.a);
  const double beta = (st.a - 1.0) / a_next;
  st.y_hat.resize(st.y.size());
  st.z_hat.resize(st.z.size());
  for (size_t i = 0; i < st.y.size(); ++i) st.y_hat[i] = st.y[i] + beta * (st.y[i] - st.y_prev[i]);
  for (size_t i = 0; i < st.z.size(); ++i) st.z_hat[i] = st.z[i] + beta * (st.z[i] - st.z_prev[i]);
  st.a = a_next;
}

// padmm_residuals: padmm.cpp:73-85
void padmm_residuals(const Vec& x, const Vec& y, const Vec& y_prev, const Vec& z, double rho,
                     const ConeProduct& cones, double& r_p, double& r_d, double& r_c) {
  r_p = 0.0;
  double dmax = 0.0;
  for (size_t i = 0; i < x.size(); ++i) {
    r_p = std::max(r_p, std::abs(x[i] - y[i]));
    dmax = std::max(dmax, std::abs(y[i] - y_prev[i]));
  }
  r_d = rho * dmax;
  r_c = 0.0;
  for (const ConeGroup& g : cones.groups) {
    if (g.kind == ConeKind::Bilateral) continue;
    double yn = 0, zn = 0;
    for (int k = 0; k < g.dim; ++k) {
      yn = std::max(yn, std::abs(y[g.begin + k]));
      zn = std::max(zn, std::abs(z[g.begin + k]));
    }
    r_c = std::max(r_c, std::min(yn, zn));
  }
}

// padmm_solve: padmm.cpp:87-159
PadmmResult padmm_solve(const DelassusBackend& backend, const Vec& v_f, const ConeProduct& cones,
                        const PadmmInit& init, const PadmmConfig& cfg, std::vector<double>* hist) {
  const int n = (int)v_f.size();
  PadmmResult result;
  if (n == 0) return result;
  const double eta = cfg.eta, rho = cfg.rho;
  PadmmState st;
  st.x = (int)init.x0.size() == n ? init.x0 : Vec(n, 0.0);
  st.z = (int)init.z0.size() == n ? init.z0 : Vec(n, 0.0);
  st.y = project_cone(st.x, cones);
  st.y_prev = st.y;
  st.z_prev = st.z;
  st.y_hat = st.y;
  st.z_hat = st.z;
  double prev_combined = std::numeric_limits<double>::infinity();
  Vec rhs(n), w(n), y_new, z_new(n);
  bool converged = false;
  for (st.iteration = 1; st.iteration <= cfg.max_iters; ++st.iteration) {
    st.s = desaxce_shift(st.z_hat, cones);
    for (int i = 0; i < n; ++i)
      rhs[i] = -((((v_f[i] + st.s[i]) - eta * st.x[i]) - rho * st.y_hat[i]) - st.z_hat[i]);
    backend.solve(rhs, st.x);
    for (int i = 0; i < n; ++i) w[i] = st.x[i] - st.z_hat[i] / rho;
    y_new = project_cone(w, cones);
    for (int i = 0; i < n; ++i) z_new[i] = st.z_hat[i] - rho * (st.x[i] - y_new[i]);
    padmm_residuals(st.x, y_new, st.y, z_new, rho, cones, st.r_p, st.r_d, st.r_c);
    const double combined = std::max(st.r_p, std::max(st.r_d, st.r_c));
    if (hist) hist->push_back(combined);
    st.y_prev = st.y;
    st.z_prev = st.z;
    st.y = y_new;
    st.z = z_new;
    if (!cfg.fixed_iteration_mode && combined < cfg.eps) {
      converged = true;
      break;
    }
    if (cfg.acceleration) {
      const bool restart_now = cfg.restart && combined > prev_combined;
      nesterov_update(st, restart_now);
    } else {
      st.y_hat = st.y;
      st.z_hat = st.z;
    }
    prev_combined = combined;
  }
  result.lambda = st.y;
  result.z = st.z;
  result.diagnostics.iterations = std::min(st.iteration, cfg.max_iters);
  result.diagnostics.r_p = st.r_p;
  result.diagnostics.r_d = st.r_d;
  result.diagnostics.r_c = st.r_c;
  result.diagnostics.restarts = st.restarts;
  result.diagnostics.converged = converged || std::max(st.r_p, std::max(st.r_d, st.r_c)) < cfg.eps;
  result.diagnostics.cr_iterations = backend.cr_iterations_total;
  result.diagnostics.cr_breakdown = backend.cr_breakdown;
  return result;
}

// ============================================================ stepper.cpp
namespace {
// gather_warmstart: stepper.cpp:19-46
PadmmInit gather_warmstart(const WorldState& state, const ConstraintSet& cs, const Preconditioner& p) {
  PadmmInit init;
  Vec x0(cs.n_rows, 0.0), z0(cs.n_rows, 0.0);
  const int n_jd = cs.n_bilateral + cs.n_dynamics;
  if (state.joint_cache.valid && (int)state.joint_cache.lambda.size() == n_jd)
    for (int i = 0; i < n_jd; ++i) {
      x0[i] = state.joint_cache.lambda[i];
      z0[i] = state.joint_cache.z[i];
    }
  for (int k = 0; k < cs.n_limits; ++k) {
    auto it = state.limit_cache.find(cs.limit_keys[k]);
    if (it != state.limit_cache.end()) {
      x0[cs.first_limit_row() + k] = it->second.first;
      z0[cs.first_limit_row() + k] = it->second.second;
    }
  }
  const std::vector<ContactInit> matched = match_warmstart(state.contact_cache, cs.contacts);
  for (size_t c = 0; c < cs.contacts.size(); ++c) {
    const int r = cs.first_contact_row() + 3 * (int)c;
    for (int d = 0; d < 3; ++d) {
      x0[r + d] = matched[c].impulse[d];
      z0[r + d] = matched[c].dual[d];
    }
  }
  init.x0.resize(cs.n_rows);
  init.z0.resize(cs.n_rows);
  for (int i = 0; i < cs.n_rows; ++i) {
    init.x0[i] = x0[i] / p.scale[i];
    init.z0[i] = z0[i] * p.scale[i];
  }
  return init;
}

// store_caches: stepper.cpp:48-70
void store_caches(WorldState& state, const ConstraintSet& cs, const Vec& lambda, const Vec& z) {
  const int n_jd = cs.n_bilateral + cs.n_dynamics;
  state.joint_cache.lambda.assign(lambda.begin(), lambda.begin() + n_jd);
  state.joint_cache.z.assign(z.begin(), z.begin() + n_jd);
  state.joint_cache.valid = true;
  state.limit_cache.clear();
  for (int k = 0; k < cs.n_limits; ++k) {
    const int r = cs.first_limit_row() + k;
    state.limit_cache[cs.limit_keys[k]] = {lambda[r], z[r]};
  }
  state.contact_cache.clear();
  for (size_t c = 0; c < cs.contacts.size(); ++c) {
    const int r = cs.first_contact_row() + 3 * (int)c;
    ReactionCacheEntry e;
    e.geom_a = cs.contacts[c].geom_a;
    e.geom_b = cs.contacts[c].geom_b;
    e.position = cs.contacts[c].position;
    e.impulse = Vec3(lambda[r], lambda[r + 1], lambda[r + 2]);
    e.dual = Vec3(z[r], z[r + 1], z[r + 2]);
    state.contact_cache.push_back(e);
  }
}
}  // namespace

// initial_state: stepper.cpp:97-106
WorldState initial_state(const MechanismModel& m) {
  WorldState s;
  for (const BodySpec& b : m.bodies) {
    s.poses.push_back(b.initial_pose);
    s.twists.push_back(b.initial_twist);
  }
  return s;
}

// free_forces: stepper.cpp:108-121
Vec free_forces(const MechanismModel& m, const std::vector<Pose>& poses, const std::vector<Twist>& twists) {
  const int nb = m.n_bodies();
  Vec h(6 * nb);
  for (int b = 0; b < nb; ++b) {
    const InertiaBlock& in = m.bodies[b].inertia;
    const Vec3 w = twists[b].angular;
    const Mat3 iw = world_inertia(in, poses[b].orientation);
    const Vec3 f = in.mass * m.gravity;
    const Vec3 t = -cross(w, iw * w);
    h[6 * b + 0] = f.x;
    h[6 * b + 1] = f.y;
    h[6 * b + 2] = f.z;
    h[6 * b + 3] = t.x;
    h[6 * b + 4] = t.y;
    h[6 * b + 5] = t.z;
  }
  return h;
}

static Vec3 seg3(const Vec& v, int off) { return {v[off], v[off + 1], v[off + 2]}; }

// step: stepper.cpp:134-236
StepDiagnostics step(const MechanismModel& m, WorldState& state, const StepConfig& cfg, StepTrace* trace) {
  StepDiagnostics diag;
  const int nb = m.n_bodies();
  const double dt = cfg.dt;
  std::vector<Pose> eval(state.poses);
  if (cfg.integrator == Integrator::MoreauJean)
    for (int b = 0; b < nb; ++b) {
      eval[b].position = eval[b].position + (0.5 * dt) * state.twists[b].linear;
      const Vec3 w_body = eval[b].orientation.to_rotation_matrix().transpose() * state.twists[b].angular;
      eval[b].orientation = quat_integrate(eval[b].orientation, w_body, 0.5 * dt);
    }
  const std::vector<ContactPoint> contacts = collide(m, eval, cfg.contact_margin);
  const ConstraintSet cs = assemble_constraints(m, eval, state.twists, contacts, cfg.assemble_config());
  const std::vector<BodyInertiaWorld> in = world_inertias(m, eval);
  const Vec h = free_forces(m, state.poses, state.twists);
  Vec u_minus(6 * nb), ufree(6 * nb);
  for (int b = 0; b < nb; ++b) {
    const Twist& t = state.twists[b];
    u_minus[6 * b + 0] = t.linear.x;
    u_minus[6 * b + 1] = t.linear.y;
    u_minus[6 * b + 2] = t.linear.z;
    u_minus[6 * b + 3] = t.angular.x;
    u_minus[6 * b + 4] = t.angular.y;
    u_minus[6 * b + 5] = t.angular.z;
    const Vec3 lin = t.linear + (dt * in[b].inv_mass) * seg3(h, 6 * b);
    const Vec3 ang = t.angular + dt * (in[b].inv_inertia_world * seg3(h, 6 * b + 3));
    ufree[6 * b + 0] = lin.x;
    ufree[6 * b + 1] = lin.y;
    ufree[6 * b + 2] = lin.z;
    ufree[6 * b + 3] = ang.x;
    ufree[6 * b + 4] = ang.y;
    ufree[6 * b + 5] = ang.z;
  }
  diag.n_rows = cs.n_rows;
  diag.contact_count = (int)contacts.size();
  diag.first_contact_row = cs.first_contact_row();
  diag.n_limits = cs.n_limits;
  diag.f_inf = 0.0;
  for (int i = 0; i < cs.n_bilateral; ++i) diag.f_inf = std::max(diag.f_inf, std::abs(cs.bilateral_f[i]));
  Vec u_plus = ufree;
  Vec lambda(cs.n_rows, 0.0);
  if (trace) trace->cs = cs;
  if (cs.n_rows > 0) {
    const Preconditioner precond = jacobi_preconditioner(cs, in);
    const Vec jv = cs.apply_jacobian(ufree);
    Vec vfs(cs.n_rows);
    for (int i = 0; i < cs.n_rows; ++i) vfs[i] = precond.scale[i] * (jv[i] - cs.bias[i]);
    const double eta_rho = cfg.solver.eta + cfg.solver.rho;
    const DelassusBackend backend = build_backend(cs, in, precond, eta_rho, cfg.backend, cfg.cr_iters);
    PadmmInit init;
    if (cfg.warm_start) init = gather_warmstart(state, cs, precond);
    const PadmmResult solved =
        padmm_solve(backend, vfs, cs.cones, init, cfg.solver, trace ? &trace->history : nullptr);
    diag.solver = solved.diagnostics;
    for (int i = 0; i < cs.n_rows; ++i) lambda[i] = precond.scale[i] * solved.lambda[i];
    Vec z_phys(cs.n_rows);
    for (int i = 0; i < cs.n_rows; ++i) z_phys[i] = solved.z[i] / precond.scale[i];
    store_caches(state, cs, lambda, z_phys);
    if (trace) {
      trace->precond = precond;
      trace->v_f_scaled = vfs;
      trace->lambda_scaled = solved.lambda;
      trace->z_scaled = solved.z;
    }
    const Vec wrench = cs.apply_jacobian_transpose(lambda);
    for (int b = 0; b < nb; ++b) {
      const Vec3 dl = in[b].inv_mass * seg3(wrench, 6 * b);
      const Vec3 da = in[b].inv_inertia_world * seg3(wrench, 6 * b + 3);
      for (int k = 0; k < 3; ++k) {
        u_plus[6 * b + k] += dl[k];
        u_plus[6 * b + 3 + k] += da[k];
      }
    }
    const Vec ju = cs.apply_jacobian(u_plus);
    double worst = 0.0;
    for (int rr = 0; rr < cs.n_bilateral + cs.n_dynamics; ++rr)
      worst = std::max(worst, precond.scale[rr] * std::abs(ju[rr] + cs.reg[rr] * lambda[rr] - cs.bias[rr]));
    diag.bilateral_velocity_inf = worst;
  }
  diag.impulses = lambda;
  {
    const Vec jt = cs.apply_jacobian_transpose(lambda);
    double worst = 0.0;
    for (int b = 0; b < nb; ++b) {
      Vec3 du_l, du_a;
      for (int k = 0; k < 3; ++k) {
        du_l[k] = u_plus[6 * b + k] - u_minus[6 * b + k];
        du_a[k] = u_plus[6 * b + 3 + k] - u_minus[6 * b + 3 + k];
      }
      const Vec3 ml = in[b].mass * du_l;
      const Vec3 ma = in[b].inertia_world * du_a;
      for (int k = 0; k < 3; ++k) {
        const double vl = (-dt * h[6 * b + k] - jt[6 * b + k]) + ml[k];
        const double va = (-dt * h[6 * b + 3 + k] - jt[6 * b + 3 + k]) + ma[k];
        worst = std::max(worst, std::max(std::abs(vl), std::abs(va)));
      }
    }
    diag.kkt_momentum_inf = worst;
  }
  const bool midpoint = cfg.integrator == Integrator::MoreauJean;
  for (int b = 0; b < nb; ++b) {
    const Vec3 up_l = seg3(u_plus, 6 * b), up_a = seg3(u_plus, 6 * b + 3);
    const Vec3 um_l = seg3(u_minus, 6 * b), um_a = seg3(u_minus, 6 * b + 3);
    state.twists[b].linear = up_l;
    state.twists[b].angular = up_a;
    const Vec3 v_int = midpoint ? 0.5 * (um_l + up_l) : up_l;
    const Vec3 w_int = midpoint ? 0.5 * (um_a + up_a) : up_a;
    state.poses[b].position = state.poses[b].position + dt * v_int;
    const Vec3 w_body = state.poses[b].orientation.to_rotation_matrix().transpose() * w_int;
    state.poses[b].orientation = quat_integrate(state.poses[b].orientation, w_body, dt);
  }
  state.time += dt;
  return diag;
}

// kinetic_energy / potential_energy: stepper.cpp:238-255
double kinetic_energy(const MechanismModel& m, const WorldState& s) {
  double e = 0.0;
  for (int b = 0; b < m.n_bodies(); ++b) {
    const InertiaBlock& in = m.bodies[b].inertia;
    const Mat3 iw = world_inertia(in, s.poses[b].orientation);
    e += 0.5 * in.mass * squared_norm(s.twists[b].linear);
    e += 0.5 * dot(s.twists[b].angular, iw * s.twists[b].angular);
  }
  return e;
}
double potential_energy(const MechanismModel& m, const WorldState& s) {
  double e = 0.0;
  for (int b = 0; b < m.n_bodies(); ++b) e -= m.bodies[b].inertia.mass * dot(m.gravity, s.poses[b].position);
  return e;
}

// ============================================================ batch.cpp
int WorldBatch::add_world(std::shared_ptr<const MechanismModel> model) {  // batch.cpp:8-11
  const WorldState s = initial_state(*model);
  return add_world(std::move(model), s);
}
int WorldBatch::add_world(std::shared_ptr<const MechanismModel> model, const WorldState& s) {  // :13-25
  Entry e;
  e.model = std::move(model);
  e.pose_offset = (int)poses_.size();
  e.twist_offset = (int)twists_.size();
  const int nb = e.model->n_bodies();
  poses_.resize(poses_.size() + 7 * nb);
  twists_.resize(twists_.size() + 6 * nb);
  entries_.push_back(std::move(e));
  traces_.emplace_back();
  const int w = (int)entries_.size() - 1;
  insert_state(w, s);
  return w;
}
WorldState WorldBatch::extract_state(int w) const {  // batch.cpp:27-46
  const Entry& e = entries_[w];
  const int nb = e.model->n_bodies();
  WorldState s;
  s.poses.resize(nb);
  s.twists.resize(nb);
  for (int b = 0; b < nb; ++b) {
    const double* p = &poses_[e.pose_offset + 7 * b];
    s.poses[b].position = Vec3(p[0], p[1], p[2]);
    s.poses[b].orientation = Quat(p[3], p[4], p[5], p[6]);
    const double* t = &twists_[e.twist_offset + 6 * b];
    s.twists[b].linear = Vec3(t[0], t[1], t[2]);
    s.twists[b].angular = Vec3(t[3], t[4], t[5]);
  }
  s.time = e.time;
  s.joint_cache = e.joint_cache;
  s.limit_cache = e.limit_cache;
  s.contact_cache = e.contact_cache;
  return s;
}
void WorldBatch::insert_state(int w, const WorldState& s) {  // batch.cpp:48-72
  Entry& e = entries_[w];
  const int nb = e.model->n_bodies();
  for (int b = 0; b < nb; ++b) {
    double* p = &poses_[e.pose_offset + 7 * b];
    p[0] = s.poses[b].position.x;
    p[1] = s.poses[b].position.y;
    p[2] = s.poses[b].position.z;
    p[3] = s.poses[b].orientation.w;
    p[4] = s.poses[b].orientation.x;
    p[5] = s.poses[b].orientation.y;
    p[6] = s.poses[b].orientation.z;
    double* t = &twists_[e.twist_offset + 6 * b];
    t[0] = s.twists[b].linear.x;
    t[1] = s.twists[b].linear.y;
    t[2] = s.twists[b].linear.z;
    t[3] = s.twists[b].angular.x;
    t[4] = s.twists[b].angular.y;
    t[5] = s.twists[b].angular.z;
  }
  e.time = s.time;
  e.joint_cache = s.joint_cache;
  e.limit_cache = s.limit_cache;
  e.contact_cache = s.contact_cache;
}

// batch_step: batch.cpp:74-110
void batch_step(WorldBatch& batch, const StepConfig& cfg, int n_threads) {
  std::vector<int> work;
  for (int w = 0; w < batch.size(); ++w)
    if (batch.entries_[w].active) work.push_back(w);
  if (work.empty()) return;
  if (n_threads <= 0) {
    n_threads = (int)std::thread::hardware_concurrency();
    if (n_threads <= 0) n_threads = 1;
  }
  n_threads = std::min<int>(n_threads, (int)work.size());
  std::atomic<size_t> next{0};
  auto run = [&]() {
    for (;;) {
      const size_t i = next.fetch_add(1);
      if (i >= work.size()) break;
      const int w = work[i];
      WorldBatch::Entry& e = batch.entries_[w];
      WorldState s = batch.extract_state(w);
      StepTrace tr;
      e.diag = step(*e.model, s, cfg, batch.record_trace ? &tr : nullptr);
      if (batch.record_trace) batch.traces_[w] = std::move(tr);
      e.converged = e.diag.solver.converged;
      batch.insert_state(w, s);
    }
  };
  if (n_threads == 1) {
    run();
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < n_threads; ++t) pool.emplace_back(run);
  for (std::thread& t : pool) t.join();
}

// ---------------------------------------------------------------- fk (fk.cpp:7-106)
namespace {

// fk_residual (fk.cpp:9-24): [bilateral f; coordinate - target], revolute
// differences wrapped with std::remainder(d, 2 pi).
Vec fk_residual(const MechanismModel& m, const std::vector<std::pair<int, double>>& targets,
                const std::vector<Pose>& poses) {
  Vec r = build_bilateral(m, poses).f;
  for (const auto& [joint, target] : targets) {
    double d = joint_coordinate(m, joint, poses) - target;
    if (m.joints[joint].type == JointType::Revolute) d = std::remainder(d, 2.0 * M_PI);
    r.push_back(d);
  }
  return r;
}

// fk_jacobian (fk.cpp:28-52): rows x 6 nb, the angular block of each
// world-frame row post-multiplied by R_i (local chart, q <- q exp(delta/2)).
std::vector<double> fk_jacobian(const MechanismModel& m, const std::vector<std::pair<int, double>>& targets,
                                const std::vector<Pose>& poses, int& n_rows) {
  const BilateralBlock bb = build_bilateral(m, poses);
  const int nf = (int)bb.rows.size(), nt = (int)targets.size(), nc = 6 * m.n_bodies();
  n_rows = nf + nt;
  std::vector<double> j((size_t)n_rows * nc, 0.0);
  auto scatter = [&](int out, const JacobianRow& row) {
    for (int side = 0; side < 2; ++side) {
      const int b = side == 0 ? row.body_a : row.body_b;
      if (b < 0) continue;
      const Row6& blk = side == 0 ? row.block_a : row.block_b;
      const Mat3 rot = poses[b].rotation();
      double* dst = j.data() + (size_t)out * nc + 6 * b;
      for (int k = 0; k < 3; ++k) dst[k] = blk[k];
      for (int c = 0; c < 3; ++c) dst[3 + c] = blk[3] * rot(0, c) + blk[4] * rot(1, c) + blk[5] * rot(2, c);
    }
  };
  for (int r = 0; r < nf; ++r) scatter(r, bb.rows[r]);
  for (int k = 0; k < nt; ++k) scatter(nf + k, coordinate_rate_row(m, targets[k].first, poses));
  return j;
}

// apply_update (fk.cpp:54-62)
std::vector<Pose> fk_apply_update(const std::vector<Pose>& poses, const Vec& delta) {
  std::vector<Pose> out = poses;
  for (size_t b = 0; b < out.size(); ++b) {
    out[b].position = out[b].position + Vec3{delta[6 * b], delta[6 * b + 1], delta[6 * b + 2]};
    out[b].orientation = (out[b].orientation * quat_exp(Vec3{0.5 * delta[6 * b + 3], 0.5 * delta[6 * b + 4],
                                                             0.5 * delta[6 * b + 5]}))
                             .normalized();
  }
  return out;
}

double norm2(const Vec& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}
double norm_inf(const Vec& v) {
  double s = 0.0;
  for (double x : v) s = std::max(s, std::abs(x));
  return s;
}

}  // namespace

FkResult fk_solve(const MechanismModel& m, const std::vector<std::pair<int, double>>& targets,
                  const std::vector<Pose>& initial_poses, const FkConfig& cfg) {
  FkResult res;
  res.poses = initial_poses;
  Vec r = fk_residual(m, targets, res.poses);
  double r_norm = norm2(r);
  res.residual_inf = norm_inf(r);
  if (res.residual_inf < cfg.tolerance) {
    res.converged = true;
    return res;  // already consistent, poses untouched
  }
  const int nc = 6 * m.n_bodies();
  double lm = cfg.lm_initial;
  for (int iter = 0; iter < cfg.max_iters; ++iter) {
    res.iterations = iter + 1;
    int nr = 0;
    const std::vector<double> j = fk_jacobian(m, targets, res.poses, nr);
    // normal = J^T J + lm I ; g = -J^T r
    std::vector<double> a((size_t)nc * nc, 0.0);
    Vec g(nc, 0.0);
    for (int p = 0; p < nc; ++p) {
      for (int q = 0; q <= p; ++q) {
        double s = 0.0;
        for (int k = 0; k < nr; ++k) s += j[(size_t)k * nc + p] * j[(size_t)k * nc + q];
        a[(size_t)p * nc + q] = s;
      }
      a[(size_t)p * nc + p] += lm;
      double t = 0.0;
      for (int k = 0; k < nr; ++k) t += j[(size_t)k * nc + p] * r[k];
      g[p] = -t;
    }
    // unblocked LLT (lower) and the two substitutions
    bool spd = true;
    for (int c = 0; c < nc && spd; ++c) {
      double d = a[(size_t)c * nc + c];
      for (int k = 0; k < c; ++k) d -= a[(size_t)c * nc + k] * a[(size_t)c * nc + k];
      if (!(d > 0.0)) spd = false;
      d = std::sqrt(d);
      a[(size_t)c * nc + c] = d;
      for (int i = c + 1; i < nc; ++i) {
        double v = a[(size_t)i * nc + c];
        for (int k = 0; k < c; ++k) v -= a[(size_t)i * nc + k] * a[(size_t)c * nc + k];
        a[(size_t)i * nc + c] = v / d;
      }
    }
    if (!spd) break;
    Vec delta = g;
    for (int i = 0; i < nc; ++i) {
      for (int k = 0; k < i; ++k) delta[i] -= a[(size_t)i * nc + k] * delta[k];
      delta[i] /= a[(size_t)i * nc + i];
    }
    for (int i = nc - 1; i >= 0; --i) {
      for (int k = i + 1; k < nc; ++k) delta[i] -= a[(size_t)k * nc + i] * delta[k];
      delta[i] /= a[(size_t)i * nc + i];
    }
    const std::vector<Pose> cand = fk_apply_update(res.poses, delta);
    const Vec r_c = fk_residual(m, targets, cand);
    const double cn = norm2(r_c);
    if (cn < r_norm) {
      res.poses = cand;
      r = r_c;
      r_norm = cn;
      res.residual_inf = norm_inf(r);
      lm = std::max(lm / 10.0, 1e-12);
      if (res.residual_inf < cfg.tolerance) {
        res.converged = true;
        return res;
      }
    } else {
      lm *= 10.0;
      if (lm > 1e10) break;  // stuck; report the best iterate
    }
  }
  res.converged = res.residual_inf < cfg.tolerance;
  return res;
}

}  // namespace oracle
