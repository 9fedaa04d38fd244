// oracle_tests.cpp — TEST INFRASTRUCTURE ONLY.
//
// Pins the oracle (oracle.cpp) against the reference's own known-answer tests
// and acceptance criteria (/root/reference/proj/tests/*.cpp).
// Each TEST names the reference test it restates.  Run by tests/test_oracle.py;
// prints one "[PASS]/[FAIL] name" line per test and exits with the number of
// failed tests.  Usage: oracle_tests <scenes_bundle.json> [filter]
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <random>
#include <sstream>

#include "json.hpp"
#include "oracle.hpp"

using namespace oracle;
using nlohmann::json;

namespace {

struct TestCase {
  const char* name;
  std::function<void()> fn;
};
std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
int g_fail_count = 0;
std::string g_fail_msg;
#define TEST(id, name) \
  static void id();    \
  static Reg reg_##id(name, id); \
  static void id()
#define CHECK(cond)                                                          \
  do {                                                                       \
    if (!(cond)) {                                                           \
      ++g_fail_count;                                                        \
      if (g_fail_msg.size() < 400) g_fail_msg += std::string(" line ") + std::to_string(__LINE__) + ": " #cond; \
    }                                                                        \
  } while (0)
#define REQUIRE(cond)   \
  do {                  \
    CHECK(cond);        \
    if (!(cond)) return; \
  } while (0)
bool approx(double a, double b, double eps = 1e-5) {  // doctest::Approx default epsilon
  return std::abs(a - b) <= eps * (1.0 + std::max(std::abs(a), std::abs(b))) ;
}

json g_bundle;

// parse_scene (scene.cpp:86-174) over an already-parsed JSON object.
Vec3 jv3(const json& j, const char* k, Vec3 d) {
  if (!j.contains(k)) return d;
  const json& v = j[k];
  return {v[0].get<double>(), v[1].get<double>(), v[2].get<double>()};
}
Quat jq(const json& j, const char* k) {
  if (!j.contains(k)) return Quat();
  const json& v = j[k];
  Quat q(v[0].get<double>(), v[1].get<double>(), v[2].get<double>(), v[3].get<double>());
  q.normalize();
  return q;
}
double jnum(const json& j, const char* k, double d) { return j.contains(k) ? j[k].get<double>() : d; }

struct LoadedScene {
  SceneDescription scene;
  StepConfig config;
};

LoadedScene scene_from_json(const json& root) {
  LoadedScene ls;
  SceneDescription& s = ls.scene;
  s.name = root.value("name", std::string("scene"));
  s.gravity = jv3(root, "gravity", Vec3(0, 0, -9.81));
  for (const json& jb : root.value("bodies", json::array())) {
    SceneBody b;
    b.name = jb["name"].get<std::string>();
    b.mass = jb["mass"].get<double>();
    const json& in = jb["inertia"];
    if (in[0].is_number()) {
      b.inertia = Mat3::diagonal(Vec3(in[0].get<double>(), in[1].get<double>(), in[2].get<double>()));
    } else {
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) b.inertia(r, c) = in[r][c].get<double>();
    }
    b.pose.position = jv3(jb, "position", Vec3());
    b.pose.orientation = jq(jb, "orientation");
    b.twist.linear = jv3(jb, "linear_velocity", Vec3());
    b.twist.angular = jv3(jb, "angular_velocity", Vec3());
    s.bodies.push_back(b);
  }
  int idx = 0;
  for (const json& jj : root.value("joints", json::array())) {
    SceneJoint j;
    j.name = jj.value("name", "joint" + std::to_string(idx));
    ++idx;
    j.type = jj["type"].get<std::string>();
    j.parent = jj["parent"].get<std::string>();
    j.child = jj["child"].get<std::string>();
    j.frame_in_parent.position = jv3(jj, "parent_position", Vec3());
    j.frame_in_parent.orientation = jq(jj, "parent_orientation");
    j.frame_in_child.position = jv3(jj, "child_position", Vec3());
    j.frame_in_child.orientation = jq(jj, "child_orientation");
    j.axis = jv3(jj, "axis", Vec3(0, 0, 1));
    if (jj.contains("limits")) {
      j.has_limits = true;
      j.lower = jj["limits"][0].get<double>();
      j.upper = jj["limits"][1].get<double>();
    }
    j.kp = jnum(jj, "kp", 0);
    j.kd = jnum(jj, "kd", 0);
    if (jj.contains("target")) {
      j.has_target = true;
      j.target = jj["target"].get<double>();
    }
    j.target_rate = jnum(jj, "target_rate", 0);
    j.armature = jnum(jj, "armature", 0);
    j.damping = jnum(jj, "damping", 0);
    s.joints.push_back(j);
  }
  for (const json& jg : root.value("geoms", json::array())) {
    SceneGeom g;
    g.body = jg["body"].get<std::string>();
    g.shape = jg["shape"].get<std::string>();
    if (g.shape == "sphere") g.radius = jg["radius"].get<double>();
    if (g.shape == "box") g.half_extents = jv3(jg, "half_extents", Vec3());
    if (g.shape == "plane") {
      g.normal = jv3(jg, "normal", Vec3(0, 0, 1));
      g.offset = jnum(jg, "offset", 0);
    }
    g.mu = jnum(jg, "mu", 0);
    g.restitution = jnum(jg, "restitution", 0);
    s.geoms.push_back(g);
  }
  // apply_scene_config (stepper.cpp:74-95)
  if (root.contains("config")) {
    const json& jc = root["config"];
    if (jc.contains("dt")) ls.config.dt = jc["dt"].get<double>();
    if (jc.contains("integrator"))
      ls.config.integrator =
          jc["integrator"].get<std::string>() == "moreau" ? Integrator::MoreauJean : Integrator::SemiImplicitEuler;
    if (jc.contains("backend")) {
      const std::string b = jc["backend"].get<std::string>();
      ls.config.backend = b == "dense" ? BackendChoice::Dense
                          : b == "sparse" ? BackendChoice::MatrixFree
                                          : BackendChoice::Auto;
    }
    if (jc.contains("beta")) ls.config.baumgarte_beta = jc["beta"].get<double>();
    const json& js = jc.contains("solver") ? jc["solver"] : jc;
    if (js.contains("rho")) ls.config.solver.rho = js["rho"].get<double>();
    if (js.contains("eta")) ls.config.solver.eta = js["eta"].get<double>();
    if (js.contains("eps")) ls.config.solver.eps = js["eps"].get<double>();
    if (js.contains("max_iters")) ls.config.solver.max_iters = js["max_iters"].get<int>();
    if (js.contains("cr_iters")) ls.config.cr_iters = js["cr_iters"].get<int>();
  }
  return ls;
}

LoadedScene load(const std::string& name) { return scene_from_json(g_bundle.at(name)); }
MechanismModel load_model(const std::string& name) { return build_model(load(name).scene); }

std::vector<Pose> initial_poses(const MechanismModel& m) {
  std::vector<Pose> p;
  for (const BodySpec& b : m.bodies) p.push_back(b.initial_pose);
  return p;
}

Quat axis_angle(double a, const Vec3& axis) {
  const double s = std::sin(0.5 * a);
  return Quat(std::cos(0.5 * a), s * axis.x, s * axis.y, s * axis.z);
}

SceneBody body(const std::string& name, double inertia = 0.05) {
  SceneBody b;
  b.name = name;
  b.inertia = inertia * Mat3::identity();
  return b;
}

std::mt19937 g_rng(20240812);
Quat random_quat(std::mt19937& rng) {
  std::normal_distribution<double> n;
  Quat q(n(rng), n(rng), n(rng), n(rng));
  q.normalize();
  return q;
}
Vec3 random_vec(std::mt19937& rng, double s = 1.0) {
  std::normal_distribution<double> n(0.0, s);
  return Vec3(n(rng), n(rng), n(rng));
}

double maxabs(const Vec& v) {
  double m = 0;
  for (double x : v) m = std::max(m, std::abs(x));
  return m;
}

bool states_bitwise_equal(const WorldState& a, const WorldState& b) {
  if (a.poses.size() != b.poses.size()) return false;
  for (size_t i = 0; i < a.poses.size(); ++i) {
    if (std::memcmp(&a.poses[i].position, &b.poses[i].position, sizeof(Vec3))) return false;
    if (std::memcmp(&a.poses[i].orientation, &b.poses[i].orientation, sizeof(Quat))) return false;
    if (std::memcmp(&a.twists[i], &b.twists[i], sizeof(Twist))) return false;
  }
  return true;
}

// Golden-section SOC projection oracle (tests/oracles.hpp:17-51).
Vec3 cone_project_oracle(const Vec3& w, double mu) {
  const double wn = w[0];
  const double tnorm = std::hypot(w[1], w[2]);
  if (tnorm <= mu * wn) return w;
  auto obj = [&](double tau) {
    const double dn = tau - wn, dt = mu * tau - tnorm;
    return dn * dn + dt * dt;
  };
  double lo = 0.0, hi = 2.0 * (std::abs(wn) + tnorm + 1.0) * (1.0 + mu);
  const double gr = 0.5 * (std::sqrt(5.0) - 1.0);
  for (int it = 0; it < 300; ++it) {
    const double m1 = hi - gr * (hi - lo), m2 = lo + gr * (hi - lo);
    if (obj(m1) < obj(m2)) hi = m2; else lo = m1;
  }
  double tau = 0.5 * (lo + hi);
  if (obj(0.0) <= obj(tau)) tau = 0.0;
  Vec3 p(tau, 0, 0);
  if (tnorm > 0) {
    p[1] = mu * tau * w[1] / tnorm;
    p[2] = mu * tau * w[2] / tnorm;
  }
  return p;
}

ConeProduct single_soc(double mu) {
  ConeProduct c;
  c.n_rows = 3;
  c.groups.push_back({ConeKind::SecondOrder, 0, 3, mu});
  return c;
}

}  // namespace

// ======================================================================= se3
TEST(se3_zero_rate, "test_se3.cpp:27 quat_integrate zero rate is identity") {
  const Quat q = quat_integrate(Quat(), Vec3(), 0.123);
  CHECK(approx(q.w, 1.0));
  CHECK(norm(q.vec()) < 1e-12);
}
TEST(se3_half_turn, "test_se3.cpp:33 quat_integrate half turn about z") {
  const Quat q = quat_integrate(Quat(), Vec3(0, 0, M_PI), 1.0);
  CHECK(std::abs(q.w) < 1e-12);
  CHECK(std::abs(std::abs(q.z) - 1.0) < 1e-12);
}
TEST(se3_rodrigues, "test_se3.cpp:41 quat_integrate matches Rodrigues") {
  std::mt19937 rng(20240811);
  for (int t = 0; t < 200; ++t) {
    const Quat q = random_quat(rng);
    const Vec3 w = random_vec(rng, 3.0);
    const double dt = std::uniform_real_distribution<double>(1e-4, 0.3)(rng);
    const Mat3 got = quat_integrate(q, w, dt).to_rotation_matrix();
    const Mat3 exp = q.to_rotation_matrix() * so3_exp(dt * w);
    double e = 0;
    for (int k = 0; k < 9; ++k) e = std::max(e, std::abs(got.m[k] - exp.m[k]));
    CHECK(e < 1e-12);
  }
}
TEST(se3_compose, "test_se3.cpp:52 quat_integrate composes over dt") {
  std::mt19937 rng(3);
  for (int t = 0; t < 50; ++t) {
    const Quat q = random_quat(rng);
    const Vec3 w = random_vec(rng, 2.0);
    const Quat a = quat_integrate(quat_integrate(q, w, 0.05), w, 0.11);
    const Quat b = quat_integrate(q, w, 0.16);
    CHECK(std::max({std::abs(a.w - b.w), std::abs(a.x - b.x), std::abs(a.y - b.y), std::abs(a.z - b.z)}) < 1e-10);
  }
}
TEST(se3_small_angle, "test_se3.cpp:63 small-angle branch stays normalized") {
  std::mt19937 rng(9);
  const Quat q = quat_integrate(random_quat(rng), Vec3(1e-10, -2e-10, 5e-11), 1.0);
  CHECK(std::abs(q.norm() - 1.0) < 1e-15);
}
TEST(se3_log_exp, "test_se3.cpp:69 so3 log inverts exp") {
  std::mt19937 rng(4);
  for (int t = 0; t < 100; ++t) {
    Vec3 phi = random_vec(rng, 1.2);
    if (norm(phi) > 0.95 * M_PI) phi = (0.95 * M_PI / norm(phi)) * phi;
    CHECK(norm(so3_log(so3_exp(phi)) - phi) < 1e-10);
  }
}
TEST(se3_jl_inv, "test_se3.cpp:77 left_jacobian_inverse vs numeric derivative") {
  std::mt19937 rng(5);
  for (int t = 0; t < 100; ++t) {
    const Vec3 phi = random_vec(rng, 0.8), delta = random_vec(rng, 1.0);
    const double h = 1e-6;
    const Mat3 e = so3_exp(phi);
    const Vec3 fd = (1.0 / (2.0 * h)) * (so3_log(so3_exp(h * delta) * e) - so3_log(so3_exp(-h * delta) * e));
    CHECK(norm(left_jacobian_inverse(phi) * delta - fd) < 1e-6);
  }
}
TEST(se3_quarter_turn, "test_se3.cpp:99 world inertia permutes axes under a quarter turn") {
  InertiaBlock in;
  in.body_inertia = Mat3::diagonal(Vec3(1, 2, 3));
  const Mat3 iw = world_inertia(in, axis_angle(M_PI / 2, Vec3(0, 0, 1)));
  const Mat3 ex = Mat3::diagonal(Vec3(2, 1, 3));
  double e = 0;
  for (int k = 0; k < 9; ++k) e = std::max(e, std::abs(iw.m[k] - ex.m[k]));
  CHECK(e < 1e-14);
}
TEST(se3_complement, "test_se3.cpp:152 orthonormal_complement is right-handed") {
  std::mt19937 rng(6);
  for (int t = 0; t < 50; ++t) {
    const Vec3 a = normalized(random_vec(rng));
    Vec3 b1, b2;
    orthonormal_complement(a, b1, b2);
    CHECK(std::abs(dot(b1, a)) < 1e-14);
    CHECK(std::abs(dot(b2, a)) < 1e-14);
    CHECK(std::abs(dot(b1, b2)) < 1e-14);
    CHECK(norm(cross(a, b1) - b2) < 1e-14);
  }
}

// ======================================================================= model
TEST(model_fourbar, "test_model.cpp:42 four-bar bookkeeping: 20 rows, 18 DOF, one loop") {
  const MechanismModel m = load_model("fourbar");
  CHECK(m.n_bilateral_rows == 20);
  CHECK(6 * m.n_bodies() == 18);
  CHECK(m.n_loops == 1);
  CHECK(m.n_dynamics_rows == 1);
  CHECK(m.joint_layout[0].row_offset == 0);
  CHECK(m.joint_layout[1].row_offset == 5);
  CHECK(m.joint_layout[2].row_offset == 10);
  CHECK(m.joint_layout[3].row_offset == 15);
}
TEST(model_legs_loops, "test_model.cpp:57 31-body 36-joint graph has six loops") {
  SceneDescription s;
  for (int i = 0; i < 31; ++i) s.bodies.push_back(body("b" + std::to_string(i), 0.01));
  auto rev = [](const std::string& n, const std::string& p, const std::string& c) {
    SceneJoint j;
    j.name = n;
    j.type = "revolute";
    j.parent = p;
    j.child = c;
    return j;
  };
  for (int i = 1; i < 31; ++i)
    s.joints.push_back(rev("t" + std::to_string(i), "b" + std::to_string(i - 1), "b" + std::to_string(i)));
  for (int k = 0; k < 6; ++k)
    s.joints.push_back(rev("loop" + std::to_string(k), "b" + std::to_string(3 * k), "b" + std::to_string(3 * k + 2)));
  const MechanismModel m = build_model(s);
  CHECK(m.joints.size() == 36);
  CHECK(m.n_loops == 6);
}
TEST(model_validation, "test_model.cpp:80 validation failures carry distinct codes and messages") {
  auto minimal = [] {
    SceneDescription s;
    s.bodies.push_back(body("a", 0.1));
    s.bodies[0].mass = 1.0;
    return s;
  };
  auto rev = [](const std::string& p, const std::string& c) {
    SceneJoint j;
    j.name = "j";
    j.type = "revolute";
    j.parent = p;
    j.child = c;
    return j;
  };
  auto expect = [](const SceneDescription& s, int code, const char* frag) {
    try {
      build_model(s);
      return false;
    } catch (const ModelError& e) {
      return e.code == code && std::string(e.what()).find(frag) != std::string::npos;
    }
  };
  {
    auto s = minimal();
    s.joints.push_back(rev("a", "nosuch"));
    CHECK(expect(s, InvalidReference, "unknown body"));
  }
  {
    auto s = minimal();
    auto j = rev("world", "a");
    j.axis = Vec3(0, 0, 2);
    s.joints.push_back(j);
    CHECK(expect(s, NonUnitAxis, "unit length"));
  }
  {
    auto s = minimal();
    s.bodies[0].inertia = -1.0 * Mat3::identity();
    CHECK(expect(s, BadInertia, "positive definite"));
  }
  {
    auto s = minimal();
    s.bodies[0].inertia = Mat3::diagonal(Vec3(1.0, 0.1, 0.1));
    CHECK(expect(s, BadInertia, "triangle"));
  }
  {
    auto s = minimal();
    auto j = rev("world", "a");
    j.type = "spherical";
    j.has_limits = true;
    j.lower = -1;
    j.upper = 1;
    s.joints.push_back(j);
    CHECK(expect(s, UnsupportedOnJointType, "limits"));
  }
  {
    auto s = minimal();
    auto j = rev("world", "a");
    j.has_limits = true;
    j.lower = 1;
    j.upper = -1;
    s.joints.push_back(j);
    CHECK(expect(s, BadLimits, "limit"));
  }
  {
    auto s = minimal();
    s.joints.push_back(rev("a", "a"));
    CHECK(expect(s, InvalidReference, "differ"));
  }
  {
    auto s = minimal();
    s.bodies.push_back(s.bodies[0]);
    CHECK(expect(s, DuplicateName, "duplicated"));
  }
  {
    auto s = minimal();
    SceneGeom g;
    g.body = "a";
    g.shape = "plane";
    s.geoms.push_back(g);
    CHECK(expect(s, BadGeometry, "world"));
  }
  {
    auto s = minimal();
    SceneBody b2 = s.bodies[0];
    b2.name = "b";
    s.bodies.push_back(b2);
    SceneGeom box, sph;
    box.body = "a";
    box.shape = "box";
    box.half_extents = Vec3(0.1, 0.1, 0.1);
    sph.body = "b";
    sph.shape = "sphere";
    sph.radius = 0.1;
    s.geoms.push_back(box);
    s.geoms.push_back(sph);
    CHECK(expect(s, UnsupportedCollisionPair, "unsupported collision pair"));
  }
}
TEST(model_coord_pi6, "test_model.cpp:166 joint coordinate reads +pi/6") {
  SceneDescription s;
  s.bodies.push_back(body("a", 0.1));
  SceneJoint j;
  j.name = "j";
  j.type = "revolute";
  j.parent = "world";
  j.child = "a";
  s.joints.push_back(j);
  const MechanismModel m = build_model(s);
  std::vector<Pose> p(1);
  CHECK(std::abs(joint_coordinate(m, 0, p)) < 1e-12);
  p[0].orientation = axis_angle(M_PI / 6, Vec3(0, 0, 1));
  CHECK(std::abs(joint_coordinate(m, 0, p) - M_PI / 6) < 1e-12);
}
TEST(model_coord_random, "test_model.cpp:175 joint coordinate matches rotation-log oracle") {
  std::mt19937 rng(7);
  std::normal_distribution<double> n;
  for (int t = 0; t < 50; ++t) {
    SceneDescription s;
    s.bodies.push_back(body("a", 0.1));
    s.bodies.push_back(body("p", 0.1));
    SceneJoint j;
    j.name = "j";
    j.type = "revolute";
    j.parent = "p";
    j.child = "a";
    j.axis = normalized(Vec3(n(rng), n(rng), n(rng)));
    j.frame_in_parent.position = Vec3(n(rng), n(rng), n(rng));
    j.frame_in_parent.orientation = Quat(n(rng), n(rng), n(rng), n(rng)).normalized();
    j.frame_in_child.position = Vec3(n(rng), n(rng), n(rng));
    j.frame_in_child.orientation = Quat(n(rng), n(rng), n(rng), n(rng)).normalized();
    s.joints.push_back(j);
    const MechanismModel m = build_model(s);
    const double theta = std::uniform_real_distribution<double>(-3.0, 3.0)(rng);
    std::vector<Pose> poses(2);
    poses[1].position = Vec3(n(rng), n(rng), n(rng));
    poses[1].orientation = Quat(n(rng), n(rng), n(rng), n(rng)).normalized();
    const JointFrames fr = joint_world_frames(m, 0, poses);
    const Mat3 wc = fr.frame_parent * so3_exp(theta * m.joints[0].axis);
    poses[0].orientation = Quat::from_matrix(wc * m.joints[0].frame_in_child.rotation().transpose());
    poses[0].position = fr.anchor_parent - poses[0].orientation * m.joints[0].frame_in_child.position;
    const double coord = joint_coordinate(m, 0, poses);
    const JointFrames fr2 = joint_world_frames(m, 0, poses);
    const double orc = dot(so3_log(fr2.frame_parent.transpose() * fr2.frame_child), m.joints[0].axis);
    CHECK(std::abs(coord - orc) <= 1e-10 * (1 + std::abs(orc)));
  }
}
TEST(model_wrong_type, "test_model.cpp:213 joint coordinate rejects joints without a coordinate") {
  SceneDescription s;
  s.bodies.push_back(body("a", 0.1));
  SceneJoint j;
  j.name = "ball";
  j.type = "spherical";
  j.parent = "world";
  j.child = "a";
  s.joints.push_back(j);
  const MechanismModel m = build_model(s);
  bool threw = false;
  try {
    joint_coordinate(m, 0, std::vector<Pose>(1));
  } catch (const ModelError& e) {
    threw = e.code == WrongJointType;
  }
  CHECK(threw);
}

// ======================================================================= constraints
static MechanismModel single_joint_model(const std::string& type, bool to_world) {
  SceneDescription s;
  s.bodies.push_back(body("a"));
  if (!to_world) s.bodies.push_back(body("p"));
  SceneJoint j;
  j.name = "j";
  j.type = type;
  j.parent = to_world ? "world" : "p";
  j.child = "a";
  j.axis = normalized(Vec3(1, 2, 2));
  j.frame_in_parent.position = Vec3(0.1, -0.2, 0.3);
  j.frame_in_parent.orientation = random_quat(g_rng);
  j.frame_in_child.position = Vec3(-0.3, 0.1, 0.2);
  j.frame_in_child.orientation = random_quat(g_rng);
  s.joints.push_back(j);
  return build_model(s);
}
static std::vector<Pose> random_poses(const MechanismModel& m, double scale = 0.3) {
  std::vector<Pose> p(m.bodies.size());
  for (Pose& x : p) {
    x.position = random_vec(g_rng, scale);
    x.orientation = random_quat(g_rng);
  }
  return p;
}
TEST(cons_fd_all, "test_constraints.cpp:78 analytic Jacobians match finite differences, every joint type") {
  for (const char* type : {"fixed", "revolute", "prismatic", "spherical"})
    for (bool tw : {true, false}) {
      const MechanismModel m = single_joint_model(type, tw);
      for (int t = 0; t < 5; ++t) CHECK(constraint_jacobian_fd_check(m, random_poses(m), 1e-5) < 1e-6);
    }
}
TEST(cons_fd_fourbar, "test_constraints.cpp:91 four-bar Jacobian matches finite differences") {
  const MechanismModel m = load_model("fourbar");
  CHECK(constraint_jacobian_fd_check(m, initial_poses(m), 1e-5) < 1e-6);
  CHECK(constraint_jacobian_fd_check(m, random_poses(m, 0.5), 1e-5) < 1e-6);
}
TEST(cons_static, "test_constraints.cpp:98 static fourbar: zero residual and bias, 20/1/21 rows") {
  const MechanismModel m = load_model("fourbar");
  const ConstraintSet cs =
      assemble_constraints(m, initial_poses(m), std::vector<Twist>(3), {}, AssembleConfig{});
  CHECK(maxabs(cs.bilateral_f) < 1e-12);
  double mb = 0;
  for (int i = 0; i < cs.n_bilateral; ++i) mb = std::max(mb, std::abs(cs.bias[i]));
  CHECK(mb < 1e-10);
  CHECK(cs.n_bilateral == 20);
  CHECK(cs.n_dynamics == 1);
  CHECK(cs.n_rows == 21);
  REQUIRE(cs.cones.groups.size() == 1);
  CHECK(cs.cones.groups[0].kind == ConeKind::Bilateral);
  CHECK(cs.cones.groups[0].dim == 21);
}
TEST(cons_baumgarte, "test_constraints.cpp:112 Baumgarte bias of 1 mm displacement is -0.048") {
  SceneDescription s;
  s.bodies.push_back(body("a"));
  SceneJoint j;
  j.name = "weld";
  j.type = "fixed";
  j.parent = "world";
  j.child = "a";
  s.joints.push_back(j);
  const MechanismModel m = build_model(s);
  std::vector<Pose> p(1);
  p[0].position = Vec3(0.001, 0, 0);
  const ConstraintSet cs = assemble_constraints(m, p, std::vector<Twist>(1), {}, AssembleConfig{});
  CHECK(approx(cs.bilateral_f[0], 0.001));
  CHECK(approx(cs.bias[0], -0.048));
}
TEST(cons_pd, "test_constraints.cpp:132 implicit PD regularization 1/(dt(dt Kp + Kd)) = 362.264") {
  SceneDescription s;
  s.bodies.push_back(body("a"));
  SceneJoint j;
  j.name = "servo";
  j.type = "revolute";
  j.parent = "world";
  j.child = "a";
  j.kp = 15.0;
  j.kd = 0.6;
  j.has_target = true;
  j.target = 0.3;
  j.target_rate = 0.25;
  s.joints.push_back(j);
  const MechanismModel m = build_model(s);
  const ConstraintSet cs = assemble_constraints(m, initial_poses(m), std::vector<Twist>(1), {}, AssembleConfig{});
  const double expected = 1.0 / ((1.0 / 240.0) * ((1.0 / 240.0) * 15.0 + 0.6));
  CHECK(std::abs(cs.reg[cs.n_bilateral] - expected) <= 1e-12 * expected);
  CHECK(std::abs(expected - 362.264) <= 1e-4 * 362.264);
  const double bias = (15.0 * 0.3 + 0.6 * 0.25) / ((1.0 / 240.0) * 15.0 + 0.6);
  CHECK(std::abs(cs.bias[cs.n_bilateral] - bias) <= 1e-12 * bias);
}
TEST(cons_arm_damp, "test_constraints.cpp:159 armature and damping rows") {
  SceneDescription s;
  s.bodies.push_back(body("a"));
  SceneJoint j;
  j.name = "j";
  j.type = "revolute";
  j.parent = "world";
  j.child = "a";
  j.armature = 0.02;
  j.damping = 0.5;
  s.joints.push_back(j);
  const MechanismModel m = build_model(s);
  std::vector<Twist> tw(1);
  tw[0].angular = Vec3(0, 0, 1.5);
  AssembleConfig cfg;
  const ConstraintSet cs = assemble_constraints(m, initial_poses(m), tw, {}, cfg);
  REQUIRE(cs.n_dynamics == 2);
  CHECK(approx(cs.reg[cs.n_bilateral], 50.0));
  CHECK(approx(cs.bias[cs.n_bilateral], 1.5));
  CHECK(approx(cs.reg[cs.n_bilateral + 1], 1.0 / (cfg.dt * 0.5)));
  CHECK(approx(cs.bias[cs.n_bilateral + 1], 0.0));
}
TEST(cons_limits, "test_constraints.cpp:185 limit rows activate inside the margin") {
  SceneDescription s;
  s.bodies.push_back(body("a"));
  SceneJoint j;
  j.name = "j";
  j.type = "revolute";
  j.parent = "world";
  j.child = "a";
  j.has_limits = true;
  j.lower = -0.1;
  j.upper = 0.4;
  s.joints.push_back(j);
  const MechanismModel m = build_model(s);
  auto at = [&](double a) {
    std::vector<Pose> p(1);
    p[0].orientation = axis_angle(a, Vec3(0, 0, 1));
    return assemble_constraints(m, p, std::vector<Twist>(1), {}, AssembleConfig{});
  };
  CHECK(at(0.1).n_limits == 0);
  {
    const ConstraintSet cs = at(0.395);
    REQUIRE(cs.n_limits == 1);
    CHECK(cs.limit_keys[0] == std::make_pair(0, 1));
    CHECK(approx(cs.limit_gap[0], 0.005));
    CHECK(approx(cs.bias[cs.first_limit_row()], 0.0));
    CHECK(approx(cs.rows[cs.first_limit_row()].block_a[5], -1.0));
    CHECK(cs.cones.groups.back().kind == ConeKind::Nonnegative);
  }
  {
    const ConstraintSet cs = at(0.45);
    REQUIRE(cs.n_limits == 1);
    CHECK(approx(cs.limit_gap[0], -0.05));
    CHECK(approx(cs.bias[cs.first_limit_row()], 0.2 * 240.0 * 0.05));
  }
  {
    const ConstraintSet cs = at(-0.095);
    REQUIRE(cs.n_limits == 1);
    CHECK(cs.limit_keys[0] == std::make_pair(0, 0));
    CHECK(approx(cs.rows[cs.first_limit_row()].block_a[5], 1.0));
  }
}
TEST(cons_contact, "test_constraints.cpp:230 contact rows: frame, restitution threshold, Baumgarte") {
  SceneDescription s;
  SceneBody ball = body("ball");
  ball.pose.position = Vec3(0, 0, 0.09);
  s.bodies.push_back(ball);
  SceneGeom gs, gp;
  gs.body = "ball";
  gs.shape = "sphere";
  gs.radius = 0.1;
  gs.mu = 0.64;
  gs.restitution = 0.5;
  gp.body = "world";
  gp.shape = "plane";
  gp.mu = 0.25;
  gp.restitution = 0.5;
  s.geoms.push_back(gs);
  s.geoms.push_back(gp);
  const MechanismModel m = build_model(s);
  const auto poses = initial_poses(m);
  const auto contacts = collide(m, poses, 0.01);
  REQUIRE(contacts.size() == 1);
  CHECK(approx(contacts[0].mu, 0.4));
  {
    std::vector<Twist> tw(1);
    tw[0].linear = Vec3(0, 0, -0.05);
    const ConstraintSet cs = assemble_constraints(m, poses, tw, contacts, AssembleConfig{});
    REQUIRE(cs.n_contact_rows == 3);
    const int r = cs.first_contact_row();
    CHECK(approx(cs.rows[r].block_a[2], 1.0));
    CHECK(approx(cs.bias[r], 0.2 * 240.0 * 0.01));
    CHECK(approx(cs.bias[r + 1], 0.0));
    CHECK(cs.cones.groups.back().kind == ConeKind::SecondOrder);
    CHECK(approx(cs.cones.groups.back().mu, 0.4));
  }
  {
    std::vector<Twist> tw(1);
    tw[0].linear = Vec3(0, 0, -1.0);
    const ConstraintSet cs = assemble_constraints(m, poses, tw, contacts, AssembleConfig{});
    CHECK(approx(cs.bias[cs.first_contact_row()], 0.2 * 240.0 * 0.01 + 0.5));
  }
}
TEST(cons_invariance, "test_constraints.cpp:292 bilateral residual invariant under a rigid transform") {
  const LoadedScene base = load("fourbar");
  const MechanismModel m0 = build_model(base.scene);
  for (int t = 0; t < 10; ++t) {
    const Quat rot = random_quat(g_rng);
    const Vec3 trans = random_vec(g_rng, 2.0);
    SceneDescription moved = base.scene;
    for (SceneJoint& j : moved.joints)
      if (j.parent == "world") {
        j.frame_in_parent.position = trans + rot * j.frame_in_parent.position;
        j.frame_in_parent.orientation = rot * j.frame_in_parent.orientation;
      }
    for (SceneBody& b : moved.bodies) {
      b.pose.position = trans + rot * b.pose.position;
      b.pose.orientation = rot * b.pose.orientation;
    }
    const MechanismModel m1 = build_model(moved);
    const auto p0 = random_poses(m0, 0.3);
    auto p1 = p0;
    for (Pose& p : p1) {
      p.position = trans + rot * p.position;
      p.orientation = rot * p.orientation;
    }
    const Vec f0 = build_bilateral(m0, p0).f, f1 = build_bilateral(m1, p1).f;
    double e = 0;
    for (size_t i = 0; i < f0.size(); ++i) e = std::max(e, std::abs(f0[i] - f1[i]));
    CHECK(e < 1e-10);
  }
}
TEST(cons_ju_dfdt, "test_constraints.cpp:323 J u equals df/dt along a twist field") {
  const MechanismModel m = load_model("fourbar");
  const auto poses = random_poses(m, 0.3);
  const ConstraintSet cs = assemble_constraints(m, poses, std::vector<Twist>(3), {}, AssembleConfig{});
  std::mt19937 local(5);
  std::normal_distribution<double> n;
  Vec u(6 * m.n_bodies());
  for (double& x : u) x = n(local);
  const double h = 1e-6;
  auto flow = [&](double e) {
    std::vector<Pose> mv = poses;
    for (int b = 0; b < m.n_bodies(); ++b) {
      mv[b].position = mv[b].position + e * Vec3(u[6 * b], u[6 * b + 1], u[6 * b + 2]);
      mv[b].orientation = quat_exp((0.5 * e) * Vec3(u[6 * b + 3], u[6 * b + 4], u[6 * b + 5])) * mv[b].orientation;
    }
    return build_bilateral(m, mv).f;
  };
  const Vec fp = flow(h), fm = flow(-h), ju = cs.apply_jacobian(u);
  double e = 0;
  for (int i = 0; i < cs.n_bilateral; ++i) e = std::max(e, std::abs((fp[i] - fm[i]) / (2 * h) - ju[i]));
  CHECK(e < 1e-6);
}

// ======================================================================= delassus
static DenseMatrix naive_delassus(const ConstraintSet& cs, const std::vector<BodyInertiaWorld>& in) {
  DenseMatrix d;
  d.n = cs.n_rows;
  d.a.assign((size_t)d.n * d.n, 0.0);
  for (int i = 0; i < cs.n_rows; ++i)
    for (int j = 0; j < cs.n_rows; ++j) {
      double s = 0;
      for (int side_i = 0; side_i < 2; ++side_i)
        for (int side_j = 0; side_j < 2; ++side_j) {
          const int bi = side_i ? cs.rows[i].body_b : cs.rows[i].body_a;
          const int bj = side_j ? cs.rows[j].body_b : cs.rows[j].body_a;
          if (bi < 0 || bi != bj) continue;
          const Row6& gi = side_i ? cs.rows[i].block_b : cs.rows[i].block_a;
          const Row6& gj = side_j ? cs.rows[j].block_b : cs.rows[j].block_a;
          for (int k = 0; k < 3; ++k) s += gi[k] * in[bi].inv_mass * gj[k];
          for (int k = 0; k < 3; ++k)
            for (int l = 0; l < 3; ++l) s += gi[3 + k] * in[bi].inv_inertia_world(k, l) * gj[3 + l];
        }
      d(i, j) = s + (i == j ? cs.reg[i] : 0.0);
    }
  return d;
}
TEST(del_d00, "test_delassus.cpp:63 single row on one body: D entry is the inverse mass") {
  SceneDescription s;
  SceneBody b = body("a", 0.1);
  b.mass = 4.0;
  s.bodies.push_back(b);
  const MechanismModel m = build_model(s);
  ConstraintSet cs;
  cs.n_rows = 1;
  cs.n_bodies = 1;
  JacobianRow row;
  row.body_a = 0;
  row.block_a[0] = 1;
  cs.rows.push_back(row);
  cs.bias = Vec(1, 0.0);
  cs.reg = Vec(1, 0.0);
  const DenseDelassus dd = assemble_dense(cs, world_inertias(m, initial_poses(m)), 0.0);
  CHECK(approx(dd.matrix(0, 0), 0.25));
}
TEST(del_blockwise, "test_delassus.cpp:111 blockwise assembly matches the naive triple product") {
  const MechanismModel m = load_model("fourbar");
  const auto poses = initial_poses(m);
  const ConstraintSet cs = assemble_constraints(m, poses, std::vector<Twist>(3), {}, AssembleConfig{});
  const auto in = world_inertias(m, poses);
  const DenseDelassus dd = assemble_dense(cs, in, 1e-3);
  DenseMatrix ex = naive_delassus(cs, in);
  double e = 0;
  for (int i = 0; i < cs.n_rows; ++i)
    for (int j = 0; j < cs.n_rows; ++j)
      e = std::max(e, std::abs(dd.matrix(i, j) - (ex(i, j) + (i == j ? 1e-3 : 0.0))));
  CHECK(e < 1e-10);
  CHECK(dd.factorized);
}
TEST(del_solve, "test_delassus.cpp:125 dense solve: identity and random SPD residual") {
  std::mt19937 rng(99);
  std::uniform_real_distribution<double> u(-1, 1);
  DenseDelassus dd;
  dd.matrix.n = 30;
  dd.matrix.a.assign(900, 0.0);
  std::vector<double> b(900);
  for (double& x : b) x = u(rng);
  for (int i = 0; i < 30; ++i)
    for (int j = 0; j < 30; ++j) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int k = 0; k < 30; ++k) s += b[k * 30 + i] * b[k * 30 + j];
      dd.matrix(i, j) = s;
    }
  REQUIRE(dd.factorize());
  Vec rhs(30);
  for (double& x : rhs) x = u(rng);
  const Vec x = dd.solve(rhs);
  double e = 0;
  for (int i = 0; i < 30; ++i) {
    double s = 0;
    for (int j = 0; j < 30; ++j) s += dd.matrix(i, j) * x[j];
    e = std::max(e, std::abs(s - rhs[i]));
  }
  CHECK(e < 1e-10);
}
TEST(del_probes, "test_delassus.cpp:145 baked operator reproduces the preconditioned dense matrix") {
  const MechanismModel m = load_model("fourbar");
  const auto poses = initial_poses(m);
  const ConstraintSet cs = assemble_constraints(m, poses, std::vector<Twist>(3), {}, AssembleConfig{});
  const auto in = world_inertias(m, poses);
  const double er = 1.0 + 1e-6;
  const Preconditioner p = jacobi_preconditioner(cs, in);
  const MatrixFreeDelassus op = bake_jacobian(cs, in, p, er);
  const DenseDelassus dd = assemble_dense(cs, in, er, &p);
  double e = 0;
  for (int k = 0; k < cs.n_rows; ++k) {
    Vec unit(cs.n_rows, 0.0);
    unit[k] = 1.0;
    const Vec col = op.apply(unit);
    for (int i = 0; i < cs.n_rows; ++i) e = std::max(e, std::abs(col[i] - dd.matrix(i, k)));
  }
  CHECK(e < 1e-9);
  const MatrixFreeDelassus opi = bake_jacobian(cs, in, Preconditioner::identity(cs.n_rows), er);
  DenseMatrix ex = naive_delassus(cs, in);
  std::mt19937 rng(1);
  std::uniform_real_distribution<double> u(-1, 1);
  for (int t = 0; t < 10; ++t) {
    Vec v(cs.n_rows);
    for (double& x : v) x = u(rng);
    const Vec o = opi.apply(v);
    double err = 0;
    for (int i = 0; i < cs.n_rows; ++i) {
      double s = er * v[i];
      for (int j = 0; j < cs.n_rows; ++j) s += ex(i, j) * v[j];
      err = std::max(err, std::abs(o[i] - s));
    }
    CHECK(err < 1e-9);
  }
}
static MatrixFreeDelassus diag_op(const Vec& d) {
  MatrixFreeDelassus op;
  op.n_bodies = 1;
  op.rows.resize(d.size());
  op.diag_add = d;
  return op;
}
TEST(del_cr_exact, "test_delassus.cpp:192 cr_solve returns an exact warm start unchanged") {
  const MatrixFreeDelassus op = diag_op(Vec(4, 2.0));
  const Vec rhs = {0.3, -0.7, 0.11, 0.5};
  Vec x(4);
  for (int i = 0; i < 4; ++i) x[i] = rhs[i] / 2.0;
  const Vec x0 = x;
  const CrResult r = cr_solve(op, rhs, x, 10);
  CHECK(x == x0);
  CHECK(r.breakdown);
  CHECK(r.iterations == 0);
}
TEST(del_cr_one, "test_delassus.cpp:205 cr_solve converges in one iteration on a uniform diagonal") {
  const MatrixFreeDelassus op = diag_op(Vec(6, 3.0));
  const Vec rhs = {0.3, -0.7, 0.11, 0.5, 0.9, -0.2};
  Vec x(6, 0.0);
  cr_solve(op, rhs, x, 1);
  for (int i = 0; i < 6; ++i) CHECK(std::abs(x[i] - rhs[i] / 3.0) < 1e-14);
}
TEST(del_cr_distinct, "test_delassus.cpp:217 cr_solve finishes in n_distinct iterations") {
  const MatrixFreeDelassus op = diag_op({1, 1, 2, 2, 2, 5, 5, 1});
  const Vec rhs = {0.3, -0.7, 0.11, 0.5, 0.9, -0.2, 0.4, 0.8};
  Vec x(8, 0.0);
  cr_solve(op, rhs, x, 3);
  const Vec ax = op.apply(x);
  double e = 0;
  for (int i = 0; i < 8; ++i) e = std::max(e, std::abs(ax[i] - rhs[i]));
  CHECK(e < 1e-10);
}
TEST(del_cr_monotone, "test_delassus.cpp:230 cr residual norm is non-increasing (serial chain)") {
  const MechanismModel m = load_model("serial_chain_10");
  const auto poses = initial_poses(m);
  const ConstraintSet cs = assemble_constraints(m, poses, std::vector<Twist>(10), {}, AssembleConfig{});
  const auto in = world_inertias(m, poses);
  const MatrixFreeDelassus op = bake_jacobian(cs, in, jacobi_preconditioner(cs, in), 1.0);
  std::mt19937 rng(2);
  std::uniform_real_distribution<double> u(-1, 1);
  Vec rhs(cs.n_rows), x(cs.n_rows, 0.0);
  for (double& v : rhs) v = u(rng);
  std::vector<double> h;
  cr_solve(op, rhs, x, 40, &h);
  for (size_t k = 1; k < h.size(); ++k) CHECK(h[k] <= h[k - 1] + 1e-12);
}
TEST(del_jacobi, "test_delassus.cpp:247 jacobi preconditioner basics (P=1, P=0.5)") {
  for (double mass : {1.0, 0.25}) {
    SceneDescription s;
    SceneBody b = body("a", mass == 1.0 ? 1.0 : 0.01);
    b.mass = mass;
    s.bodies.push_back(b);
    const MechanismModel m = build_model(s);
    ConstraintSet cs;
    cs.n_rows = 1;
    cs.n_bodies = 1;
    JacobianRow row;
    row.body_a = 0;
    row.block_a[0] = 1;
    cs.rows.push_back(row);
    cs.reg = Vec(1, 0.0);
    cs.bias = Vec(1, 0.0);
    const Preconditioner p = jacobi_preconditioner(cs, world_inertias(m, initial_poses(m)));
    CHECK(approx(p.scale[0], mass == 1.0 ? 1.0 : 0.5));
  }
}
TEST(del_unit_diag, "test_delassus.cpp:294 preconditioned dense matrix has unit diagonal") {
  const MechanismModel m = load_model("fourbar");
  const auto poses = initial_poses(m);
  const ConstraintSet cs = assemble_constraints(m, poses, std::vector<Twist>(3), {}, AssembleConfig{});
  const auto in = world_inertias(m, poses);
  const Preconditioner p = jacobi_preconditioner(cs, in);
  const DenseDelassus dd = assemble_dense(cs, in, 0.0, &p);
  for (int r = 0; r < cs.n_rows; ++r) CHECK(std::abs(dd.matrix(r, r) - 1.0) <= 1e-12 * 2);
}
TEST(del_contact_scale, "test_delassus.cpp:307 contact groups share the normal-row scale") {
  SceneDescription s;
  SceneBody ball = body("ball", 0.004);
  ball.pose.position = Vec3(0, 0, 0.1);
  s.bodies.push_back(ball);
  SceneGeom gs, gp;
  gs.body = "ball";
  gs.shape = "sphere";
  gs.radius = 0.1;
  gs.mu = 0.5;
  gp.body = "world";
  gp.shape = "plane";
  gp.mu = 0.5;
  s.geoms.push_back(gs);
  s.geoms.push_back(gp);
  const MechanismModel m = build_model(s);
  const auto poses = initial_poses(m);
  const auto contacts = collide(m, poses, 0.01);
  const ConstraintSet cs = assemble_constraints(m, poses, std::vector<Twist>(1), contacts, AssembleConfig{});
  REQUIRE(cs.n_contact_rows == 3);
  const Preconditioner p = jacobi_preconditioner(cs, world_inertias(m, poses));
  const int r = cs.first_contact_row();
  CHECK(p.scale[r + 1] == p.scale[r]);
  CHECK(p.scale[r + 2] == p.scale[r]);
}
TEST(del_dense_cr, "test_delassus.cpp:321 dense and matrix-free backends agree, budget 200") {
  const MechanismModel m = load_model("fourbar");
  const auto poses = initial_poses(m);
  const ConstraintSet cs = assemble_constraints(m, poses, std::vector<Twist>(3), {}, AssembleConfig{});
  const auto in = world_inertias(m, poses);
  const DenseDelassus dd = assemble_dense(cs, in, 1.0);
  const MatrixFreeDelassus op = bake_jacobian(cs, in, Preconditioner::identity(cs.n_rows), 1.0);
  std::mt19937 rng(8);
  std::uniform_real_distribution<double> u(-1, 1);
  for (int t = 0; t < 5; ++t) {
    Vec rhs(cs.n_rows), xi(cs.n_rows, 0.0);
    for (double& v : rhs) v = u(rng);
    const Vec xd = dd.solve(rhs);
    cr_solve(op, rhs, xi, 200);
    double e = 0;
    for (int i = 0; i < cs.n_rows; ++i) e = std::max(e, std::abs(xd[i] - xi[i]));
    CHECK(e < 1e-6 * std::max(1.0, maxabs(xd)));
  }
}
TEST(del_spd_random, "test_delassus.cpp:339 D stays SPD whenever eta+rho > 0 (1000 random systems)") {
  std::mt19937 rng(77);
  std::normal_distribution<double> n;
  int ok = 0;
  for (int t = 0; t < 1000; ++t) {
    const int nb = 1 + (int)(rng() % 3);
    SceneDescription s;
    for (int b = 0; b < nb; ++b) {
      SceneBody bd;
      bd.name = "b" + std::to_string(b);
      bd.mass = 0.1 + std::abs(n(rng));
      bd.inertia = (0.01 + std::abs(n(rng)) * 0.1) * Mat3::identity();
      s.bodies.push_back(bd);
    }
    const MechanismModel m = build_model(s);
    std::vector<Pose> poses(nb);
    for (Pose& p : poses) {
      p.position = Vec3(n(rng), n(rng), n(rng));
      p.orientation = Quat(n(rng), n(rng), n(rng), n(rng)).normalized();
    }
    const int nr = 1 + (int)(rng() % 12);
    ConstraintSet cs;
    cs.n_rows = nr;
    cs.n_bodies = nb;
    cs.reg = Vec(nr, 0.0);
    cs.bias = Vec(nr, 0.0);
    for (int r = 0; r < nr; ++r) {
      JacobianRow row;
      row.body_a = (int)(rng() % nb);
      for (int k = 0; k < 6; ++k) row.block_a[k] = n(rng);
      if (nb > 1 && (rng() % 2) == 0) {
        row.body_b = (row.body_a + 1) % nb;
        for (int k = 0; k < 6; ++k) row.block_b[k] = n(rng);
      }
      if ((rng() % 3) == 0) cs.reg[r] = std::abs(n(rng));
      cs.rows.push_back(row);
    }
    if (assemble_dense(cs, world_inertias(m, poses), 1e-6).factorized) ++ok;
  }
  CHECK(ok == 1000);
}

// ======================================================================= padmm
struct ChainProblem {
  ConstraintSet cs;
  std::vector<BodyInertiaWorld> in;
  Vec v_f;
};
static ChainProblem chain_problem() {  // test_padmm.cpp:35-55
  const MechanismModel m = load_model("serial_chain_10");
  ChainProblem p;
  const auto poses = initial_poses(m);
  p.cs = assemble_constraints(m, poses, std::vector<Twist>(m.n_bodies()), {}, AssembleConfig{});
  p.in = world_inertias(m, poses);
  Vec uf(6 * m.n_bodies(), 0.0);
  for (int b = 0; b < m.n_bodies(); ++b) {
    const Vec3 h = m.bodies[b].inertia.mass * m.gravity;
    const Vec3 v = (1.0 / m.bodies[b].inertia.mass) * ((1.0 / 240.0) * h);
    uf[6 * b] = v.x;
    uf[6 * b + 1] = v.y;
    uf[6 * b + 2] = v.z;
  }
  const Vec ju = p.cs.apply_jacobian(uf);
  p.v_f.resize(ju.size());
  for (size_t i = 0; i < ju.size(); ++i) p.v_f[i] = ju[i] - p.cs.bias[i];
  return p;
}
static Vec scaled(const Vec& s, const Vec& v) {
  Vec o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = s[i] * v[i];
  return o;
}
TEST(pad_cones, "test_padmm.cpp:59-106 cone projection: identity, clamp, interior/polar, mu=0") {
  ConeProduct bil;
  bil.n_rows = 4;
  bil.groups.push_back({ConeKind::Bilateral, 0, 4, 0.0});
  const Vec w = {0.3, -0.4, 1.2, -7.0};
  CHECK(project_cone(w, bil) == w);
  ConeProduct nn;
  nn.n_rows = 3;
  for (int k = 0; k < 3; ++k) nn.groups.push_back({ConeKind::Nonnegative, k, 1, 0.0});
  const Vec y = project_cone({-1.0, 0.5, -0.2}, nn);
  CHECK(y[0] == 0.0 && y[1] == 0.5 && y[2] == 0.0);
  CHECK(project_cone({1.0, 0.5, 0.0}, single_soc(1.0)) == Vec({1.0, 0.5, 0.0}));
  const Vec p = project_cone({-2.0, 1.0, 0.0}, single_soc(1.0));
  CHECK(p[0] == 0.0 && p[1] == 0.0 && p[2] == 0.0);
  const Vec q = project_cone({2.0, 0.7, -0.4}, single_soc(0.0));
  CHECK(approx(q[0], 2.0) && q[1] == 0.0 && q[2] == 0.0);
}
TEST(pad_cone_oracle, "test_padmm.cpp:87 + acceptance #12(a): SOC projection vs golden-section oracle") {
  std::mt19937 rng(20240813);
  std::normal_distribution<double> n(0.0, 2.0);
  std::uniform_real_distribution<double> mu_d(0.0, 1.5);
  double worst = 0;
  for (int t = 0; t < 10000; ++t) {
    const double mu = mu_d(rng);
    const Vec3 w(n(rng), n(rng), n(rng));
    const Vec y = project_cone({w.x, w.y, w.z}, single_soc(mu));
    const Vec3 e = cone_project_oracle(w, mu);
    for (int k = 0; k < 3; ++k) worst = std::max(worst, std::abs(y[k] - e[k]));
  }
  CHECK(worst < 1e-6);
}
TEST(pad_desaxce, "test_padmm.cpp:108 De Saxce shift examples") {
  ConeProduct bil;
  bil.n_rows = 2;
  bil.groups.push_back({ConeKind::Bilateral, 0, 2, 0.0});
  CHECK(maxabs(desaxce_shift({0.4, -0.3}, bil)) == 0.0);
  CHECK(maxabs(desaxce_shift({-1.0, 0.0, 0.0}, single_soc(0.7))) == 0.0);
  const Vec s = desaxce_shift({-1.0, 3.0, 4.0}, single_soc(0.5));
  CHECK(approx(s[0], 2.5) && s[1] == 0.0 && s[2] == 0.0);
}
TEST(pad_nesterov, "test_padmm.cpp:130 + acceptance #12(c): Nesterov sequence exact") {
  CHECK(approx(nesterov_next_coefficient(1.0), 0.5 * (1.0 + std::sqrt(5.0))));
  double a = 1.0;
  for (int i = 0; i < 20; ++i) {
    const double ex = (1.0 + std::sqrt(1.0 + 4.0 * a * a)) / 2.0;
    a = nesterov_next_coefficient(a);
    CHECK(a == ex);
  }
}
TEST(pad_nesterov_update, "test_padmm.cpp:140 nesterov_update extrapolates / no-ops / restarts") {
  PadmmState st;
  st.x = st.y = st.z = Vec(2, 1.0);
  st.y_prev = st.z_prev = Vec(2, 0.0);
  st.a = 2.0;
  nesterov_update(st, false);
  const double an = nesterov_next_coefficient(2.0);
  CHECK(approx(st.y_hat[0], 1.0 + (2.0 - 1.0) / an));
  CHECK(approx(st.a, an));
  PadmmState same;
  same.y = same.y_prev = Vec(3, 0.7);
  same.z = same.z_prev = Vec(3, -0.1);
  same.a = 3.0;
  nesterov_update(same, false);
  CHECK(same.y_hat == same.y);
  PadmmState rs;
  rs.y = rs.z = Vec(1, 1.0);
  rs.y_prev = rs.z_prev = Vec(1, 0.0);
  rs.a = 5.0;
  nesterov_update(rs, true);
  CHECK(rs.a == 1.0 && rs.y_hat == rs.y && rs.restarts == 1);
}
TEST(pad_residuals, "test_padmm.cpp:170 residual triple definitions") {
  ConeProduct c;
  c.n_rows = 2;
  c.groups.push_back({ConeKind::Nonnegative, 0, 1, 0.0});
  c.groups.push_back({ConeKind::Nonnegative, 1, 1, 0.0});
  double rp, rd, rc;
  padmm_residuals({1.0, 0.0}, {1.0, 0.0}, {1.0, 0.0}, {0.0, 2.0}, 1.0, c, rp, rd, rc);
  CHECK(rp == 0.0 && rd == 0.0 && rc == 0.0);
  padmm_residuals({1.1, 0.0}, {1.0, 0.0}, {1.0, 0.0}, {0.0, 2.0}, 1.0, c, rp, rd, rc);
  CHECK(approx(rp, 0.1));
  ConeProduct b;
  b.n_rows = 2;
  b.groups.push_back({ConeKind::Bilateral, 0, 2, 0.0});
  padmm_residuals({3.0, 1.0}, {3.0, 1.0}, {3.0, 1.0}, {2.0, 2.0}, 1.0, b, rp, rd, rc);
  CHECK(rc == 0.0);
}
TEST(pad_zero_vf, "test_padmm.cpp:201 zero free velocity converges in one iteration") {
  ChainProblem p = chain_problem();
  PadmmConfig cfg;
  const DelassusBackend be = build_backend(p.cs, p.in, Preconditioner::identity(p.cs.n_rows),
                                           cfg.eta + cfg.rho, BackendChoice::Dense, 9);
  const PadmmResult r = padmm_solve(be, Vec(p.cs.n_rows, 0.0), p.cs.cones, {}, cfg);
  CHECK(maxabs(r.lambda) == 0.0);
  CHECK(r.diagnostics.iterations == 1);
  CHECK(r.diagnostics.converged);
}
TEST(pad_bilateral, "test_padmm.cpp:214 bilateral-only system solves D lambda = -v_f") {
  ChainProblem p = chain_problem();
  const Preconditioner pc = jacobi_preconditioner(p.cs, p.in);
  PadmmConfig cfg;
  cfg.eps = 1e-10;
  cfg.max_iters = 2000;
  const DelassusBackend be = build_backend(p.cs, p.in, pc, cfg.eta + cfg.rho, BackendChoice::Dense, 9);
  const PadmmResult r = padmm_solve(be, scaled(pc.scale, p.v_f), p.cs.cones, {}, cfg);
  REQUIRE(r.diagnostics.converged);
  const Vec lam = scaled(pc.scale, r.lambda);
  const DenseDelassus dd = assemble_dense(p.cs, p.in, 0.0);
  Vec mv(p.v_f.size());
  for (size_t i = 0; i < mv.size(); ++i) mv[i] = -p.v_f[i];
  const Vec ex = dd.solve(mv);
  double e = 0;
  for (size_t i = 0; i < ex.size(); ++i) e = std::max(e, std::abs(lam[i] - ex[i]));
  CHECK(e / std::max(1.0, maxabs(ex)) < 1e-6);
}
TEST(pad_invariance, "test_padmm.cpp:234 solution invariant in eta and rho") {
  ChainProblem p = chain_problem();
  const Preconditioner pc = jacobi_preconditioner(p.cs, p.in);
  const Vec vfs = scaled(pc.scale, p.v_f);
  std::vector<Vec> sols;
  for (auto [eta, rho] : std::vector<std::pair<double, double>>{{1e-5, 0.1}, {1e-5, 1.0}, {1e-3, 1.0}}) {
    PadmmConfig cfg;
    cfg.eta = eta;
    cfg.rho = rho;
    cfg.eps = 1e-9;
    cfg.max_iters = 5000;
    const DelassusBackend be = build_backend(p.cs, p.in, pc, eta + rho, BackendChoice::Dense, 9);
    const PadmmResult r = padmm_solve(be, vfs, p.cs.cones, {}, cfg);
    REQUIRE(r.diagnostics.converged);
    sols.push_back(scaled(pc.scale, r.lambda));
  }
  const double sc = std::max(1.0, maxabs(sols[0]));
  for (int k = 1; k < 3; ++k) {
    double e = 0;
    for (size_t i = 0; i < sols[0].size(); ++i) e = std::max(e, std::abs(sols[0][i] - sols[k][i]));
    CHECK(e / sc < 1e-5);
  }
}
TEST(pad_monotone, "test_padmm.cpp:257 without acceleration the combined residual is non-increasing") {
  ChainProblem p = chain_problem();
  const Preconditioner pc = jacobi_preconditioner(p.cs, p.in);
  PadmmConfig cfg;
  cfg.acceleration = false;
  cfg.restart = false;
  cfg.eps = 1e-12;
  cfg.max_iters = 400;
  const DelassusBackend be = build_backend(p.cs, p.in, pc, cfg.eta + cfg.rho, BackendChoice::Dense, 9);
  std::vector<double> h;
  padmm_solve(be, scaled(pc.scale, p.v_f), p.cs.cones, {}, cfg, &h);
  REQUIRE(h.size() > 2);
  for (size_t k = 1; k < h.size(); ++k) CHECK(h[k] <= h[k - 1] + 1e-12);
}
TEST(pad_fixed, "test_padmm.cpp:275 fixed-iteration mode runs exactly max_iters") {
  ChainProblem p = chain_problem();
  const Preconditioner pc = jacobi_preconditioner(p.cs, p.in);
  PadmmConfig cfg;
  cfg.fixed_iteration_mode = true;
  cfg.max_iters = 17;
  const DelassusBackend be = build_backend(p.cs, p.in, pc, cfg.eta + cfg.rho, BackendChoice::Dense, 9);
  std::vector<double> h;
  const PadmmResult r = padmm_solve(be, scaled(pc.scale, p.v_f), p.cs.cones, {}, cfg, &h);
  CHECK(r.diagnostics.iterations == 17);
  CHECK(h.size() == 17);
  const PadmmResult z = padmm_solve(be, Vec(p.cs.n_rows, 0.0), p.cs.cones, {}, cfg);
  CHECK(z.diagnostics.iterations == 17);
  CHECK(z.diagnostics.converged);
}
TEST(pad_y_in_cone, "test_padmm.cpp:295 y stays inside the cone product") {
  ConeProduct c;
  c.n_rows = 7;
  c.groups.push_back({ConeKind::Bilateral, 0, 3, 0.0});
  c.groups.push_back({ConeKind::Nonnegative, 3, 1, 0.0});
  c.groups.push_back({ConeKind::SecondOrder, 4, 3, 0.8});
  std::mt19937 rng(4242);
  std::normal_distribution<double> n;
  for (int t = 0; t < 20; ++t) {
    Vec w(7);
    for (double& x : w) x = n(rng);
    const Vec y = project_cone(w, c);
    CHECK(y[3] >= 0.0);
    CHECK(std::hypot(y[5], y[6]) <= 0.8 * y[4] + 1e-15);
  }
}

// ======================================================================= stepper
TEST(step_free_forces, "test_stepper.cpp:38 free_forces: gravity, aligned spin, gyroscopic") {
  SceneDescription s;
  SceneBody b = body("a");
  b.mass = 2.0;
  b.inertia = Mat3::diagonal(Vec3(1.0, 2.0, 3.0));
  s.bodies.push_back(b);
  const MechanismModel m = build_model(s);
  const std::vector<Pose> poses(1);
  std::vector<Twist> tw(1);
  Vec h = free_forces(m, poses, tw);
  CHECK(h[0] == 0.0 && h[1] == 0.0 && h[2] == 2.0 * -9.81 && h[3] == 0.0 && h[4] == 0.0 && h[5] == 0.0);
  tw[0].angular = Vec3(0, 5.0, 0);
  h = free_forces(m, poses, tw);
  CHECK(std::abs(h[3]) + std::abs(h[4]) + std::abs(h[5]) < 1e-14);
  tw[0].angular = Vec3(1, 2, 3);
  h = free_forces(m, poses, tw);
  CHECK(norm(Vec3(h[3], h[4], h[5]) - Vec3(-6.0, 6.0, -2.0)) < 1e-13);
}
TEST(step_freefall, "test_stepper.cpp:112 + acceptance #7: free fall closed form, bitwise deterministic") {
  const MechanismModel m = load_model("freefall");
  StepConfig cfg;
  WorldState s1 = initial_state(m), s2 = initial_state(m);
  const int n = 240;
  for (int k = 0; k < n; ++k) {
    step(m, s1, cfg);
    step(m, s2, cfg);
  }
  CHECK(states_bitwise_equal(s1, s2));
  const double g = 9.81, dt = cfg.dt;
  CHECK(std::abs(s1.twists[0].linear.z + g * n * dt) < 1e-9);
  CHECK(std::abs(s1.poses[0].position.z + g * dt * dt * (n * (n + 1)) / 2.0) < 1e-9);
}
TEST(step_pendulum, "test_stepper.cpp:128 pendulum: drift, energy, small-angle period") {
  const MechanismModel m = load_model("pendulum");
  StepConfig cfg;
  WorldState st = initial_state(m);
  const double L = 1.0, mass = 1.0, iyy = 0.02, g = 9.81, th0 = 0.05;
  const double e0 = kinetic_energy(m, st) + potential_energy(m, st);
  const double e_amp = mass * g * L * (1.0 - std::cos(th0));
  double max_f = 0, max_e = 0, max_kkt = 0, max_v = 0;
  std::vector<double> cross_t;
  double prev = joint_coordinate(m, 0, st.poses);
  for (int k = 0; k < 2400; ++k) {
    const StepDiagnostics d = step(m, st, cfg);
    max_kkt = std::max(max_kkt, d.kkt_momentum_inf);
    max_v = std::max(max_v, d.bilateral_velocity_inf);
    max_f = std::max(max_f, maxabs(build_bilateral(m, st.poses).f));
    max_e = std::max(max_e, std::abs(kinetic_energy(m, st) + potential_energy(m, st) - e0));
    const double c = joint_coordinate(m, 0, st.poses);
    if (prev < 0.0 && c >= 0.0) cross_t.push_back(st.time - cfg.dt + (-prev / (c - prev)) * cfg.dt);
    prev = c;
  }
  CHECK(max_f < 1e-5);
  CHECK(max_e / e_amp < 0.02);
  CHECK(max_kkt < 1e-5);
  CHECK(max_v < 1e-5);
  REQUIRE(cross_t.size() >= 3);
  const double period = (cross_t.back() - cross_t.front()) / (cross_t.size() - 1);
  const double expected = 2.0 * M_PI / std::sqrt(mass * g * L / (mass * L * L + iyy));
  CHECK(std::abs(period - expected) / expected < 0.01);
}
TEST(step_fourbar_pd, "test_stepper.cpp:172 four-bar under PD drive keeps the loop closed") {
  const LoadedScene ls = load("fourbar");
  const MechanismModel m = build_model(ls.scene);
  WorldState st = initial_state(m);
  const double start = joint_coordinate(m, 0, st.poses);
  double max_f = 0;
  for (int k = 0; k < 480; ++k) {
    step(m, st, ls.config);
    max_f = std::max(max_f, maxabs(build_bilateral(m, st.poses).f));
  }
  CHECK(max_f < 1e-4);
  double turned = joint_coordinate(m, 0, st.poses) - start;
  if (turned < -M_PI) turned += 2.0 * M_PI;
  CHECK(turned > 1.2);
  CHECK(turned < 3.2);
}
TEST(step_mj_vs_si, "test_stepper.cpp:193 Moreau-Jean and semi-implicit agree to O(dt^2)") {
  const MechanismModel m = load_model("pendulum");
  StepConfig eu;
  eu.dt = 1e-4;
  StepConfig mj = eu;
  mj.integrator = Integrator::MoreauJean;
  WorldState se = initial_state(m), sm = initial_state(m);
  for (int k = 0; k < 1000; ++k) {
    step(m, se, eu);
    step(m, sm, mj);
  }
  CHECK(inf_norm(se.poses[0].position - sm.poses[0].position) < 1e-5);
  CHECK(inf_norm(se.twists[0].linear - sm.twists[0].linear) < 1e-4);
}
TEST(step_warmstart, "test_stepper.cpp:209 + acceptance #10: warm start halves mean iterations") {
  const MechanismModel m = load_model("sphere_on_plane");
  StepConfig warm, cold;
  cold.warm_start = false;
  WorldState sw = initial_state(m), sc = initial_state(m);
  double wi = 0, ci = 0;
  for (int k = 0; k < 200; ++k) {
    wi += step(m, sw, warm).solver.iterations;
    ci += step(m, sc, cold).solver.iterations;
  }
  CHECK(wi <= 0.5 * ci);
  CHECK(std::abs(sw.poses[0].position.z - 0.1) < 1e-4);
  CHECK(norm(sw.twists[0].linear) < 1e-6);
}
TEST(step_limits, "test_stepper.cpp:228 joint limits stop the swing inside the bound") {
  LoadedScene ls = load("pendulum");
  ls.scene.joints[0].has_limits = true;
  ls.scene.joints[0].lower = -0.02;
  ls.scene.joints[0].upper = 1.0;
  const MechanismModel m = build_model(ls.scene);
  StepConfig cfg;
  WorldState st = initial_state(m);
  double mn = 1.0;
  for (int k = 0; k < 2400; ++k) {
    step(m, st, cfg);
    mn = std::min(mn, joint_coordinate(m, 0, st.poses));
  }
  CHECK(mn > -0.021);
  CHECK(mn < 0.0);
}
TEST(step_unit_quat, "test_stepper.cpp:245 quaternions stay unit through long runs") {
  for (const char* name : {"pendulum", "fourbar"}) {
    const LoadedScene ls = load(name);
    const MechanismModel m = build_model(ls.scene);
    WorldState st = initial_state(m);
    for (int k = 0; k < 1200; ++k) step(m, st, ls.config);
    for (const Pose& p : st.poses) CHECK(std::abs(p.orientation.norm() - 1.0) < 1e-9);
  }
}
static SceneDescription incline_scene(double theta, double mu) {  // acceptance.cpp:60-89
  SceneDescription s;
  s.name = "incline";
  s.gravity = Vec3(0, 0, -9.81);
  const Vec3 nrm(-std::sin(theta), 0.0, std::cos(theta));
  SceneBody crate;
  crate.name = "crate";
  crate.mass = 1.0;
  const double hx = 0.1, hy = 0.1, hz = 0.05;
  crate.inertia = Mat3::diagonal(Vec3((hy * hy + hz * hz) / 3.0, (hx * hx + hz * hz) / 3.0, (hx * hx + hy * hy) / 3.0));
  crate.pose.position = hz * nrm;
  crate.pose.orientation = axis_angle(-theta, Vec3(0, 1, 0));
  s.bodies.push_back(crate);
  SceneGeom box, plane;
  box.body = "crate";
  box.shape = "box";
  box.half_extents = Vec3(hx, hy, hz);
  box.mu = mu;
  plane.body = "world";
  plane.shape = "plane";
  plane.normal = nrm;
  plane.mu = mu;
  s.geoms.push_back(box);
  s.geoms.push_back(plane);
  return s;
}
TEST(step_sliding, "test_stepper.cpp:260 sliding contacts keep zero normal relative velocity") {
  const double mu = 0.5, theta = std::atan(mu) * 1.3;
  const MechanismModel m = build_model(incline_scene(theta, mu));
  const Vec3 nrm(-std::sin(theta), 0.0, std::cos(theta));
  StepConfig cfg;
  WorldState st = initial_state(m);
  for (int k = 0; k < 240; ++k) step(m, st, cfg);
  CHECK(norm(st.twists[0].linear) > 0.3);
  CHECK(std::abs(dot(nrm, st.twists[0].linear)) < 1e-5);
  CHECK(std::abs(dot(nrm, st.poses[0].position) - 0.05) < 1e-4);
}
TEST(step_dense_vs_mf, "test_stepper.cpp:295 dense and matrix-free trajectories within 1e-6") {
  const LoadedScene ls = load("fourbar");
  const MechanismModel m = build_model(ls.scene);
  StepConfig dense = ls.config;
  dense.backend = BackendChoice::Dense;
  StepConfig sparse = dense;
  sparse.backend = BackendChoice::MatrixFree;
  sparse.cr_iters = 50;
  WorldState sd = initial_state(m), ss = initial_state(m);
  double worst = 0;
  for (int k = 0; k < 480; ++k) {
    step(m, sd, dense);
    step(m, ss, sparse);
    for (int b = 0; b < m.n_bodies(); ++b) worst = std::max(worst, inf_norm(sd.poses[b].position - ss.poses[b].position));
  }
  CHECK(worst < 1e-6);
}
TEST(step_restitution, "test_stepper.cpp:319 sphere impacting with restitution bounces back") {
  LoadedScene ls = load("sphere_on_plane");
  ls.scene.bodies[0].pose.position = Vec3(0, 0, 0.15);
  ls.scene.bodies[0].twist.linear = Vec3(0, 0, -1.0);
  ls.scene.geoms[0].restitution = 0.5;
  const MechanismModel m = build_model(ls.scene);
  StepConfig cfg;
  WorldState st = initial_state(m);
  double up = -1.0;
  for (int k = 0; k < 240; ++k) {
    step(m, st, cfg);
    up = std::max(up, st.twists[0].linear.z);
  }
  CHECK(up > 0.3);
  CHECK(up < 0.75);
}

// ======================================================================= batch
TEST(batch_identical, "test_batch.cpp:43 two identical worlds stay bitwise identical") {
  WorldBatch b;
  auto m = std::make_shared<const MechanismModel>(load_model("fourbar"));
  b.add_world(m);
  b.add_world(m);
  for (int k = 0; k < 100; ++k) batch_step(b, StepConfig{}, 2);
  CHECK(states_bitwise_equal(b.extract_state(0), b.extract_state(1)));
}
TEST(batch_hetero, "test_batch.cpp:53 + acceptance #9: heterogeneous batch equals solo runs") {
  WorldBatch b;
  std::vector<std::shared_ptr<const MechanismModel>> ms;
  for (const char* n : {"fourbar", "sphere_on_plane", "freefall"}) {
    ms.push_back(std::make_shared<const MechanismModel>(load_model(n)));
    b.add_world(ms.back());
  }
  std::vector<WorldState> solo;
  for (auto& m : ms) solo.push_back(initial_state(*m));
  for (int k = 0; k < 200; ++k) {
    batch_step(b, StepConfig{}, 2);
    for (size_t w = 0; w < ms.size(); ++w) step(*ms[w], solo[w], StepConfig{});
  }
  for (size_t w = 0; w < ms.size(); ++w) CHECK(states_bitwise_equal(b.extract_state((int)w), solo[w]));
}
TEST(batch_mask, "test_batch.cpp:79 inactive worlds are skipped") {
  WorldBatch b;
  auto m = std::make_shared<const MechanismModel>(load_model("freefall"));
  b.add_world(m);
  b.add_world(m);
  b.set_active(0, false);
  batch_step(b, StepConfig{});
  CHECK(b.extract_state(0).time == 0.0);
  CHECK(approx(b.extract_state(1).time, 1.0 / 240.0));
  CHECK(b.converged(1));
}
TEST(batch_offsets, "test_batch.cpp:93 per-world storage offsets are prefix sums") {
  WorldBatch b;
  auto fb = std::make_shared<const MechanismModel>(load_model("fourbar"));
  auto sp = std::make_shared<const MechanismModel>(load_model("sphere_on_plane"));
  b.add_world(fb);
  b.add_world(sp);
  b.add_world(fb);
  CHECK(b.pose_offset(0) == 0 && b.pose_offset(1) == 21 && b.pose_offset(2) == 28);
  CHECK(b.twist_offset(1) == 18 && b.twist_offset(2) == 24);
  CHECK(b.pose_storage().size() == 49);
}
TEST(batch_threads, "test_batch.cpp:108 results independent of thread count") {
  auto m = std::make_shared<const MechanismModel>(load_model("serial_chain_10"));
  WorldBatch one, many;
  for (int w = 0; w < 6; ++w) {
    one.add_world(m);
    many.add_world(m);
  }
  for (int k = 0; k < 50; ++k) {
    batch_step(one, StepConfig{}, 1);
    batch_step(many, StepConfig{}, 4);
  }
  for (int w = 0; w < 6; ++w) CHECK(states_bitwise_equal(one.extract_state(w), many.extract_state(w)));
}

// ======================================================================= acceptance
TEST(acc1_kkt, "acceptance.cpp:93 #1 KKT momentum balance <= 1e-5 on all scenes") {
  double worst = 0;
  for (const char* n : {"freefall", "pendulum", "sphere_on_plane", "inclined_box", "fourbar", "double_fourbar",
                        "serial_chain_10"}) {
    const LoadedScene ls = load(n);
    const MechanismModel m = build_model(ls.scene);
    WorldState st = initial_state(m);
    for (int k = 0; k < 480; ++k) worst = std::max(worst, step(m, st, ls.config).kkt_momentum_inf);
  }
  CHECK(worst <= 1e-5);
}
TEST(acc2_backend, "acceptance.cpp:114 #2 backend equivalence <= 1e-6 relative") {
  double worst = 0;
  for (const char* n : {"fourbar", "serial_chain_10"}) {
    const LoadedScene ls = load(n);
    const MechanismModel m = build_model(ls.scene);
    StepConfig dc = ls.config, mc = ls.config;
    dc.backend = BackendChoice::Dense;
    mc.backend = BackendChoice::MatrixFree;
    mc.cr_iters = 50;
    WorldState st = initial_state(m);
    for (int k = 0; k < 100; ++k) {
      WorldState ms = st;
      const StepDiagnostics mf = step(m, ms, mc);
      const StepDiagnostics dd = step(m, st, dc);
      const double sc = std::max(1e-9, maxabs(dd.impulses));
      double e = 0;
      for (size_t i = 0; i < dd.impulses.size(); ++i) e = std::max(e, std::abs(dd.impulses[i] - mf.impulses[i]));
      worst = std::max(worst, e / sc);
    }
  }
  CHECK(worst <= 1e-6);
}
TEST(acc3_budget, "acceptance.cpp:137 #3 PADMM <= 30 iterations after warm-up") {
  int worst = 0;
  for (const char* n : {"sphere_on_plane", "fourbar"}) {
    LoadedScene ls = load(n);
    ls.config.dt = 1.0 / 240.0;
    ls.config.solver.eps = 1e-6;
    const MechanismModel m = build_model(ls.scene);
    WorldState st = initial_state(m);
    for (int k = 0; k < 2400; ++k) {
      const StepDiagnostics d = step(m, st, ls.config);
      if (k >= 10) worst = std::max(worst, d.solver.iterations);
    }
  }
  CHECK(worst <= 30);
}
TEST(acc4_cr9, "acceptance.cpp:157 #4 9-iteration CR viability: KKT <= 5e-5 over 10 s") {
  LoadedScene ls = load("fourbar");
  ls.config.backend = BackendChoice::MatrixFree;
  ls.config.cr_iters = 9;
  const MechanismModel m = build_model(ls.scene);
  WorldState st = initial_state(m);
  double worst = 0;
  for (int k = 0; k < 2400; ++k) worst = std::max(worst, step(m, st, ls.config).kkt_momentum_inf);
  CHECK(worst <= 5e-5);
}
TEST(acc5_loops, "acceptance.cpp:170 #5 loop closure on fourbar and double_fourbar") {
  for (const char* n : {"fourbar", "double_fourbar"}) {
    const LoadedScene ls = load(n);
    const MechanismModel m = build_model(ls.scene);
    WorldState st = initial_state(m);
    double mf = 0, ce = 0;
    for (int k = 0; k < 2400; ++k) {
      step(m, st, ls.config);
      mf = std::max(mf, maxabs(build_bilateral(m, st.poses).f));
      if ((k + 1) % 240 == 0 && std::string(n) == "fourbar") {
        // circle-circle closed form (tests/oracles.hpp:61-79)
        const double crank = joint_coordinate(m, 0, st.poses);
        const double ax = 0.5 * std::cos(crank), ay = 0.5 * std::sin(crank);
        const double dx = 2.0 - ax, dy = -ay, d = std::hypot(dx, dy);
        const double alpha = (d * d + 4.0 - 2.25) / (2.0 * d);
        const double h = std::sqrt(std::max(0.0, 4.0 - alpha * alpha));
        const double ux = dx / d, uy = dy / d;
        const double bx = ax + alpha * ux - h * uy, by = ay + alpha * uy + h * ux;
        const double coupler = std::atan2(by - ay, bx - ax);
        const Vec3 xa = st.poses[1].orientation * Vec3(1, 0, 0);
        ce = std::max(ce, std::abs(std::remainder(std::atan2(xa.y, xa.x) - coupler, 2.0 * M_PI)));
      }
    }
    CHECK(mf < 1e-4);
    CHECK(ce < 1e-3);
  }
}
TEST(acc6_friction, "acceptance.cpp:206 #6 friction threshold physics") {
  const double mu = 0.5;
  {
    const MechanismModel m = build_model(incline_scene(std::atan(mu) * 0.9, mu));
    WorldState st = initial_state(m);
    StepDiagnostics last;
    for (int k = 0; k < 480; ++k) last = step(m, st, StepConfig{});
    bool interior = last.contact_count > 0;
    for (int c = 0; c < last.contact_count; ++c) {
      const int r = last.first_contact_row + 3 * c;
      if (!(std::hypot(last.impulses[r + 1], last.impulses[r + 2]) < mu * last.impulses[r])) interior = false;
    }
    CHECK(norm(st.twists[0].linear) < 1e-6);
    CHECK(interior);
  }
  {
    const MechanismModel m = build_model(incline_scene(std::atan(mu) * 1.1, mu));
    WorldState st = initial_state(m);
    StepDiagnostics last;
    for (int k = 0; k < 240; ++k) last = step(m, st, StepConfig{});
    bool boundary = last.contact_count > 0;
    for (int c = 0; c < last.contact_count; ++c) {
      const int r = last.first_contact_row + 3 * c;
      const double ln = last.impulses[r], lt = std::hypot(last.impulses[r + 1], last.impulses[r + 2]);
      if (ln > 1e-8 && std::abs(lt - mu * ln) > 1e-3 * std::max(1e-12, mu * ln)) boundary = false;
    }
    CHECK(norm(st.twists[0].linear) > 0.1);
    CHECK(boundary);
  }
  {
    const LoadedScene ls = load("sphere_on_plane");
    const MechanismModel m = build_model(ls.scene);
    WorldState st = initial_state(m);
    StepDiagnostics last;
    for (int k = 0; k < 480; ++k) last = step(m, st, ls.config);
    const double ex = 1.0 * 9.81 * ls.config.dt;
    CHECK(std::abs(last.impulses[last.first_contact_row] - ex) / ex < 1e-3);
  }
}
TEST(acc8_energy, "acceptance.cpp:281 #8 pendulum energy: euler < 2%, moreau <= euler") {
  auto drift = [](Integrator integ) {
    LoadedScene ls = load("pendulum");
    ls.config.integrator = integ;
    const MechanismModel m = build_model(ls.scene);
    WorldState st = initial_state(m);
    const double e0 = kinetic_energy(m, st) + potential_energy(m, st);
    const double amp = 9.81 * (1.0 - std::cos(0.05));
    double worst = 0;
    for (int k = 0; k < 2400; ++k) {
      step(m, st, ls.config);
      worst = std::max(worst, std::abs(kinetic_energy(m, st) + potential_energy(m, st) - e0) / amp);
    }
    return worst;
  };
  const double eu = drift(Integrator::SemiImplicitEuler), mj = drift(Integrator::MoreauJean);
  CHECK(eu < 0.02);
  CHECK(mj <= eu);
}

// ---------------------------------------------------------------- fk (test_fk.cpp)
namespace {
std::vector<Pose> fk_initial(const MechanismModel& m) {
  std::vector<Pose> p;
  for (const BodySpec& b : m.bodies) p.push_back(b.initial_pose);
  return p;
}
double body_plane_angle(const Pose& pose) {  // test_fk.cpp:26-30
  const Vec3 x_axis = pose.orientation * Vec3{1, 0, 0};
  return std::atan2(x_axis.y, x_axis.x);
}
// oracles::solve_fourbar (oracles.hpp:61-79), branch +1
bool solve_fourbar(double crank_angle, double& coupler_angle, double& rocker_angle, double ground = 2.0,
                   double crank = 0.5, double coupler = 2.0, double rocker = 1.5) {
  const double ax = crank * std::cos(crank_angle), ay = crank * std::sin(crank_angle);
  const double dx = ground - ax, dy = -ay;
  const double d = std::sqrt(dx * dx + dy * dy);
  if (d > coupler + rocker || d < std::abs(coupler - rocker)) return false;
  const double alpha = (d * d + coupler * coupler - rocker * rocker) / (2.0 * d);
  const double h = std::sqrt(std::max(0.0, coupler * coupler - alpha * alpha));
  const double ux = dx / d, uy = dy / d;
  const double bx = ax + alpha * ux - h * uy, by = ay + alpha * uy + h * ux;
  coupler_angle = std::atan2(by - ay, bx - ax);
  rocker_angle = std::atan2(by, bx - ground);
  return true;
}
}  // namespace

TEST(fk_consistent, "test_fk.cpp:33 fk on an already-consistent input returns immediately, poses untouched") {
  const MechanismModel m = build_model(load("fourbar").scene);
  const std::vector<Pose> init = fk_initial(m);
  const FkResult r = fk_solve(m, {{0, joint_coordinate(m, 0, init)}}, init);
  CHECK(r.converged);
  CHECK(r.iterations == 0);
  for (size_t b = 0; b < r.poses.size(); ++b) {
    CHECK(r.poses[b].position.x == init[b].position.x && r.poses[b].position.y == init[b].position.y &&
          r.poses[b].position.z == init[b].position.z);
    CHECK(r.poses[b].orientation.w == init[b].orientation.w && r.poses[b].orientation.z == init[b].orientation.z);
  }
}

TEST(fk_two_link, "test_fk.cpp:49 fk on a serial two-link chain matches composed transforms") {
  SceneDescription s;
  for (int i = 0; i < 2; ++i) {
    SceneBody b;
    b.name = "link" + std::to_string(i);
    b.inertia = Mat3::identity();
    b.inertia(0, 0) = 1e-4;
    b.inertia(1, 1) = 0.02;
    b.inertia(2, 2) = 0.02;
    b.pose.position = Vec3{0.5 + i, 0.0, 0.0};
    s.bodies.push_back(b);
  }
  SceneJoint j0;
  j0.name = "q0";
  j0.type = "revolute";
  j0.parent = "world";
  j0.child = "link0";
  j0.frame_in_child.position = Vec3{-0.5, 0, 0};
  j0.axis = Vec3{0, 0, 1};
  s.joints.push_back(j0);
  SceneJoint j1 = j0;
  j1.name = "q1";
  j1.parent = "link0";
  j1.child = "link1";
  j1.frame_in_parent.position = Vec3{0.5, 0, 0};
  s.joints.push_back(j1);
  const MechanismModel m = build_model(s);
  const double q0 = 0.4, q1 = -0.9;
  const FkResult r = fk_solve(m, {{0, q0}, {1, q1}}, fk_initial(m));
  REQUIRE(r.converged);
  CHECK(r.residual_inf < 1e-8);
  const Vec3 elbow{std::cos(q0), std::sin(q0), 0.0};
  const Vec3 com0 = 0.5 * elbow;
  const Vec3 com1 = elbow + 0.5 * Vec3{std::cos(q0 + q1), std::sin(q0 + q1), 0.0};
  CHECK(norm(r.poses[0].position - com0) < 1e-7);
  CHECK(norm(r.poses[1].position - com1) < 1e-7);
  CHECK(approx(body_plane_angle(r.poses[0]), q0, 1e-7));
  CHECK(approx(body_plane_angle(r.poses[1]), q0 + q1, 1e-7));
}

TEST(fk_fourbar, "test_fk.cpp:95 fk on the four-bar matches the analytic position solution") {
  const MechanismModel m = build_model(load("fourbar").scene);
  for (double delta : {0.1, 0.4, -0.3, 0.9}) {
    const double crank = M_PI / 2 + delta;
    const FkResult r = fk_solve(m, {{0, crank}}, fk_initial(m));
    REQUIRE(r.converged);
    CHECK(r.residual_inf < 1e-8);
    double ca = 0, ra = 0;
    REQUIRE(solve_fourbar(crank, ca, ra));
    CHECK(approx(body_plane_angle(r.poses[1]), ca, 1e-6));
    CHECK(approx(body_plane_angle(r.poses[2]), ra, 1e-6));
  }
}

TEST(fk_no_close, "test_fk.cpp:114 fk flags non-convergence when the loop cannot close") {
  const json j = json::parse(R"json({
    "name": "fourbar_long_crank", "gravity": [0, -9.81, 0],
    "bodies": [
      {"name": "crank", "mass": 1.0, "inertia": [1e-4, 0.2, 0.2],
       "position": [0.0, 0.75, 0.0], "orientation": [0.7071067811865476, 0, 0, 0.7071067811865476]},
      {"name": "coupler", "mass": 1.0, "inertia": [1e-4, 0.1, 0.1],
       "position": [0.43014417303072305, 1.2450961153538151, 0.0],
       "orientation": [0.964439823436757, 0.0, 0.0, -0.26430252925251585]},
      {"name": "rocker", "mass": 1.0, "inertia": [1e-4, 0.1, 0.1],
       "position": [0.930144173030723, 0.49509611535381526, 0.0],
       "orientation": [0.6558537741224968, 0.0, 0.0, 0.7548879565665867]}],
    "joints": [
      {"name": "crank_pivot", "type": "revolute", "parent": "world", "child": "crank",
       "parent_position": [0, 0, 0], "child_position": [-0.75, 0, 0], "axis": [0, 0, 1]},
      {"name": "crank_coupler", "type": "revolute", "parent": "crank", "child": "coupler",
       "parent_position": [0.75, 0, 0], "child_position": [-0.5, 0, 0], "axis": [0, 0, 1]},
      {"name": "coupler_rocker", "type": "revolute", "parent": "coupler", "child": "rocker",
       "parent_position": [0.5, 0, 0], "child_position": [0.5, 0, 0], "axis": [0, 0, 1]},
      {"name": "rocker_ground", "type": "revolute", "parent": "world", "child": "rocker",
       "parent_position": [1, 0, 0], "child_position": [-0.5, 0, 0], "axis": [0, 0, 1]}],
    "geoms": []})json");
  const MechanismModel m = build_model(scene_from_json(j).scene);
  const FkResult r = fk_solve(m, {{0, M_PI}}, fk_initial(m));
  CHECK(!r.converged);
  CHECK(r.residual_inf > 1e-3);
  CHECK((int)r.poses.size() == m.n_bodies());
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s scenes_bundle.json [filter]\n", argv[0]);
    return 2;
  }
  std::ifstream in(argv[1]);
  std::stringstream ss;
  ss << in.rdbuf();
  g_bundle = json::parse(ss.str());
  const char* filter = argc > 2 ? argv[2] : nullptr;
  int failed = 0, ran = 0;
  for (const TestCase& t : registry()) {
    if (filter && std::string(t.name).find(filter) == std::string::npos) continue;
    g_fail_count = 0;
    g_fail_msg.clear();
    try {
      t.fn();
    } catch (const std::exception& e) {
      ++g_fail_count;
      g_fail_msg += std::string(" exception: ") + e.what();
    }
    ++ran;
    std::printf("[%s] %s%s\n", g_fail_count ? "FAIL" : "PASS", t.name, g_fail_msg.c_str());
    if (g_fail_count) ++failed;
  }
  std::printf("%d/%d oracle tests passed\n", ran - failed, ran);
  return failed;
}
