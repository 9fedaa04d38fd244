// oracle.hpp — TEST INFRASTRUCTURE ONLY.
//
// CPU fp64 restatement of the reference loopdyn solver path
// (/root/reference/proj/src/*.cpp), used by tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg as the parity checker.  It is never linked into
// or called by the product (paper_2603_16536_b200/).  Eigen is absent from this
// image, so the few Eigen operations the reference relies on are restated here
// with Eigen's own formulas: Quaternion product,
// toRotationMatrix, Quaternion(Mat3), q*v, normalize, unblocked LLT.
// Bitwise agreement with Eigen itself is unpinned (Eigen cannot be built here);
// the oracle is pinned by the reference's own known-answer tests instead
// (oracle/oracle_tests.cpp).
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------- small math
struct Vec3 {
  double x = 0, y = 0, z = 0;
  Vec3() = default;
  Vec3(double a, double b, double c) : x(a), y(b), z(c) {}
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
};
inline Vec3 operator+(const Vec3& a, const Vec3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline Vec3 operator-(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline Vec3 operator-(const Vec3& a) { return {-a.x, -a.y, -a.z}; }
inline Vec3 operator*(double s, const Vec3& a) { return {s * a.x, s * a.y, s * a.z}; }
inline Vec3 operator/(const Vec3& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline double dot(const Vec3& a, const Vec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline double squared_norm(const Vec3& a) { return a.x * a.x + a.y * a.y + a.z * a.z; }
inline double norm(const Vec3& a) { return std::sqrt(squared_norm(a)); }
inline Vec3 cross(const Vec3& a, const Vec3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline Vec3 normalized(const Vec3& a) { return a / norm(a); }
inline double inf_norm(const Vec3& a) {
  return std::max(std::abs(a.x), std::max(std::abs(a.y), std::abs(a.z)));
}

struct Mat3 {
  double m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // row-major
  double operator()(int r, int c) const { return m[3 * r + c]; }
  double& operator()(int r, int c) { return m[3 * r + c]; }
  static Mat3 identity() {
    Mat3 a;
    a(0, 0) = a(1, 1) = a(2, 2) = 1.0;
    return a;
  }
  static Mat3 diagonal(const Vec3& d) {
    Mat3 a;
    a(0, 0) = d.x;
    a(1, 1) = d.y;
    a(2, 2) = d.z;
    return a;
  }
  Vec3 row(int r) const { return {m[3 * r], m[3 * r + 1], m[3 * r + 2]}; }
  Vec3 col(int c) const { return {m[c], m[3 + c], m[6 + c]}; }
  Mat3 transpose() const {
    Mat3 t;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) t(c, r) = (*this)(r, c);
    return t;
  }
};
inline Mat3 operator*(const Mat3& a, const Mat3& b) {
  Mat3 o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double s = a(r, 0) * b(0, c);
      s += a(r, 1) * b(1, c);
      s += a(r, 2) * b(2, c);
      o(r, c) = s;
    }
  return o;
}
inline Vec3 operator*(const Mat3& a, const Vec3& v) {
  return {a(0, 0) * v.x + a(0, 1) * v.y + a(0, 2) * v.z,
          a(1, 0) * v.x + a(1, 1) * v.y + a(1, 2) * v.z,
          a(2, 0) * v.x + a(2, 1) * v.y + a(2, 2) * v.z};
}
inline Mat3 operator+(const Mat3& a, const Mat3& b) {
  Mat3 o;
  for (int i = 0; i < 9; ++i) o.m[i] = a.m[i] + b.m[i];
  return o;
}
inline Mat3 operator-(const Mat3& a, const Mat3& b) {
  Mat3 o;
  for (int i = 0; i < 9; ++i) o.m[i] = a.m[i] - b.m[i];
  return o;
}
inline Mat3 operator*(double s, const Mat3& a) {
  Mat3 o;
  for (int i = 0; i < 9; ++i) o.m[i] = s * a.m[i];
  return o;
}
inline Mat3 operator-(const Mat3& a) { return -1.0 * a; }
// Row vector times matrix: v^T A.
inline Vec3 row_times(const Vec3& v, const Mat3& a) {
  return {v.x * a(0, 0) + v.y * a(1, 0) + v.z * a(2, 0),
          v.x * a(0, 1) + v.y * a(1, 1) + v.z * a(2, 1),
          v.x * a(0, 2) + v.y * a(1, 2) + v.z * a(2, 2)};
}

// Hamilton quaternion, Eigen formulas (Quaternion.h).
struct Quat {
  double w = 1, x = 0, y = 0, z = 0;
  Quat() = default;
  Quat(double w_, double x_, double y_, double z_) : w(w_), x(x_), y(y_), z(z_) {}
  Vec3 vec() const { return {x, y, z}; }
  double norm() const { return std::sqrt(x * x + y * y + z * z + w * w); }
  void normalize() {
    const double n = norm();
    w /= n;
    x /= n;
    y /= n;
    z /= n;
  }
  Quat normalized() const {
    Quat q = *this;
    q.normalize();
    return q;
  }
  Mat3 to_rotation_matrix() const;
  static Quat from_matrix(const Mat3& m);
};
Quat operator*(const Quat& a, const Quat& b);
Vec3 operator*(const Quat& q, const Vec3& v);

using Vec = std::vector<double>;
struct Row6 {
  double v[6] = {0, 0, 0, 0, 0, 0};
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
};

// ---------------------------------------------------------------- se3 (se3.cpp)
Mat3 skew(const Vec3& v);
Quat quat_exp(const Vec3& v);
Quat quat_integrate(const Quat& q, const Vec3& w, double dt);
Mat3 so3_exp(const Vec3& phi);
Vec3 so3_log(const Quat& q);
Vec3 so3_log(const Mat3& r);
Mat3 left_jacobian_inverse(const Vec3& phi);
struct InertiaBlock {
  double mass = 1.0;
  Mat3 body_inertia = Mat3::identity();
};
Mat3 world_inertia(const InertiaBlock& in, const Quat& q);
Mat3 llt_inverse3(const Mat3& a);  // Mat3::llt().solve(Identity)
void orthonormal_complement(const Vec3& axis, Vec3& b1, Vec3& b2);

struct Pose {
  Vec3 position;
  Quat orientation;
  Mat3 rotation() const { return orientation.to_rotation_matrix(); }
  Vec3 transform(const Vec3& p) const { return position + orientation * p; }
};
struct Twist {
  Vec3 linear, angular;
};

// ---------------------------------------------------------------- scene/model
struct SceneBody {
  std::string name;
  double mass = 1.0;
  Mat3 inertia = Mat3::identity();
  Pose pose;
  Twist twist;
};
struct SceneJoint {
  std::string name, type, parent, child;
  Pose frame_in_parent, frame_in_child;
  Vec3 axis{0, 0, 1};
  bool has_limits = false;
  double lower = 0, upper = 0;
  double kp = 0, kd = 0;
  bool has_target = false;
  double target = 0;
  double target_rate = 0, armature = 0, damping = 0;
};
struct SceneGeom {
  std::string body, shape;
  double radius = 0;
  Vec3 half_extents;
  Vec3 normal{0, 0, 1};
  double offset = 0, mu = 0, restitution = 0;
};
struct SceneDescription {
  std::string name;
  Vec3 gravity{0, 0, -9.81};
  std::vector<SceneBody> bodies;
  std::vector<SceneJoint> joints;
  std::vector<SceneGeom> geoms;
  bool box_box = false;  // extension (not in the reference, which rejects box-box pairs, model.cpp:56-62)
};

constexpr int kWorld = -1;
enum class JointType { Fixed, Revolute, Prismatic, Spherical };
enum class Shape { Sphere, Plane, Box };

struct ModelError : std::runtime_error {
  int code;  // ModelError::Code index (model.hpp:78-88)
  ModelError(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};
enum ModelCode {
  InvalidReference = 0, NonUnitAxis, BadInertia, BadLimits, UnsupportedOnJointType, BadGeometry,
  UnsupportedCollisionPair, WrongJointType, DuplicateName
};

struct JointSpec {
  std::string name;
  JointType type = JointType::Fixed;
  int parent = kWorld, child = 0;
  Pose frame_in_parent, frame_in_child;
  Vec3 axis{0, 0, 1};
  bool has_limits = false;
  double lower = 0, upper = 0;
  bool has_actuation = false;
  double kp = 0, kd = 0, target = 0, target_rate = 0, armature = 0, damping = 0;
};
struct GeomSpec {
  int body = kWorld;
  Shape shape = Shape::Sphere;
  double radius = 0;
  Vec3 half_extents;
  Vec3 plane_normal{0, 0, 1};
  double plane_offset = 0, mu = 0, restitution = 0;
};
struct BodySpec {
  std::string name;
  InertiaBlock inertia;
  Pose initial_pose;
  Twist initial_twist;
};
struct JointLayout {
  int row_offset = 0, row_count = 0, dyn_offset = 0, dyn_count = 0;
  bool has_pd = false, has_armature = false, has_damping = false;
  Vec3 comp0, comp1;  // orthonormal complement columns
};
struct MechanismModel {
  std::string name;
  std::vector<BodySpec> bodies;
  std::vector<JointSpec> joints;
  std::vector<GeomSpec> geoms;
  Vec3 gravity{0, 0, -9.81};
  std::vector<JointLayout> joint_layout;
  int n_bilateral_rows = 0, n_dynamics_rows = 0, n_loops = 0;
  bool box_box = false;  // extension: box-box pairs collide (box_box below)
  int n_bodies() const { return (int)bodies.size(); }
};
int joint_row_count(JointType t);
MechanismModel build_model(const SceneDescription& scene);
struct JointFrames {
  Vec3 anchor_parent, anchor_child;
  Mat3 frame_parent, frame_child;
};
JointFrames joint_world_frames(const MechanismModel& m, int joint, const std::vector<Pose>& poses);
double joint_coordinate(const MechanismModel& m, int joint, const std::vector<Pose>& poses);

// ---------------------------------------------------------------- contacts
struct ContactPoint {
  int geom_a = -1, geom_b = -1;
  Vec3 position, normal{0, 0, 1};
  double depth = 0, mu = 0, restitution = 0;
};
Mat3 contact_frame(const Vec3& normal);  // columns n, t1, t2
std::vector<ContactPoint> collide(const MechanismModel& m, const std::vector<Pose>& poses,
                                  double margin);
struct ReactionCacheEntry {
  int geom_a = -1, geom_b = -1;
  Vec3 position, impulse, dual;
};
struct ContactInit {
  Vec3 impulse, dual;
};
std::vector<ContactInit> match_warmstart(const std::vector<ReactionCacheEntry>& cache,
                                         const std::vector<ContactPoint>& contacts,
                                         double tolerance = 1e-3);

// ---------------------------------------------------------------- constraints
struct JacobianRow {
  int body_a = -1, body_b = -1;
  Row6 block_a, block_b;
  double dot(const Vec& u) const;
};
enum class ConeKind { Bilateral, Nonnegative, SecondOrder };
struct ConeGroup {
  ConeKind kind = ConeKind::Bilateral;
  int begin = 0, dim = 0;
  double mu = 0;
};
struct ConeProduct {
  std::vector<ConeGroup> groups;
  int n_rows = 0;
};
struct ConstraintSet {
  int n_rows = 0, n_bodies = 0, n_bilateral = 0, n_dynamics = 0, n_limits = 0, n_contact_rows = 0;
  std::vector<JacobianRow> rows;
  Vec bias, reg, bilateral_f, limit_gap;
  std::vector<std::pair<int, int>> limit_keys;
  ConeProduct cones;
  std::vector<ContactPoint> contacts;
  std::vector<Mat3> contact_frames;
  int first_limit_row() const { return n_bilateral + n_dynamics; }
  int first_contact_row() const { return n_bilateral + n_dynamics + n_limits; }
  Vec apply_jacobian(const Vec& u) const;
  Vec apply_jacobian_transpose(const Vec& lambda) const;
};
struct AssembleConfig {
  double dt = 1.0 / 240.0, beta = 0.2, bias_clamp = 10.0, limit_margin_angular = 0.01,
         limit_margin_linear = 0.001, impact_velocity_threshold = 0.1;
};
struct BilateralBlock {
  std::vector<JacobianRow> rows;
  Vec f;
};
BilateralBlock build_bilateral(const MechanismModel& m, const std::vector<Pose>& poses);
JacobianRow coordinate_rate_row(const MechanismModel& m, int joint, const std::vector<Pose>& poses);
ConstraintSet assemble_constraints(const MechanismModel& m, const std::vector<Pose>& poses,
                                   const std::vector<Twist>& twists,
                                   const std::vector<ContactPoint>& contacts,
                                   const AssembleConfig& cfg);
double constraint_jacobian_fd_check(const MechanismModel& m, const std::vector<Pose>& poses,
                                    double step = 1e-5);

// ---------------------------------------------------------------- delassus
struct BodyInertiaWorld {
  double mass = 1, inv_mass = 1;
  Mat3 inertia_world = Mat3::identity(), inv_inertia_world = Mat3::identity();
};
std::vector<BodyInertiaWorld> world_inertias(const MechanismModel& m, const std::vector<Pose>& poses);
struct Preconditioner {
  Vec scale;
  static Preconditioner identity(int n) { return {Vec(n, 1.0)}; }
};
Preconditioner jacobi_preconditioner(const ConstraintSet& cs, const std::vector<BodyInertiaWorld>& in);
struct DenseMatrix {
  int n = 0;
  Vec a;  // row-major n x n
  double& operator()(int r, int c) { return a[(size_t)r * n + c]; }
  double operator()(int r, int c) const { return a[(size_t)r * n + c]; }
};
struct DenseDelassus {
  DenseMatrix matrix;
  DenseMatrix factor;  // lower Cholesky factor
  bool factorized = false;
  bool factorize();
  Vec solve(const Vec& rhs) const;
};
DenseDelassus assemble_dense(const ConstraintSet& cs, const std::vector<BodyInertiaWorld>& in,
                             double eta_rho, const Preconditioner* precond = nullptr);
struct BakedRow {
  int body_a = -1, body_b = -1;
  Row6 ja, jb, jma, jmb;
};
struct MatrixFreeDelassus {
  std::vector<BakedRow> rows;
  Vec diag_add;
  int n_bodies = 0;
  mutable Vec scratch;
  void apply(const Vec& v, Vec& out) const;
  Vec apply(const Vec& v) const {
    Vec o;
    apply(v, o);
    return o;
  }
};
MatrixFreeDelassus bake_jacobian(const ConstraintSet& cs, const std::vector<BodyInertiaWorld>& in,
                                 const Preconditioner& p, double eta_rho);
struct CrResult {
  int iterations = 0;
  bool breakdown = false;
  double residual_norm = 0;
};
CrResult cr_solve(const MatrixFreeDelassus& op, const Vec& rhs, Vec& x, int max_iters,
                  std::vector<double>* history = nullptr);
enum class BackendChoice { Dense, MatrixFree, Auto };
constexpr int kDenseRowCrossover = 300;
struct DelassusBackend {
  std::unique_ptr<DenseDelassus> dense;
  std::unique_ptr<MatrixFreeDelassus> matrix_free;
  int cr_budget = 9;
  mutable long cr_iterations_total = 0;
  mutable bool cr_breakdown = false;
  void solve(const Vec& rhs, Vec& x) const;
};
DelassusBackend build_backend(const ConstraintSet& cs, const std::vector<BodyInertiaWorld>& in,
                              const Preconditioner& p, double eta_rho, BackendChoice choice,
                              int cr_budget);

// ---------------------------------------------------------------- padmm
struct PadmmConfig {
  double eta = 1e-6, rho = 0.1, eps = 1e-6;
  int max_iters = 200;
  bool acceleration = true, restart = true, fixed_iteration_mode = false;
};
struct SolveDiagnostics {
  int iterations = 0;
  double r_p = 0, r_d = 0, r_c = 0;
  int restarts = 0;
  bool converged = true;
  long cr_iterations = 0;
  bool cr_breakdown = false;
};
struct PadmmState {
  Vec x, y, z, s, y_prev, z_prev, y_hat, z_hat;
  double a = 1.0;
  double r_p = 0, r_d = 0, r_c = 0;
  int iteration = 0, restarts = 0;
};
struct PadmmInit {
  Vec x0, z0;
};
struct PadmmResult {
  Vec lambda, z;
  SolveDiagnostics diagnostics;
};
Vec project_cone(const Vec& w, const ConeProduct& cones);
Vec desaxce_shift(const Vec& v, const ConeProduct& cones);
double nesterov_next_coefficient(double a);
void nesterov_update(PadmmState& st, bool restart);
void padmm_residuals(const Vec& x, const Vec& y, const Vec& y_prev, const Vec& z, double rho,
                     const ConeProduct& cones, double& r_p, double& r_d, double& r_c);
PadmmResult padmm_solve(const DelassusBackend& backend, const Vec& v_f, const ConeProduct& cones,
                        const PadmmInit& init, const PadmmConfig& cfg,
                        std::vector<double>* combined_history = nullptr);

// ---------------------------------------------------------------- stepper
enum class Integrator { SemiImplicitEuler, MoreauJean };
struct StepConfig {
  double dt = 1.0 / 240.0;
  Integrator integrator = Integrator::SemiImplicitEuler;
  BackendChoice backend = BackendChoice::Auto;
  PadmmConfig solver;
  int cr_iters = 9;
  double baumgarte_beta = 0.2, contact_margin = 0.01, impact_velocity_threshold = 0.1,
         bias_clamp = 10.0, limit_margin_angular = 0.01, limit_margin_linear = 0.001;
  bool warm_start = true;
  AssembleConfig assemble_config() const {
    AssembleConfig a;
    a.dt = dt;
    a.beta = baumgarte_beta;
    a.bias_clamp = bias_clamp;
    a.limit_margin_angular = limit_margin_angular;
    a.limit_margin_linear = limit_margin_linear;
    a.impact_velocity_threshold = impact_velocity_threshold;
    return a;
  }
};
struct JointReactionCache {
  Vec lambda, z;
  bool valid = false;
};
struct WorldState {
  std::vector<Pose> poses;
  std::vector<Twist> twists;
  double time = 0;
  JointReactionCache joint_cache;
  std::map<std::pair<int, int>, std::pair<double, double>> limit_cache;
  std::vector<ReactionCacheEntry> contact_cache;
};
WorldState initial_state(const MechanismModel& m);
struct StepDiagnostics {
  SolveDiagnostics solver;
  int n_rows = 0, contact_count = 0, first_contact_row = 0, n_limits = 0;
  Vec impulses;
  double f_inf = 0, kkt_momentum_inf = 0, bilateral_velocity_inf = 0;
};
// Optional per-step trace for one-step parity against the device path.
struct StepTrace {
  ConstraintSet cs;
  Preconditioner precond;
  Vec v_f_scaled, lambda_scaled, z_scaled;
  std::vector<double> history;
};
Vec free_forces(const MechanismModel& m, const std::vector<Pose>& poses,
                const std::vector<Twist>& twists);
StepDiagnostics step(const MechanismModel& m, WorldState& state, const StepConfig& cfg,
                     StepTrace* trace = nullptr);
double kinetic_energy(const MechanismModel& m, const WorldState& s);
double potential_energy(const MechanismModel& m, const WorldState& s);

// ---------------------------------------------------------------- batch
class WorldBatch {
 public:
  int add_world(std::shared_ptr<const MechanismModel> model);
  int add_world(std::shared_ptr<const MechanismModel> model, const WorldState& state);
  int size() const { return (int)entries_.size(); }
  const MechanismModel& model(int w) const { return *entries_[w].model; }
  WorldState extract_state(int w) const;
  void insert_state(int w, const WorldState& s);
  void set_active(int w, bool a) { entries_[w].active = a; }
  bool active(int w) const { return entries_[w].active; }
  bool converged(int w) const { return entries_[w].converged; }
  const StepDiagnostics& diagnostics(int w) const { return entries_[w].diag; }
  int pose_offset(int w) const { return entries_[w].pose_offset; }
  int twist_offset(int w) const { return entries_[w].twist_offset; }
  std::vector<double>& pose_storage() { return poses_; }
  std::vector<double>& twist_storage() { return twists_; }
  std::vector<StepTrace>& traces() { return traces_; }
  bool record_trace = false;
  friend void batch_step(WorldBatch& batch, const StepConfig& cfg, int n_threads);

 private:
  struct Entry {
    std::shared_ptr<const MechanismModel> model;
    int pose_offset = 0, twist_offset = 0;
    bool active = true, converged = true;
    double time = 0;
    StepDiagnostics diag;
    JointReactionCache joint_cache;
    std::map<std::pair<int, int>, std::pair<double, double>> limit_cache;
    std::vector<ReactionCacheEntry> contact_cache;
  };
  std::vector<Entry> entries_;
  std::vector<double> poses_, twists_;
  std::vector<StepTrace> traces_;
};
void batch_step(WorldBatch& batch, const StepConfig& cfg, int n_threads = 0);

// ---------------------------------------------------------------- fk (fk.hpp:13-33, fk.cpp)
struct FkConfig {
  double tolerance = 1e-8;  // on |r|_inf
  int max_iters = 100;
  double lm_initial = 1e-6;  // Levenberg damping: x10 on reject, /10 on accept
};
struct FkResult {
  std::vector<Pose> poses;
  double residual_inf = 0.0;
  int iterations = 0;
  bool converged = false;
};
// Gauss-Newton with Levenberg damping on [bilateral f; coordinate - target].
// The reference solves the normal equations with Eigen's LDLT; the oracle
// uses an unblocked LLT (SPD thanks to the damping), so agreement with Eigen
// itself is to rounding, not bits.
FkResult fk_solve(const MechanismModel& m, const std::vector<std::pair<int, double>>& targets,
                  const std::vector<Pose>& initial_poses, const FkConfig& cfg = {});

}  // namespace oracle
