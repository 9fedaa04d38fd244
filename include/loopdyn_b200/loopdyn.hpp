// loopdyn_b200/loopdyn.hpp — header-only C++17 drop-in for the reference
// loopdyn solver/world/step API (/root/reference/proj/include/loopdyn), backed
// by the B200 C-ABI (include/kamino_b200.h, libkamino_b200.so).
//
// Same names and semantics as the reference:
//   SceneDescription / SceneBody / SceneJoint / SceneGeom   (scene.hpp:15-72)
//   MechanismModel build_model(const SceneDescription&)     (model.hpp:117)
//   double joint_coordinate(model, joint, poses)            (model.hpp:130)
//   StepConfig / PadmmConfig / Integrator / BackendChoice   (stepper.hpp:16-34, padmm.hpp:8-17)
//   WorldState / StepDiagnostics / SolveDiagnostics         (stepper.hpp:49-74, padmm.hpp:19-28)
//   WorldBatch {add_world, extract_state, insert_state, set_active, active,
//               converged, diagnostics, pose_offset, twist_offset,
//               pose_storage, twist_storage}                (batch.hpp:14-54)
//   void batch_step(WorldBatch&, const StepConfig&, int n_threads = 0)  (batch.hpp:58)
//   StepDiagnostics step(const MechanismModel&, WorldState&, const StepConfig&) (stepper.hpp:84)
// Errors: ModelError{Code} on build/joint-type errors (model.hpp:76-94),
// std::runtime_error for SPD failure / CUDA errors (delassus.cpp:209-215).
//
// Differences forced by the boundary: value types are plain arrays instead of
// Eigen (Eigen is not part of this build); warm-start caches stay on the device
// (extract_state/insert_state move poses, twists and time); the device batch
// is materialised on first use, after which add_world is an error.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../kamino_b200.h"

namespace loopdyn_b200 {

using Vec3 = std::array<double, 3>;
using Quat = std::array<double, 4>;  // [w, x, y, z]
using Mat3 = std::array<double, 9>;  // row-major

struct Pose {
  Vec3 position{0, 0, 0};
  Quat orientation{1, 0, 0, 0};
};
struct Twist {
  Vec3 linear{0, 0, 0};
  Vec3 angular{0, 0, 0};
};

// ---- scene (scene.hpp:15-72)
struct SceneBody {
  std::string name;
  double mass = 1.0;
  Mat3 inertia{1, 0, 0, 0, 1, 0, 0, 0, 1};
  Pose pose;
  Twist twist;
};
struct SceneJoint {
  std::string name, type, parent, child;
  Pose frame_in_parent, frame_in_child;
  Vec3 axis{0, 0, 1};
  std::optional<std::pair<double, double>> limits;
  double kp = 0, kd = 0;
  std::optional<double> target;
  double target_rate = 0, armature = 0, damping = 0;
};
struct SceneGeom {
  std::string body, shape;
  double radius = 0;
  Vec3 half_extents{0, 0, 0};
  Vec3 normal{0, 0, 1};
  double offset = 0, mu = 0, restitution = 0;
};
struct SceneConfig {
  std::optional<double> dt;
  std::optional<std::string> integrator, backend;
  std::optional<double> beta, rho, eta, eps;
  std::optional<int> max_iters, cr_iters;
};
struct SceneDescription {
  std::string name = "scene";
  Vec3 gravity{0, 0, -9.81};
  std::vector<SceneBody> bodies;
  std::vector<SceneJoint> joints;
  std::vector<SceneGeom> geoms;
  SceneConfig config;
  uint32_t extensions = 0;  // KD_EXT_* opt-in extensions (no reference counterpart)
};

// ---- errors (model.hpp:76-94)
class ModelError : public std::runtime_error {
 public:
  enum class Code {
    InvalidReference, NonUnitAxis, BadInertia, BadLimits, UnsupportedOnJointType, BadGeometry,
    UnsupportedCollisionPair, WrongJointType, DuplicateName,
  };
  ModelError(Code code, const std::string& what) : std::runtime_error(what), code_(code) {}
  Code code() const { return code_; }

 private:
  Code code_;
};

namespace detail {
[[noreturn]] inline void raise(int status) {
  const std::string msg = kd_last_error();
  if (status >= KD_ERR_MODEL_INVALID_REFERENCE && status <= KD_ERR_MODEL_DUPLICATE_NAME)
    throw ModelError(static_cast<ModelError::Code>(status - 1), msg);
  throw std::runtime_error("kamino_b200 error " + std::to_string(status) + ": " + msg);
}
inline void check(int status) {
  if (status != KD_OK) raise(status);
}
template <class T, std::size_t N>
void copy(double (&dst)[N], const std::array<T, N>& src) {
  for (std::size_t i = 0; i < N; ++i) dst[i] = src[i];
}
}  // namespace detail

// ---- model (model.hpp:97-130)
class MechanismModel {
 public:
  explicit MechanismModel(const SceneDescription& s) : scene_(s) {
    std::vector<kd_body_desc> b(s.bodies.size());
    std::vector<kd_joint_desc> j(s.joints.size());
    std::vector<kd_geom_desc> g(s.geoms.size());
    for (std::size_t i = 0; i < b.size(); ++i) {
      const SceneBody& sb = s.bodies[i];
      b[i] = kd_body_desc{};
      b[i].name = sb.name.c_str();
      b[i].mass = sb.mass;
      detail::copy(b[i].inertia, sb.inertia);
      detail::copy(b[i].position, sb.pose.position);
      detail::copy(b[i].orientation, sb.pose.orientation);
      detail::copy(b[i].linear_velocity, sb.twist.linear);
      detail::copy(b[i].angular_velocity, sb.twist.angular);
    }
    for (std::size_t i = 0; i < j.size(); ++i) {
      const SceneJoint& sj = s.joints[i];
      j[i] = kd_joint_desc{};
      j[i].name = sj.name.c_str();
      j[i].type = sj.type.c_str();
      j[i].parent = sj.parent.c_str();
      j[i].child = sj.child.c_str();
      detail::copy(j[i].parent_position, sj.frame_in_parent.position);
      detail::copy(j[i].parent_orientation, sj.frame_in_parent.orientation);
      detail::copy(j[i].child_position, sj.frame_in_child.position);
      detail::copy(j[i].child_orientation, sj.frame_in_child.orientation);
      detail::copy(j[i].axis, sj.axis);
      j[i].has_limits = sj.limits.has_value();
      if (sj.limits) {
        j[i].lower = sj.limits->first;
        j[i].upper = sj.limits->second;
      }
      j[i].kp = sj.kp;
      j[i].kd = sj.kd;
      j[i].has_target = sj.target.has_value();
      j[i].target = sj.target.value_or(0.0);
      j[i].target_rate = sj.target_rate;
      j[i].armature = sj.armature;
      j[i].damping = sj.damping;
    }
    for (std::size_t i = 0; i < g.size(); ++i) {
      const SceneGeom& sg = s.geoms[i];
      g[i] = kd_geom_desc{};
      g[i].body = sg.body.c_str();
      g[i].shape = sg.shape.c_str();
      g[i].radius = sg.radius;
      detail::copy(g[i].half_extents, sg.half_extents);
      detail::copy(g[i].normal, sg.normal);
      g[i].offset = sg.offset;
      g[i].mu = sg.mu;
      g[i].restitution = sg.restitution;
    }
    kd_scene_desc d{};
    d.name = s.name.c_str();
    detail::copy(d.gravity, s.gravity);
    d.n_bodies = (int32_t)b.size();
    d.bodies = b.data();
    d.n_joints = (int32_t)j.size();
    d.joints = j.data();
    d.n_geoms = (int32_t)g.size();
    d.geoms = g.data();
    kd_model* m = nullptr;
    detail::check(kd_model_build_ex(&d, s.extensions, &m));
    handle_.reset(m, kd_model_destroy);
    detail::check(kd_model_get_info(m, &info_));
  }
  const kd_model* handle() const { return handle_.get(); }
  const SceneDescription& scene() const { return scene_; }
  int n_bodies() const { return info_.n_bodies; }
  int velocity_dim() const { return 6 * info_.n_bodies; }
  int n_bilateral_rows() const { return info_.n_bilateral_rows; }
  int n_dynamics_rows() const { return info_.n_dynamics_rows; }
  int n_loops() const { return info_.n_loops; }
  const kd_model_info& info() const { return info_; }

 private:
  SceneDescription scene_;
  std::shared_ptr<kd_model> handle_;
  kd_model_info info_{};
};

inline MechanismModel build_model(const SceneDescription& s) { return MechanismModel(s); }

inline double joint_coordinate(const MechanismModel& m, int joint, const std::vector<Pose>& poses) {
  std::vector<double> p7;
  for (const Pose& p : poses) {
    p7.insert(p7.end(), p.position.begin(), p.position.end());
    p7.insert(p7.end(), p.orientation.begin(), p.orientation.end());
  }
  double out = 0;
  detail::check(kd_joint_coordinate(m.handle(), joint, p7.data(), &out));
  return out;
}

// ---- configuration (stepper.hpp:16-34, padmm.hpp:8-17)
enum class Integrator { SemiImplicitEuler, MoreauJean };
enum class BackendChoice { Dense, MatrixFree, Auto };
struct PadmmConfig {
  double eta = 1e-6, rho = 0.1, eps = 1e-6;
  int max_iters = 200;
  bool acceleration = true, restart = true, fixed_iteration_mode = false;
};
struct StepConfig {
  double dt = 1.0 / 240.0;
  Integrator integrator = Integrator::SemiImplicitEuler;
  BackendChoice backend = BackendChoice::Auto;
  PadmmConfig solver;
  int cr_iters = 9;
  double baumgarte_beta = 0.2, contact_margin = 0.01, impact_velocity_threshold = 0.1, bias_clamp = 10.0,
         limit_margin_angular = 0.01, limit_margin_linear = 0.001;
  bool warm_start = true;

  kd_step_config to_c() const {
    kd_step_config c{};
    c.dt = dt;
    c.integrator = integrator == Integrator::MoreauJean ? KD_INTEGRATOR_MOREAU_JEAN
                                                        : KD_INTEGRATOR_SEMI_IMPLICIT_EULER;
    c.backend = backend == BackendChoice::Dense        ? KD_BACKEND_DENSE
                : backend == BackendChoice::MatrixFree ? KD_BACKEND_MATRIX_FREE
                                                       : KD_BACKEND_AUTO;
    c.eta = solver.eta;
    c.rho = solver.rho;
    c.eps = solver.eps;
    c.max_iters = solver.max_iters;
    c.acceleration = solver.acceleration;
    c.restart = solver.restart;
    c.fixed_iteration_mode = solver.fixed_iteration_mode;
    c.cr_iters = cr_iters;
    c.baumgarte_beta = baumgarte_beta;
    c.contact_margin = contact_margin;
    c.impact_velocity_threshold = impact_velocity_threshold;
    c.bias_clamp = bias_clamp;
    c.limit_margin_angular = limit_margin_angular;
    c.limit_margin_linear = limit_margin_linear;
    c.warm_start = warm_start;
    return c;
  }
};

// apply_scene_config (stepper.cpp:74-95)
inline void apply_scene_config(StepConfig& c, const SceneConfig& o) {
  if (o.dt) c.dt = *o.dt;
  if (o.integrator) c.integrator = *o.integrator == "moreau" ? Integrator::MoreauJean : Integrator::SemiImplicitEuler;
  if (o.backend)
    c.backend = *o.backend == "dense" ? BackendChoice::Dense
                : *o.backend == "sparse" ? BackendChoice::MatrixFree
                                         : BackendChoice::Auto;
  if (o.beta) c.baumgarte_beta = *o.beta;
  if (o.rho) c.solver.rho = *o.rho;
  if (o.eta) c.solver.eta = *o.eta;
  if (o.eps) c.solver.eps = *o.eps;
  if (o.max_iters) c.solver.max_iters = *o.max_iters;
  if (o.cr_iters) c.cr_iters = *o.cr_iters;
}

struct SolveDiagnostics {
  int iterations = 0;
  double r_p = 0, r_d = 0, r_c = 0;
  int restarts = 0;
  bool converged = true;
  long cr_iterations = 0;
  bool cr_breakdown = false;
};
struct StepDiagnostics {
  SolveDiagnostics solver;
  int n_rows = 0, contact_count = 0, first_contact_row = 0;
  std::vector<double> impulses;
  double f_inf = 0, kkt_momentum_inf = 0, bilateral_velocity_inf = 0;
};
// Warm-start caches (stepper.hpp:38-47, contacts.hpp:32-38), physical scale.
struct JointReactionCache {
  std::vector<double> lambda, z;
  bool valid = false;
};
struct LimitReactionCache {
  std::map<std::pair<int, int>, std::pair<double, double>> entries;  // (joint, bound) -> (lambda, z)
};
struct ReactionCacheEntry {
  int geom_a = -1, geom_b = -1;
  std::array<double, 3> position{}, impulse{}, dual{};  // impulse / dual in the contact frame (n, t1, t2)
};
struct ReactionCache {
  std::vector<ReactionCacheEntry> entries;
};
struct WorldState {
  std::vector<Pose> poses;
  std::vector<Twist> twists;
  double time = 0.0;
  JointReactionCache joint_cache;
  LimitReactionCache limit_cache;
  ReactionCache contact_cache;
};

inline WorldState initial_state(const MechanismModel& m) {
  WorldState s;
  for (const SceneBody& b : m.scene().bodies) {
    Pose p = b.pose;
    double n = 0;
    for (double q : p.orientation) n += q * q;
    n = std::sqrt(n);
    for (double& q : p.orientation) q /= n;
    s.poses.push_back(p);
    s.twists.push_back(b.twist);
  }
  return s;
}

// ---- batch (batch.hpp:14-58)
class WorldBatch {
 public:
  explicit WorldBatch(int device = 0) : device_(device) {}
  int add_world(std::shared_ptr<const MechanismModel> model) { return add_world(model, initial_state(*model)); }
  int add_world(std::shared_ptr<const MechanismModel> model, const WorldState& state) {
    if (batch_) throw std::runtime_error("add_world after the batch was materialised on the device");
    int idx = -1;
    for (std::size_t i = 0; i < models_.size(); ++i)
      if (models_[i] == model) idx = (int)i;
    if (idx < 0) {
      models_.push_back(model);
      idx = (int)models_.size() - 1;
    }
    world_model_.push_back(idx);
    init_.push_back(state);
    return (int)world_model_.size() - 1;
  }
  int size() const { return (int)world_model_.size(); }
  const MechanismModel& model(int w) const { return *models_[world_model_[w]]; }

  WorldState extract_state(int w) {
    sync_host();
    const int nb = model(w).n_bodies();
    WorldState s;
    for (int b = 0; b < nb; ++b) {
      const double* p = &poses_[pose_off_[w] + 7 * b];
      const double* t = &twists_[twist_off_[w] + 6 * b];
      s.poses.push_back(Pose{{p[0], p[1], p[2]}, {p[3], p[4], p[5], p[6]}});
      s.twists.push_back(Twist{{t[0], t[1], t[2]}, {t[3], t[4], t[5]}});
    }
    s.time = time_[w];
    get_caches(w, s);
    return s;
  }
  // extract_state's cache part (batch.cpp:42-44)
  void get_caches(int w, WorldState& s) {
    ensure();
    int32_t jl = 0, jv = 0, nl = 0, nc = 0;
    detail::check(kd_batch_get_cache_sizes(batch_.get(), w, &jl, &jv, &nl, &nc));
    s.joint_cache.lambda.assign(jl, 0.0);
    s.joint_cache.z.assign(jl, 0.0);
    std::vector<kd_limit_cache_entry> lim(std::max(1, nl));
    std::vector<kd_contact_cache_entry> con(std::max(1, nc));
    int32_t jv2 = 0, nl2 = 0, nc2 = 0;
    detail::check(kd_batch_get_caches(batch_.get(), w, s.joint_cache.lambda.data(), s.joint_cache.z.data(), &jv2,
                                      lim.data(), (int32_t)lim.size(), &nl2, con.data(), (int32_t)con.size(), &nc2));
    s.joint_cache.valid = jv2 != 0;
    s.limit_cache.entries.clear();
    for (int k = 0; k < nl2; ++k) s.limit_cache.entries[{lim[k].joint, lim[k].bound}] = {lim[k].lambda, lim[k].z};
    s.contact_cache.entries.clear();
    for (int k = 0; k < nc2; ++k) {
      ReactionCacheEntry e;
      e.geom_a = con[k].geom_a;
      e.geom_b = con[k].geom_b;
      for (int d = 0; d < 3; ++d) e.position[d] = con[k].position[d], e.impulse[d] = con[k].impulse[d],
                                  e.dual[d] = con[k].dual[d];
      s.contact_cache.entries.push_back(e);
    }
  }
  // insert_state's cache part (batch.cpp:68-70)
  void set_caches(int w, const WorldState& s) {
    ensure();
    std::vector<kd_limit_cache_entry> lim;
    for (const auto& [key, val] : s.limit_cache.entries)
      lim.push_back(kd_limit_cache_entry{key.first, key.second, val.first, val.second});
    std::vector<kd_contact_cache_entry> con;
    for (const ReactionCacheEntry& e : s.contact_cache.entries) {
      kd_contact_cache_entry c{};
      c.geom_a = e.geom_a;
      c.geom_b = e.geom_b;
      for (int d = 0; d < 3; ++d) c.position[d] = e.position[d], c.impulse[d] = e.impulse[d], c.dual[d] = e.dual[d];
      con.push_back(c);
    }
    const bool jok = s.joint_cache.z.size() == s.joint_cache.lambda.size();
    detail::check(kd_batch_set_caches(batch_.get(), w, s.joint_cache.lambda.data(), s.joint_cache.z.data(),
                                      jok ? (int32_t)s.joint_cache.lambda.size() : -1, s.joint_cache.valid ? 1 : 0,
                                      lim.data(), (int32_t)lim.size(), con.data(), (int32_t)con.size()));
  }
  void insert_state(int w, const WorldState& s) {
    sync_host();
    for (int b = 0; b < model(w).n_bodies(); ++b) {
      double* p = &poses_[pose_off_[w] + 7 * b];
      double* t = &twists_[twist_off_[w] + 6 * b];
      for (int k = 0; k < 3; ++k) p[k] = s.poses[b].position[k];
      for (int k = 0; k < 4; ++k) p[3 + k] = s.poses[b].orientation[k];
      for (int k = 0; k < 3; ++k) t[k] = s.twists[b].linear[k], t[3 + k] = s.twists[b].angular[k];
    }
    time_[w] = s.time;
    detail::check(kd_batch_set_state(batch_.get(), poses_.data(), twists_.data(), time_.data()));
    set_caches(w, s);
  }
  void set_active(int w, bool a) {
    ensure();
    active_[w] = a ? 1 : 0;
    detail::check(kd_batch_set_active(batch_.get(), active_.data()));
  }
  bool active(int w) {
    ensure();
    return active_[w] != 0;
  }
  bool converged(int w) { return diagnostics(w).solver.converged; }
  StepDiagnostics diagnostics(int w) {
    ensure();
    std::vector<kd_step_diag> d(size());
    detail::check(kd_batch_get_diagnostics(batch_.get(), d.data()));
    std::vector<double> imp((std::size_t)std::max<int64_t>(1, total_rows_));
    detail::check(kd_batch_get_impulses(batch_.get(), imp.data()));
    StepDiagnostics o;
    const kd_step_diag& x = d[w];
    o.solver = SolveDiagnostics{x.iterations, x.r_p, x.r_d, x.r_c, x.restarts, x.converged != 0,
                                (long)x.cr_iterations, x.cr_breakdown != 0};
    o.n_rows = x.n_rows;
    o.contact_count = x.contact_count;
    o.first_contact_row = x.first_contact_row;
    o.impulses.assign(imp.begin() + row_off_[w], imp.begin() + row_off_[w] + x.n_rows);
    o.f_inf = x.f_inf;
    o.kkt_momentum_inf = x.kkt_momentum_inf;
    o.bilateral_velocity_inf = x.bilateral_velocity_inf;
    return o;
  }
  int pose_offset(int w) {
    ensure();
    return pose_off_[w];
  }
  int twist_offset(int w) {
    ensure();
    return twist_off_[w];
  }
  const std::vector<double>& pose_storage() {
    sync_host();
    return poses_;
  }
  const std::vector<double>& twist_storage() {
    sync_host();
    return twists_;
  }
  kd_batch* handle() {
    ensure();
    return batch_.get();
  }
  friend void batch_step(WorldBatch& batch, const StepConfig& config, int n_threads);

 private:
  void ensure() {
    if (batch_) return;
    std::vector<const kd_model*> hs;
    for (const auto& m : models_) hs.push_back(m->handle());
    kd_batch* b = nullptr;
    detail::check(kd_batch_create(device_, hs.data(), (int32_t)hs.size(), world_model_.data(), size(), &b));
    batch_.reset(b, kd_batch_destroy);
    const int n = size();
    pose_off_.assign(n, 0);
    twist_off_.assign(n, 0);
    row_off_.assign(n, 0);
    detail::check(kd_batch_offsets(b, pose_off_.data(), twist_off_.data()));
    detail::check(kd_batch_row_offsets(b, row_off_.data(), &total_rows_));
    int32_t nw = 0;
    int64_t pl = 0, tl = 0;
    detail::check(kd_batch_size(b, &nw, &pl, &tl));
    poses_.assign(pl, 0.0);
    twists_.assign(tl, 0.0);
    time_.assign(n, 0.0);
    active_.assign(n, 1);
    for (int w = 0; w < n; ++w) {
      const WorldState& s = init_[w];
      for (int k = 0; k < model(w).n_bodies(); ++k) {
        double* p = &poses_[pose_off_[w] + 7 * k];
        double* t = &twists_[twist_off_[w] + 6 * k];
        for (int q = 0; q < 3; ++q) p[q] = s.poses[k].position[q];
        for (int q = 0; q < 4; ++q) p[3 + q] = s.poses[k].orientation[q];
        for (int q = 0; q < 3; ++q) t[q] = s.twists[k].linear[q], t[3 + q] = s.twists[k].angular[q];
      }
      time_[w] = s.time;
    }
    detail::check(kd_batch_set_state(b, poses_.data(), twists_.data(), time_.data()));
    host_valid_ = true;
    for (int w = 0; w < n; ++w) set_caches(w, init_[w]);
  }
  void sync_host() {
    ensure();
    if (host_valid_) return;
    detail::check(kd_batch_get_state(batch_.get(), poses_.data(), twists_.data(), time_.data()));
    host_valid_ = true;
  }

  int device_;
  std::vector<std::shared_ptr<const MechanismModel>> models_;
  std::vector<int32_t> world_model_;
  std::vector<WorldState> init_;
  std::shared_ptr<kd_batch> batch_;
  std::vector<int32_t> pose_off_, twist_off_;
  std::vector<int64_t> row_off_;
  int64_t total_rows_ = 0;
  std::vector<double> poses_, twists_, time_;
  std::vector<uint8_t> active_;
  bool host_valid_ = false;
};

// batch_step (batch.hpp:58): every active world, one step on the device;
// n_threads is accepted for signature parity and ignored.
inline void batch_step(WorldBatch& batch, const StepConfig& config, int n_threads = 0) {
  (void)n_threads;
  const kd_step_config c = config.to_c();
  detail::check(kd_batch_step(batch.handle(), &c, 1));
  batch.host_valid_ = false;
}

// step (stepper.hpp:84) for one world: a one-world device batch that starts
// from `state` including its warm-start caches (gather_warmstart,
// stepper.cpp:19-46), and writes the new state and caches back (store_caches,
// stepper.cpp:48-70).  For many worlds use WorldBatch; this exists for drop-in
// completeness.  `scratch` (optional) keeps the one-world batch between calls.
inline StepDiagnostics step(const std::shared_ptr<const MechanismModel>& model, WorldState& state,
                            const StepConfig& config, WorldBatch* scratch = nullptr) {
  WorldBatch local;
  WorldBatch& b = scratch ? *scratch : local;
  if (b.size() == 0) b.add_world(model, state);
  else b.insert_state(0, state);
  batch_step(b, config);
  state = b.extract_state(0);
  return b.diagnostics(0);
}
// The reference signature, step(const MechanismModel&, WorldState&, const
// StepConfig&) (stepper.hpp:84): the model is borrowed for the call.
inline StepDiagnostics step(const MechanismModel& model, WorldState& state, const StepConfig& config) {
  return step(std::shared_ptr<const MechanismModel>(&model, [](const MechanismModel*) {}), state, config);
}

}  // namespace loopdyn_b200
