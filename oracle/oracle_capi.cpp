// oracle_capi.cpp — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
//
// C-ABI over the oracle, mirroring the product's kd_* surface
// (include/kamino_b200.h) with an or_ prefix so the parity tests can drive both
// implementations through the same calls.  Loaded with ctypes from tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline leg only.
#include <cstring>
#include <random>
#include <string>

#include "../include/kamino_b200.h"
#include "oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

Vec3 v3(const double* p) { return {p[0], p[1], p[2]}; }
Quat q4(const double* p) { return {p[0], p[1], p[2], p[3]}; }
std::string str(const char* s) { return s ? std::string(s) : std::string(); }

SceneDescription to_scene(const kd_scene_desc* d) {
  SceneDescription s;
  s.name = str(d->name);
  s.gravity = v3(d->gravity);
  for (int i = 0; i < d->n_bodies; ++i) {
    const kd_body_desc& b = d->bodies[i];
    SceneBody sb;
    sb.name = str(b.name);
    sb.mass = b.mass;
    for (int k = 0; k < 9; ++k) sb.inertia.m[k] = b.inertia[k];
    sb.pose.position = v3(b.position);
    sb.pose.orientation = q4(b.orientation);
    sb.twist.linear = v3(b.linear_velocity);
    sb.twist.angular = v3(b.angular_velocity);
    s.bodies.push_back(sb);
  }
  for (int i = 0; i < d->n_joints; ++i) {
    const kd_joint_desc& j = d->joints[i];
    SceneJoint sj;
    sj.name = str(j.name);
    sj.type = str(j.type);
    sj.parent = str(j.parent);
    sj.child = str(j.child);
    sj.frame_in_parent.position = v3(j.parent_position);
    sj.frame_in_parent.orientation = q4(j.parent_orientation);
    sj.frame_in_child.position = v3(j.child_position);
    sj.frame_in_child.orientation = q4(j.child_orientation);
    sj.axis = v3(j.axis);
    sj.has_limits = j.has_limits != 0;
    sj.lower = j.lower;
    sj.upper = j.upper;
    sj.kp = j.kp;
    sj.kd = j.kd;
    sj.has_target = j.has_target != 0;
    sj.target = j.target;
    sj.target_rate = j.target_rate;
    sj.armature = j.armature;
    sj.damping = j.damping;
    s.joints.push_back(sj);
  }
  for (int i = 0; i < d->n_geoms; ++i) {
    const kd_geom_desc& g = d->geoms[i];
    SceneGeom sg;
    sg.body = str(g.body);
    sg.shape = str(g.shape);
    sg.radius = g.radius;
    sg.half_extents = v3(g.half_extents);
    sg.normal = v3(g.normal);
    sg.offset = g.offset;
    sg.mu = g.mu;
    sg.restitution = g.restitution;
    s.geoms.push_back(sg);
  }
  return s;
}

StepConfig to_cfg(const kd_step_config* c) {
  StepConfig s;
  s.dt = c->dt;
  s.integrator = c->integrator == KD_INTEGRATOR_MOREAU_JEAN ? Integrator::MoreauJean
                                                              : Integrator::SemiImplicitEuler;
  s.backend = c->backend == KD_BACKEND_DENSE        ? BackendChoice::Dense
              : c->backend == KD_BACKEND_MATRIX_FREE ? BackendChoice::MatrixFree
                                                     : BackendChoice::Auto;
  s.solver.eta = c->eta;
  s.solver.rho = c->rho;
  s.solver.eps = c->eps;
  s.solver.max_iters = c->max_iters;
  s.solver.acceleration = c->acceleration != 0;
  s.solver.restart = c->restart != 0;
  s.solver.fixed_iteration_mode = c->fixed_iteration_mode != 0;
  s.cr_iters = c->cr_iters;
  s.baumgarte_beta = c->baumgarte_beta;
  s.contact_margin = c->contact_margin;
  s.impact_velocity_threshold = c->impact_velocity_threshold;
  s.bias_clamp = c->bias_clamp;
  s.limit_margin_angular = c->limit_margin_angular;
  s.limit_margin_linear = c->limit_margin_linear;
  s.warm_start = c->warm_start != 0;
  return s;
}

struct OrModel {
  std::shared_ptr<const MechanismModel> m;
  kd_model_info info;
};

kd_model_info make_info(const MechanismModel& m) {
  kd_model_info in{};
  in.n_bodies = m.n_bodies();
  in.n_joints = (int)m.joints.size();
  in.n_geoms = (int)m.geoms.size();
  in.n_bilateral_rows = m.n_bilateral_rows;
  in.n_dynamics_rows = m.n_dynamics_rows;
  in.n_loops = m.n_loops;
  int lim = 0;
  for (const JointSpec& j : m.joints) lim += j.has_limits ? 1 : 0;
  in.n_limited_joints = lim;
  int mc = 0;
  for (size_t i = 0; i < m.geoms.size(); ++i)
    for (size_t j = i + 1; j < m.geoms.size(); ++j) {
      const GeomSpec& a = m.geoms[i];
      const GeomSpec& b = m.geoms[j];
      if (a.body == b.body || (a.body == kWorld && b.body == kWorld)) continue;
      mc += (a.shape == Shape::Box || b.shape == Shape::Box) ? 4 : 1;
    }
  in.max_contacts = mc;
  in.row_capacity = m.n_bilateral_rows + m.n_dynamics_rows + 2 * lim + 3 * mc;
  return in;
}

struct OrBatch {
  std::vector<OrModel*> models;
  std::vector<int> world_model;
  WorldBatch batch;
  std::vector<int64_t> row_offset;
  int64_t total_rows = 0;
};
}  // namespace

extern "C" {

const char* or_last_error(void) { return g_err.c_str(); }

void or_step_config_default(kd_step_config* c) {
  const StepConfig s;
  c->dt = s.dt;
  c->integrator = KD_INTEGRATOR_SEMI_IMPLICIT_EULER;
  c->backend = KD_BACKEND_AUTO;
  c->eta = s.solver.eta;
  c->rho = s.solver.rho;
  c->eps = s.solver.eps;
  c->max_iters = s.solver.max_iters;
  c->acceleration = 1;
  c->restart = 1;
  c->fixed_iteration_mode = 0;
  c->cr_iters = s.cr_iters;
  c->baumgarte_beta = s.baumgarte_beta;
  c->contact_margin = s.contact_margin;
  c->impact_velocity_threshold = s.impact_velocity_threshold;
  c->bias_clamp = s.bias_clamp;
  c->limit_margin_angular = s.limit_margin_angular;
  c->limit_margin_linear = s.limit_margin_linear;
  c->warm_start = 1;
}

int or_model_build_ex(const kd_scene_desc* scene, uint32_t extensions, void** out) {
  if (!scene || !out) return fail(KD_ERR_INVALID_ARGUMENT, "null argument");
  try {
    auto* m = new OrModel;
    SceneDescription sd = to_scene(scene);
    sd.box_box = (extensions & KD_EXT_BOX_BOX) != 0;
    m->m = std::make_shared<const MechanismModel>(build_model(sd));
    m->info = make_info(*m->m);
    *out = m;
    return KD_OK;
  } catch (const ModelError& e) {
    return fail(e.code + 1, e.what());
  } catch (const std::exception& e) {
    return fail(KD_ERR_INVALID_ARGUMENT, e.what());
  }
}

int or_model_build(const kd_scene_desc* scene, void** out) { return or_model_build_ex(scene, 0, out); }

void or_model_destroy(void* m) { delete static_cast<OrModel*>(m); }

int or_model_get_info(const void* m, kd_model_info* out) {
  *out = static_cast<const OrModel*>(m)->info;
  return KD_OK;
}

int or_model_joint_layout(const void* mp, int32_t* ro, int32_t* rc, int32_t* dof, int32_t* dc) {
  const MechanismModel& m = *static_cast<const OrModel*>(mp)->m;
  for (size_t j = 0; j < m.joints.size(); ++j) {
    ro[j] = m.joint_layout[j].row_offset;
    rc[j] = m.joint_layout[j].row_count;
    dof[j] = m.joint_layout[j].dyn_offset;
    dc[j] = m.joint_layout[j].dyn_count;
  }
  return KD_OK;
}

int or_model_joint_targets(const void* mp, double* t) {
  const MechanismModel& m = *static_cast<const OrModel*>(mp)->m;
  for (size_t j = 0; j < m.joints.size(); ++j) t[j] = m.joints[j].target;
  return KD_OK;
}

static std::vector<Pose> poses_from(const MechanismModel& m, const double* p7) {
  std::vector<Pose> poses(m.n_bodies());
  for (int b = 0; b < m.n_bodies(); ++b) {
    poses[b].position = v3(p7 + 7 * b);
    poses[b].orientation = q4(p7 + 7 * b + 3);
  }
  return poses;
}

int or_joint_coordinate(const void* mp, int32_t joint, const double* poses7, double* out) {
  const MechanismModel& m = *static_cast<const OrModel*>(mp)->m;
  try {
    *out = joint_coordinate(m, joint, poses_from(m, poses7));
    return KD_OK;
  } catch (const ModelError& e) {
    return fail(e.code + 1, e.what());
  }
}

// constraint_jacobian_fd_check (constraints.hpp:98-99)
double or_fd_check(const void* mp, const double* poses7, double step) {
  const MechanismModel& m = *static_cast<const OrModel*>(mp)->m;
  return constraint_jacobian_fd_check(m, poses_from(m, poses7), step);
}

// kinetic + potential energy (stepper.hpp:86-87) of world w
int or_batch_energy(void* bp, int32_t w, double* ke, double* pe) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  const WorldState s = b->batch.extract_state(w);
  *ke = kinetic_energy(b->batch.model(w), s);
  *pe = potential_energy(b->batch.model(w), s);
  return KD_OK;
}

int or_batch_create(void* const* models, int32_t n_models, const int32_t* world_model, int32_t n_worlds,
                    void** out) {
  auto* b = new OrBatch;
  for (int i = 0; i < n_models; ++i) b->models.push_back(static_cast<OrModel*>(models[i]));
  b->row_offset.resize(n_worlds);
  for (int w = 0; w < n_worlds; ++w) {
    if (world_model[w] < 0 || world_model[w] >= n_models) {
      delete b;
      return fail(KD_ERR_INVALID_ARGUMENT, "world_model index out of range");
    }
    b->world_model.push_back(world_model[w]);
    b->batch.add_world(b->models[world_model[w]]->m);
    b->row_offset[w] = b->total_rows;
    b->total_rows += b->models[world_model[w]]->info.row_capacity;
  }
  *out = b;
  return KD_OK;
}

void or_batch_destroy(void* b) { delete static_cast<OrBatch*>(b); }

int or_batch_size(const void* bp, int32_t* nw, int64_t* pl, int64_t* tl) {
  OrBatch* b = const_cast<OrBatch*>(static_cast<const OrBatch*>(bp));
  *nw = b->batch.size();
  *pl = (int64_t)b->batch.pose_storage().size();
  *tl = (int64_t)b->batch.twist_storage().size();
  return KD_OK;
}

int or_batch_offsets(const void* bp, int32_t* po, int32_t* to) {
  const OrBatch* b = static_cast<const OrBatch*>(bp);
  for (int w = 0; w < b->batch.size(); ++w) {
    po[w] = b->batch.pose_offset(w);
    to[w] = b->batch.twist_offset(w);
  }
  return KD_OK;
}

int or_batch_set_state(void* bp, const double* poses, const double* twists, const double* time) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  if (poses) std::memcpy(b->batch.pose_storage().data(), poses, sizeof(double) * b->batch.pose_storage().size());
  if (twists)
    std::memcpy(b->batch.twist_storage().data(), twists, sizeof(double) * b->batch.twist_storage().size());
  if (time)
    for (int w = 0; w < b->batch.size(); ++w) {
      WorldState s = b->batch.extract_state(w);
      s.time = time[w];
      b->batch.insert_state(w, s);
    }
  return KD_OK;
}

int or_batch_get_state(void* bp, double* poses, double* twists, double* time) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  if (poses) std::memcpy(poses, b->batch.pose_storage().data(), sizeof(double) * b->batch.pose_storage().size());
  if (twists)
    std::memcpy(twists, b->batch.twist_storage().data(), sizeof(double) * b->batch.twist_storage().size());
  if (time)
    for (int w = 0; w < b->batch.size(); ++w) time[w] = b->batch.extract_state(w).time;
  return KD_OK;
}

int or_batch_reset_caches(void* bp) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  for (int w = 0; w < b->batch.size(); ++w) {
    WorldState s = b->batch.extract_state(w);
    s.joint_cache = JointReactionCache{};
    s.limit_cache.clear();
    s.contact_cache.clear();
    b->batch.insert_state(w, s);
  }
  return KD_OK;
}

// extract_state's caches (batch.cpp:42-44) in the kd_batch_get_caches layout.
int or_batch_get_caches(void* bp, int32_t w, double* jlam, double* jz, int32_t* jvalid, kd_limit_cache_entry* lim,
                        int32_t lcap, int32_t* nl, kd_contact_cache_entry* con, int32_t ccap, int32_t* nc) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  const WorldState s = b->batch.extract_state(w);
  if (jvalid) *jvalid = s.joint_cache.valid ? 1 : 0;
  for (size_t k = 0; k < s.joint_cache.lambda.size(); ++k) {
    if (jlam) jlam[k] = s.joint_cache.lambda[k];
    if (jz) jz[k] = s.joint_cache.z[k];
  }
  int k = 0;
  for (const auto& e : s.limit_cache) {
    if (lim && k < lcap) lim[k] = kd_limit_cache_entry{e.first.first, e.first.second, e.second.first, e.second.second};
    ++k;
  }
  if (nl) *nl = k;
  const int n = (int)s.contact_cache.size();
  if (nc) *nc = n;
  for (int c = 0; c < n && con && c < ccap; ++c) {
    const ReactionCacheEntry& e = s.contact_cache[c];
    con[c].geom_a = e.geom_a;
    con[c].geom_b = e.geom_b;
    const double p[3] = {e.position.x, e.position.y, e.position.z};
    const double i3[3] = {e.impulse.x, e.impulse.y, e.impulse.z};
    const double d3[3] = {e.dual.x, e.dual.y, e.dual.z};
    for (int d = 0; d < 3; ++d) {
      con[c].position[d] = p[d];
      con[c].impulse[d] = i3[d];
      con[c].dual[d] = d3[d];
    }
  }
  return (k > lcap || n > ccap) ? KD_ERR_CAPACITY : KD_OK;
}

// The reference bench's initial-twist jitter (tools/main.cpp:199-211): one
// std::mt19937_64(seed) stream and normal_distribution<double>(0, sigma) for
// the whole batch, world-major, per body, k = 0..2: linear[k] then angular[k];
// applied only when seed != 0.  (The bench's reference arm uses this, so it
// never loads the product library.)
int or_bench_jitter(uint64_t seed, double sigma, int32_t n_worlds, const int32_t* n_bodies, double* twists6) {
  if (!n_bodies || !twists6) return KD_ERR_INVALID_ARGUMENT;
  if (seed == 0) return KD_OK;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> jitter(0.0, sigma);
  int64_t off = 0;
  for (int w = 0; w < n_worlds; ++w)
    for (int b = 0; b < n_bodies[w]; ++b, off += 6)
      for (int k = 0; k < 3; ++k) {
        twists6[off + k] += jitter(rng);
        twists6[off + 3 + k] += jitter(rng);
      }
  return KD_OK;
}

int or_batch_set_active(void* bp, const uint8_t* active) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  for (int w = 0; w < b->batch.size(); ++w) b->batch.set_active(w, active[w] != 0);
  return KD_OK;
}

int or_batch_set_trace(void* bp, int32_t on) {
  static_cast<OrBatch*>(bp)->batch.record_trace = on != 0;
  return KD_OK;
}

int or_batch_step(void* bp, const kd_step_config* cfg, int32_t n_steps, int32_t n_threads) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  try {
    const StepConfig c = to_cfg(cfg);
    for (int k = 0; k < n_steps; ++k) batch_step(b->batch, c, n_threads);
    return KD_OK;
  } catch (const std::exception& e) {
    return fail(KD_ERR_SPD_FAILURE, e.what());
  }
}

int or_batch_get_diagnostics(void* bp, kd_step_diag* out) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  for (int w = 0; w < b->batch.size(); ++w) {
    const StepDiagnostics& d = b->batch.diagnostics(w);
    kd_step_diag& o = out[w];
    o.iterations = d.solver.iterations;
    o.restarts = d.solver.restarts;
    o.converged = d.solver.converged ? 1 : 0;
    o.cr_breakdown = d.solver.cr_breakdown ? 1 : 0;
    o.cr_iterations = d.solver.cr_iterations;
    o.r_p = d.solver.r_p;
    o.r_d = d.solver.r_d;
    o.r_c = d.solver.r_c;
    o.n_rows = d.n_rows;
    o.contact_count = d.contact_count;
    o.first_contact_row = d.first_contact_row;
    o.n_limits = d.n_limits;
    o.f_inf = d.f_inf;
    o.kkt_momentum_inf = d.kkt_momentum_inf;
    o.bilateral_velocity_inf = d.bilateral_velocity_inf;
  }
  return KD_OK;
}

int or_batch_row_offsets(const void* bp, int64_t* ro, int64_t* total) {
  const OrBatch* b = static_cast<const OrBatch*>(bp);
  for (size_t w = 0; w < b->row_offset.size(); ++w) ro[w] = b->row_offset[w];
  *total = b->total_rows;
  return KD_OK;
}

int or_batch_get_impulses(void* bp, double* out) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  for (int w = 0; w < b->batch.size(); ++w) {
    const Vec& imp = b->batch.diagnostics(w).impulses;
    for (size_t i = 0; i < imp.size(); ++i) out[b->row_offset[w] + (int64_t)i] = imp[i];
  }
  return KD_OK;
}

// Combined-residual history of the last traced step: out[w*cap + i], -1 padded.
int or_batch_get_history(void* bp, int32_t cap, double* out) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  for (int w = 0; w < b->batch.size(); ++w) {
    const auto& h = b->batch.traces()[w].history;
    for (int i = 0; i < cap; ++i) out[(int64_t)w * cap + i] = i < (int)h.size() ? h[i] : -1.0;
  }
  return KD_OK;
}

int or_batch_dump_rows(void* bp, int32_t w, kd_row_dump* out, int32_t cap, int32_t* n_rows) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  const StepTrace& t = b->batch.traces()[w];
  const ConstraintSet& cs = t.cs;
  *n_rows = cs.n_rows;
  if (cs.n_rows > cap) return fail(KD_ERR_CAPACITY, "dump capacity too small");
  std::vector<int> kind(cs.n_rows, 0);
  for (const ConeGroup& g : cs.cones.groups)
    for (int k = 0; k < g.dim; ++k)
      kind[g.begin + k] = g.kind == ConeKind::Bilateral ? 0 : (g.kind == ConeKind::Nonnegative ? 1 : 2);
  for (int r = 0; r < cs.n_rows; ++r) {
    kd_row_dump& o = out[r];
    std::memset(&o, 0, sizeof(o));
    o.body_a = cs.rows[r].body_a;
    o.body_b = cs.rows[r].body_b;
    o.kind = kind[r];
    for (int k = 0; k < 6; ++k) {
      o.block_a[k] = cs.rows[r].block_a[k];
      o.block_b[k] = cs.rows[r].block_b[k];
    }
    o.bias = cs.bias[r];
    o.reg = cs.reg[r];
    if (!t.precond.scale.empty()) {
      o.scale = t.precond.scale[r];
      o.vf_scaled = t.v_f_scaled[r];
      o.lambda = t.lambda_scaled[r];
      o.z = t.z_scaled[r];
    }
  }
  return KD_OK;
}

int or_batch_dump_contacts(void* bp, int32_t w, int32_t* geoms, double* data9, int32_t cap, int32_t* nc) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  const ConstraintSet& cs = b->batch.traces()[w].cs;
  *nc = (int)cs.contacts.size();
  if (*nc > cap) return fail(KD_ERR_CAPACITY, "dump capacity too small");
  for (int c = 0; c < *nc; ++c) {
    const ContactPoint& cp = cs.contacts[c];
    geoms[2 * c] = cp.geom_a;
    geoms[2 * c + 1] = cp.geom_b;
    double* d = data9 + 9 * c;
    d[0] = cp.position.x;
    d[1] = cp.position.y;
    d[2] = cp.position.z;
    d[3] = cp.normal.x;
    d[4] = cp.normal.y;
    d[5] = cp.normal.z;
    d[6] = cp.depth;
    d[7] = cp.mu;
    d[8] = cp.restitution;
  }
  return KD_OK;
}

int or_batch_dump_limits(void* bp, int32_t w, int32_t* keys2, int32_t cap, int32_t* nl) {
  OrBatch* b = static_cast<OrBatch*>(bp);
  const ConstraintSet& cs = b->batch.traces()[w].cs;
  *nl = cs.n_limits;
  if (*nl > cap) return fail(KD_ERR_CAPACITY, "dump capacity too small");
  for (int k = 0; k < *nl; ++k) {
    keys2[2 * k] = cs.limit_keys[k].first;
    keys2[2 * k + 1] = cs.limit_keys[k].second;
  }
  return KD_OK;
}

// fk_solve (fk.cpp) on one world: poses7 in/out (nb x 7), targets (joint, value).
int or_fk_solve(const void* mp, const int32_t* joints, const double* values, int32_t n_targets, double* poses7,
                double tol, int32_t max_iters, double lm_initial, double* residual_inf, int32_t* iterations,
                int32_t* converged) {
  const MechanismModel& m = *static_cast<const OrModel*>(mp)->m;
  std::vector<std::pair<int, double>> t;
  for (int k = 0; k < n_targets; ++k) t.push_back({joints[k], values[k]});
  FkConfig cfg;
  cfg.tolerance = tol;
  cfg.max_iters = max_iters;
  cfg.lm_initial = lm_initial;
  try {
    const FkResult r = fk_solve(m, t, poses_from(m, poses7), cfg);
    for (int b = 0; b < m.n_bodies(); ++b) {
      const Pose& p = r.poses[b];
      double* o = poses7 + 7 * b;
      o[0] = p.position.x, o[1] = p.position.y, o[2] = p.position.z;
      o[3] = p.orientation.w, o[4] = p.orientation.x, o[5] = p.orientation.y, o[6] = p.orientation.z;
    }
    *residual_inf = r.residual_inf;
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    return KD_OK;
  } catch (const ModelError& e) {
    return fail(e.code + 1, e.what());
  }
}

}  // extern "C"
