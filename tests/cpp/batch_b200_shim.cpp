// The reference-side shim of INTEGRATION.md §3 (proj/src/batch_b200.cpp in a
// maintainer's tree): loopdyn::batch_step forwarded to a device batch whose
// storage layout equals WorldBatch's (batch.hpp:41-42).  Compiled here against
// tests/cpp/ref_stub (the declarations it needs) and linked with
// libkamino_b200.so by tests/test_cpp_api.py; main() steps a free-falling
// sphere through it when a GPU is present.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "kamino_b200.h"
#include "loopdyn/batch.hpp"

namespace loopdyn {
void batch_step_b200(WorldBatch& batch, const StepConfig& cfg, kd_batch* dev) {
  // storage layouts are identical (batch.hpp:41-42): copy, step, copy back
  if (kd_batch_set_state(dev, batch.pose_storage().data(), batch.twist_storage().data(), nullptr) != KD_OK)
    throw std::runtime_error(kd_last_error());
  kd_step_config c;
  kd_step_config_default(&c);
  c.dt = cfg.dt;
  c.integrator = cfg.integrator == Integrator::MoreauJean ? KD_INTEGRATOR_MOREAU_JEAN : KD_INTEGRATOR_SEMI_IMPLICIT_EULER;
  c.backend = cfg.backend == BackendChoice::Dense        ? KD_BACKEND_DENSE
              : cfg.backend == BackendChoice::MatrixFree ? KD_BACKEND_MATRIX_FREE
                                                         : KD_BACKEND_AUTO;
  c.eta = cfg.solver.eta;
  c.rho = cfg.solver.rho;
  c.eps = cfg.solver.eps;
  c.max_iters = cfg.solver.max_iters;
  c.acceleration = cfg.solver.acceleration;
  c.restart = cfg.solver.restart;
  c.fixed_iteration_mode = cfg.solver.fixed_iteration_mode;
  c.cr_iters = cfg.cr_iters;
  c.baumgarte_beta = cfg.baumgarte_beta;
  c.contact_margin = cfg.contact_margin;
  c.impact_velocity_threshold = cfg.impact_velocity_threshold;
  c.bias_clamp = cfg.bias_clamp;
  c.limit_margin_angular = cfg.limit_margin_angular;
  c.limit_margin_linear = cfg.limit_margin_linear;
  c.warm_start = cfg.warm_start;
  if (kd_batch_step(dev, &c, 1) != KD_OK) throw std::runtime_error(kd_last_error());
  if (kd_batch_get_state(dev, const_cast<double*>(batch.pose_storage().data()),
                         const_cast<double*>(batch.twist_storage().data()), nullptr) != KD_OK)
    throw std::runtime_error(kd_last_error());
}
}  // namespace loopdyn

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  kd_body_desc body{};
  body.name = "ball";
  body.mass = 1.0;
  body.inertia[0] = body.inertia[4] = body.inertia[8] = 0.1;
  body.orientation[0] = 1.0;
  kd_scene_desc scene{};
  scene.name = "freefall";
  scene.gravity[2] = -9.81;
  scene.n_bodies = 1;
  scene.bodies = &body;
  kd_model* m = nullptr;
  if (kd_model_build(&scene, &m) != KD_OK) return 1;
  if (!gpu) {
    kd_model_destroy(m);
    std::printf("shim compiled and linked\n");
    return 0;
  }
  const int32_t wm = 0;
  kd_batch* dev = nullptr;
  if (kd_batch_create(0, &m, 1, &wm, 1, &dev) != KD_OK) return 2;
  loopdyn::WorldBatch batch({0, 0, 0, 1, 0, 0, 0}, {0, 0, 0, 0, 0, 0});
  loopdyn::StepConfig cfg;
  for (int k = 0; k < 240; ++k) loopdyn::batch_step_b200(batch, cfg, dev);
  const double vz = batch.twist_storage()[2], z = batch.pose_storage()[2];
  const double n = 240, g = 9.81, dt = cfg.dt;  // acceptance #7: closed-form free fall
  const bool ok = std::abs(vz + g * n * dt) < 1e-9 && std::abs(z + g * dt * dt * n * (n + 1) / 2) < 1e-9;
  kd_batch_destroy(dev);
  kd_model_destroy(m);
  std::printf("shim freefall %s (vz %.12f z %.12f)\n", ok ? "ok" : "FAILED", vz, z);
  return ok ? 0 : 3;
}
