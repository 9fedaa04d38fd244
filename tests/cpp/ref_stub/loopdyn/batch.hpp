// Test scaffold, not reference code: the few declarations of the reference's
// loopdyn headers (batch.hpp:14-58, stepper.hpp:14-34, padmm.hpp:8-17,
// delassus.hpp:85) that the INTEGRATION.md shim touches, so that the shim
// (tests/cpp/batch_b200_shim.cpp) is compiled and linked against the C-ABI by
// tests/test_cpp_api.py.  The real headers need Eigen, which this image lacks.
#pragma once
#include <vector>

namespace loopdyn {
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
  double baumgarte_beta = 0.2, contact_margin = 0.01, impact_velocity_threshold = 0.1, bias_clamp = 10.0;
  double limit_margin_angular = 0.01, limit_margin_linear = 0.001;
  bool warm_start = true;
};
class WorldBatch {
 public:
  explicit WorldBatch(std::vector<double> poses = {}, std::vector<double> twists = {})
      : poses_(std::move(poses)), twists_(std::move(twists)) {}
  const std::vector<double>& pose_storage() const { return poses_; }
  const std::vector<double>& twist_storage() const { return twists_; }

 private:
  std::vector<double> poses_, twists_;
};
}  // namespace loopdyn
