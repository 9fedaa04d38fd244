// C++ drop-in API test (include/loopdyn_b200): builds the reference scenes,
// checks bookkeeping and ModelError behaviour (CPU), and with --gpu steps a
// heterogeneous batch on the device (reference test_batch.cpp / acceptance #1,
// #7 semantics).  Prints PASS/FAIL lines; exit code = failures.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>

#include "json.hpp"
#include "loopdyn_b200/loopdyn.hpp"
#include "loopdyn_b200/scene_json.hpp"

using namespace loopdyn_b200;
static int failures = 0;
#define CHECK(c)                                               \
  do {                                                         \
    if (!(c)) {                                                \
      ++failures;                                              \
      std::printf("[FAIL] %s:%d %s\n", __FILE__, __LINE__, #c); \
    }                                                          \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const bool gpu = argc > 2 && std::strcmp(argv[2], "--gpu") == 0;
  std::ifstream in(argv[1]);
  std::stringstream ss;
  ss << in.rdbuf();
  const auto bundle = nlohmann::json::parse(ss.str());
  auto scene = [&](const char* n) { return parse_scene(bundle[n].dump(), n); };

  // model bookkeeping (test_model.cpp:42-55)
  const SceneDescription fb = scene("fourbar");
  auto fourbar = std::make_shared<const MechanismModel>(build_model(fb));
  CHECK(fourbar->n_bilateral_rows() == 20);
  CHECK(fourbar->velocity_dim() == 18);
  CHECK(fourbar->n_loops() == 1);
  CHECK(fourbar->n_dynamics_rows() == 1);
  std::vector<Pose> poses;
  for (const auto& b : fb.bodies) poses.push_back(b.pose);
  CHECK(std::abs(joint_coordinate(*fourbar, 0, poses) - M_PI / 2) < 1e-9);
  // ModelError codes (test_model.cpp:80-154)
  bool threw = false;
  try {
    SceneDescription s = fb;
    s.joints[0].parent = "nosuch";
    build_model(s);
  } catch (const ModelError& e) {
    threw = e.code() == ModelError::Code::InvalidReference && std::string(e.what()).find("unknown body") != std::string::npos;
  }
  CHECK(threw);
  threw = false;
  try {
    joint_coordinate(*fourbar, 99, poses);
  } catch (const std::runtime_error&) {
    threw = true;
  }
  CHECK(threw);
  // SceneError context (scene.cpp:14-16)
  threw = false;
  try {
    parse_scene("{\"bodies\":[{\"name\":\"a\",\"inertia\":[1,1,1]}]}", "x.json");
  } catch (const SceneError& e) {
    threw = std::string(e.what()) == "x.json: bodies[0]: missing field 'mass'";
  }
  CHECK(threw);

  if (gpu) {
    auto sphere = std::make_shared<const MechanismModel>(build_model(scene("sphere_on_plane")));
    auto freefall = std::make_shared<const MechanismModel>(build_model(scene("freefall")));
    WorldBatch batch;
    batch.add_world(fourbar);
    batch.add_world(sphere);
    batch.add_world(freefall);
    CHECK(batch.pose_offset(1) == 21 && batch.pose_offset(2) == 28 && batch.twist_offset(2) == 24);
    StepConfig cfg;
    double kkt = 0;
    for (int k = 0; k < 240; ++k) {
      batch_step(batch, cfg);
      for (int w = 0; w < 3; ++w) kkt = std::max(kkt, batch.diagnostics(w).kkt_momentum_inf);
    }
    CHECK(kkt <= 1e-5);
    const WorldState s = batch.extract_state(2);  // freefall closed form (acceptance #7)
    const double n = 240, g = 9.81, dt = cfg.dt;
    CHECK(std::abs(s.twists[0].linear[2] + g * n * dt) < 1e-9);
    CHECK(std::abs(s.poses[0].position[2] + g * dt * dt * n * (n + 1) / 2) < 1e-9);
    const StepDiagnostics d = batch.diagnostics(1);
    CHECK(d.contact_count == 1 && d.n_rows == 3 && d.impulses.size() == 3);
    CHECK(std::abs(d.impulses[0] - 9.81 / 240.0) < 1e-3 * 9.81 / 240.0);  // resting sphere (acceptance #6)
    // single-world step() wrapper
    WorldState st = initial_state(*fourbar);
    WorldBatch scratch;
    for (int k = 0; k < 10; ++k) step(fourbar, st, cfg, &scratch);
    CHECK(std::abs(st.time - 10 * cfg.dt) < 1e-12);
    // the reference signature step(const MechanismModel&, WorldState&, cfg)
    // warm-starts from the state's caches: a fresh one-world batch per call
    // tracks a persistent batch bit for bit (checkpoint/restore keeps the
    // trajectory, stepper.cpp:181-187)
    WorldState a = initial_state(*sphere);
    WorldBatch persistent;
    persistent.add_world(sphere);
    bool same = true;
    for (int k = 0; k < 30; ++k) {
      const StepDiagnostics da = step(*sphere, a, cfg);
      batch_step(persistent, cfg);
      const WorldState b = persistent.extract_state(0);
      same = same && da.solver.iterations == persistent.diagnostics(0).solver.iterations;
      for (int q = 0; q < 3; ++q) same = same && a.poses[0].position[q] == b.poses[0].position[q];
      for (int q = 0; q < 3; ++q) same = same && a.twists[0].linear[q] == b.twists[0].linear[q];
    }
    CHECK(same);
    CHECK(a.joint_cache.valid && a.contact_cache.entries.size() == 1);
  }
  std::printf("%s: %d failures\n", gpu ? "cpp api (gpu)" : "cpp api (cpu)", failures);
  return failures;
}
