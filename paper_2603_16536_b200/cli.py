"""Device-backed `simulate` / `bench` harness with the reference CLI's JSONL wire
format (the reference's tools/main.cpp).

    python -m paper_2603_16536_b200.cli simulate SCENE [--duration S] [--output F]
        [--emit-every K] [--seed N] [solver flags]
    python -m paper_2603_16536_b200.cli bench SCENE [SCENE ...] [--worlds 1 8 64]
        [--steps N] [--threads T] [--seed N] [solver flags]

Solver flags (main.cpp add_solver_flags): --dt --integrator {euler,moreau}
--backend {dense,sparse,auto} --beta --rho --eta --eps --max-iters --cr-iters
--fixed-iters; they override the scene's `config` block (make_config).

Records are one JSON object per line with sorted keys and compact separators,
as nlohmann::json::dump() writes them:
  step    (step_record, main.cpp:102-129): type, time, bodies[{position,
          orientation [w,x,y,z], linear_velocity, angular_velocity}], joints
          {name: coordinate} for revolute/prismatic joints, f_inf, contacts,
          solver{iterations, r_p, r_d, r_c, restarts, converged, cr_iterations}
  summary (run_simulate, main.cpp:131-184)
  bench   (run_bench, main.cpp:186-244), including the per-world memory
          estimate formula of the reference.
Every step runs on the B200 kernels; `--threads` is accepted and ignored (the
device has no thread pool, batch.hpp:58)."""
from __future__ import annotations

import argparse
import json
import math
import sys
import time

import numpy as np

from . import loopdyn as L
from .scene import StepConfig, apply_scene_config, load_scene_file

KD_DENSE_ROW_CROSSOVER = 300  # kDenseRowCrossover (delassus.hpp:89)


def dumps(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


def add_solver_flags(p: argparse.ArgumentParser):
    p.add_argument("--dt", type=float)
    p.add_argument("--integrator", choices=["euler", "moreau"])
    p.add_argument("--backend", choices=["dense", "sparse", "auto"])
    p.add_argument("--beta", type=float)
    p.add_argument("--rho", type=float)
    p.add_argument("--eta", type=float)
    p.add_argument("--eps", type=float)
    p.add_argument("--max-iters", type=int)
    p.add_argument("--cr-iters", type=int)
    p.add_argument("--fixed-iters", action="store_true")


def make_config(scene, a) -> StepConfig:
    """make_config (main.cpp:68-85): scene config block, then explicit flags."""
    cfg = apply_scene_config(StepConfig(), scene.config)
    if a.dt is not None:
        cfg.dt = a.dt
    if a.integrator is not None:
        cfg.integrator = a.integrator
    if a.backend is not None:
        cfg.backend = a.backend
    if a.beta is not None:
        cfg.baumgarte_beta = a.beta
    for name in ("rho", "eta", "eps"):
        if getattr(a, name) is not None:
            setattr(cfg, name, getattr(a, name))
    if a.max_iters is not None:
        cfg.max_iters = a.max_iters
    if a.cr_iters is not None:
        cfg.cr_iters = a.cr_iters
    if a.fixed_iters:
        cfg.fixed_iteration_mode = True
    return cfg


def body_json(pose7, twist6) -> dict:
    """body_json (main.cpp:90-100); quaternion serialised [w, x, y, z]."""
    p = [float(x) for x in pose7]
    t = [float(x) for x in twist6]
    return {"position": p[0:3], "orientation": p[3:7], "linear_velocity": t[0:3], "angular_velocity": t[3:6]}


def step_record(model: L.Model, poses7, twists6, time_s: float, d) -> dict:
    """step_record (main.cpp:102-129) from the device state and kd_step_diag."""
    nb = model.n_bodies
    poses7 = np.asarray(poses7).reshape(nb, 7)
    twists6 = np.asarray(twists6).reshape(nb, 6)
    joints = {}
    for j, js in enumerate(model.scene.joints):
        if js.type in ("revolute", "prismatic"):
            joints[model.joint_names[j]] = model.joint_coordinate(j, poses7)
    return {"type": "step", "time": float(time_s),
            "bodies": [body_json(poses7[b], twists6[b]) for b in range(nb)],
            "joints": joints, "f_inf": float(d.f_inf), "contacts": int(d.contact_count),
            "solver": {"iterations": int(d.iterations), "r_p": float(d.r_p), "r_d": float(d.r_d),
                       "r_c": float(d.r_c), "restarts": int(d.restarts), "converged": bool(d.converged),
                       "cr_iterations": int(d.cr_iterations)}}


def run_simulate(a, out) -> int:
    scene = load_scene_file(a.scene)
    model = L.build_model(scene)
    cfg = make_config(scene, a)
    batch = L.WorldBatch()
    batch.add_world(model)
    n_steps = int(round(a.duration / cfg.dt))  # std::lround
    max_f = max_kkt = sum_it = 0.0
    t0 = time.perf_counter()
    for k in range(n_steps):
        batch.step(cfg, 1)
        d = batch.diagnostics()[0]
        max_f = max(max_f, d.f_inf)
        max_kkt = max(max_kkt, d.kkt_momentum_inf)
        sum_it += d.iterations
        if a.emit_every > 0 and ((k + 1) % a.emit_every == 0 or k + 1 == n_steps):
            p, tw, tm = batch.get_state()
            out.write(dumps(step_record(model, p, tw, tm[0], d)) + "\n")
    wall = time.perf_counter() - t0
    p, tw, tm = batch.get_state()
    nb = model.n_bodies
    out.write(dumps({
        "type": "summary", "scene": model.name, "bodies": nb, "kinematic_loops": model.n_loops,
        "steps": n_steps, "wall_s": wall, "steps_per_s": n_steps / wall if wall > 0 else 0.0,
        "max_f_inf": max_f, "max_kkt_momentum_inf": max_kkt,
        "mean_padmm_iterations": sum_it / n_steps if n_steps > 0 else 0.0,
        "final_time": float(tm[0]), "seed": a.seed,
        "final_bodies": [body_json(np.reshape(p, (nb, 7))[b], np.reshape(tw, (nb, 6))[b]) for b in range(nb)],
    }) + "\n")
    return 0


def per_world_mem_estimate(model: L.Model, cfg: StepConfig) -> float:
    """The reference's rough per-world footprint (main.cpp:219-231)."""
    n_rows = model.n_bilateral_rows + model.n_dynamics_rows
    dense = cfg.backend == "dense" or (cfg.backend == "auto" and n_rows <= KD_DENSE_ROW_CROSSOVER)
    backend = n_rows * n_rows if dense else 48.0 * n_rows
    return 8.0 * (13.0 * model.n_bodies + 24.0 * n_rows + backend + 10.0 * n_rows)


def run_bench(a, out) -> int:
    if a.steps <= 0:
        return 0
    scenes = [load_scene_file(s) for s in a.scenes]
    models = [L.build_model(s) for s in scenes]
    cfg = make_config(scenes[0], a)  # the first scene's config (main.cpp:194)
    for worlds in a.worlds:
        batch = L.WorldBatch()
        wm = [w % len(models) for w in range(worlds)]
        for w in wm:
            batch.add_world(models[w])
        if a.seed != 0:  # one mt19937_64 stream, world-major (main.cpp:199-211)
            p, tw, tm = batch.get_state()
            tw = L.bench_jitter(tw, [models[w].n_bodies for w in wm], seed=a.seed)
            batch.set_state(p, tw, tm)
        batch.step(cfg, 1)  # untimed warm-up pass
        t0 = time.perf_counter()
        batch.step(cfg, a.steps)
        wall = time.perf_counter() - t0
        mem = sum(per_world_mem_estimate(models[w], cfg) for w in wm)
        out.write(dumps({"type": "bench", "scenes": list(a.scenes), "worlds": worlds, "steps": a.steps,
                         "wall_s": wall, "throughput_steps_per_s": a.steps * worlds / wall if wall > 0 else 0.0,
                         "per_world_mem_bytes_est": mem / worlds if worlds > 0 else 0.0,
                         "seed": a.seed}) + "\n")
        out.flush()
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="loopdyn-b200",
                                 description="constraint-based rigid-body dynamics in maximal coordinates (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sim = sub.add_parser("simulate", help="run a scene and emit trajectory records")
    sim.add_argument("scene")
    sim.add_argument("--duration", type=float, default=1.0)
    sim.add_argument("--output", default="")
    sim.add_argument("--emit-every", type=int, default=1)
    sim.add_argument("--seed", type=int, default=0)
    add_solver_flags(sim)
    b = sub.add_parser("bench", help="throughput over world counts")
    b.add_argument("scenes", nargs="+")
    b.add_argument("--worlds", type=int, nargs="+", default=[1, 8, 64])
    b.add_argument("--steps", type=int, default=100)
    b.add_argument("--threads", type=int, default=0)
    b.add_argument("--seed", type=int, default=0)
    add_solver_flags(b)
    a = ap.parse_args(argv)
    if a.cmd == "simulate":
        if a.output and a.output != "-":
            with open(a.output, "w") as f:
                return run_simulate(a, f)
        return run_simulate(a, sys.stdout)
    return run_bench(a, sys.stdout)


if __name__ == "__main__":
    sys.exit(main())
