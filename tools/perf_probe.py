"""Quick device-throughput probe for DR-Legs batches (diagnostic only).
Separates the per-step fixed cost (assembly + factor + inverse) from the
per-PADMM-iteration cost using fixed-iteration mode."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scenes import dr_legs  # noqa: E402


def make(nw, settle=0):
    sc = dr_legs()
    cfg = K.config_for(sc)
    m = K.build_model(sc)
    b = K.WorldBatch()
    for _ in range(nw):
        b.add_world(m)
    p, t, tm = b.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * nw, seed=1)
    b.set_state(p, t, tm)
    if settle:
        b.step(cfg, settle)
    return b, cfg


def timed(b, cfg, steps):
    b.step(cfg, 2)
    b.enable_timing(True)
    t0 = time.perf_counter()
    b.step(cfg, steps)
    dt = time.perf_counter() - t0
    return dt, b.timing()


for nw in [int(a) for a in (sys.argv[1:] or ["148", "4096"])]:
    b, cfg = make(nw, settle=50)
    out = {"worlds": nw}
    for iters in (1, 41):
        c = K.StepConfig(**{**cfg.__dict__})
        c.fixed_iteration_mode = True
        c.max_iters = iters
        dt, tim = timed(b, c, 5)
        out[f"fixed{iters}_dense_ms"] = tim["dense_ms"] / 5
    out["per_iter_ms"] = (out["fixed41_dense_ms"] - out["fixed1_dense_ms"]) / 40
    out["fixed_cost_ms"] = out["fixed1_dense_ms"] - out["per_iter_ms"]
    steps = 10
    dt, tim = timed(b, cfg, steps)
    d = b.diagnostics()
    its = np.array([x.iterations for x in d[:nw]])
    out.update({"wall_ms_per_step": 1e3 * dt / steps, "world_steps_per_s": nw * steps / dt,
                "timing_ms_per_step": {k: v / steps for k, v in tim.items() if k.endswith("ms")},
                "iters_mean": float(its.mean()), "iters_max": int(its.max())})
    print(json.dumps(out), flush=True)

# phase breakdown (cycles) of the fused dense kernel at the last step
b, cfg = make(148, settle=50)
b.step(cfg, 1)
pc = b.phase_cycles()
its = np.array([x.iterations for x in b.diagnostics()[:148]])
names = ["gram_scaled", "unused", "cholesky", "inverse", "padmm", "chol_panel", "chol_syrk", "chol_diag"]
if b.kernels()[0] == "supernodal+dense":  # slots 1, 5-7 come from the hand-off factor kernel (kd_snfactor.cu)
    names = ["scatter_diag_inverse", "k2f_panel_factor", "unused", "inverse", "padmm", "k2f_gram", "k2f_panels",
             "k2f_updates"]
print(json.dumps({"kernel": b.kernels()[0], "phase_cycles_mean": {names[k]: float(pc[:, k].mean()) for k in range(8)},
                  "iters_mean": float(its.mean()),
                  "padmm_cycles_per_iter": float((pc[:, 4] / np.maximum(its, 1)).mean())}), flush=True)
