"""Per-world phase cycles of the dense kernel (kd_batch_get_phase_cycles) and
kernel choice, on DR-Legs after settling, natural and fixed-iteration steps."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scenes import dr_legs  # noqa: E402

nw = int(sys.argv[1]) if len(sys.argv) > 1 else 148
sc = dr_legs()
cfg = K.config_for(sc)
m = K.build_model(sc)
b = K.WorldBatch()
for _ in range(nw):
    b.add_world(m)
p, t, tm = b.get_state()
t = K.bench_jitter(t, [m.n_bodies] * nw, seed=1)
b.set_state(p, t, tm)
b.step(cfg, 50)
for iters in (0, 200):
    c = K.StepConfig(**{**cfg.__dict__})
    if iters:
        c.fixed_iteration_mode = True
        c.max_iters = iters
    b.step(c, 1)
    ph = b.phase_cycles()
    d = b.diagnostics()
    kinds = b.kernels()
    it = np.array([x.iterations for x in d[:nw]])
    pad = ph[:, 4].astype(float)
    print(json.dumps({"fixed": iters, "kinds": {k: kinds.count(k) for k in set(kinds)},
                      "iters": [int(it.min()), float(it.mean()), int(it.max())],
                      "padmm_cycles": [float(pad.min()), float(pad.mean()), float(pad.max())],
                      "per_iter": float(np.mean(pad / np.maximum(it, 1)))}))

# iteration histogram and total per-world K2 cycles over a few natural steps
tot, hist = [], np.zeros(9, int)
for _ in range(5):
    b.step(cfg, 1)
    ph = b.phase_cycles().astype(float)
    d = b.diagnostics()
    it = np.array([x.iterations for x in d[:nw]])
    hist += np.histogram(it, bins=[0, 10, 20, 30, 40, 60, 100, 150, 199, 201])[0]
    tot.append(float((ph[:, 0] + ph[:, 2] + ph[:, 3] + ph[:, 4]).sum()))
b.enable_timing(True)
b.step(cfg, 5)
tim = b.timing()
print(json.dumps({"iter_hist_bins": [0, 10, 20, 30, 40, 60, 100, 150, 199, 201], "hist_per_step": (hist / 5).tolist(),
                  "k2_cycles_per_sm_per_step": float(np.mean(tot)) / 148,
                  "k2_ideal_ms": float(np.mean(tot)) / 148 / 1.965e6, "dense_family_ms": tim["dense_ms"] / 5}))
