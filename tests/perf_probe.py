"""Quick device-throughput probe for DR-Legs batches (diagnostic only)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scenes import dr_legs  # noqa: E402

for nw in [int(a) for a in (sys.argv[1:] or ["148", "1024", "4096"])]:
    sc = dr_legs()
    cfg = K.config_for(sc)
    m = K.build_model(sc)
    b = K.WorldBatch()
    for _ in range(nw):
        b.add_world(m)
    p, t, tm = b.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * nw, seed=1)
    b.set_state(p, t, tm)
    b.step(cfg, 3)
    b.enable_timing(True)
    steps = 10
    t0 = time.perf_counter()
    b.step(cfg, steps)
    dt = time.perf_counter() - t0
    tim = b.timing()
    d = b.diagnostics()
    its = np.array([x.iterations for x in d[:nw]])
    rows = np.array([x.n_rows for x in d[:nw]])
    print(json.dumps({"worlds": nw, "wall_ms_per_step": 1e3 * dt / steps, "world_steps_per_s": nw * steps / dt,
                      "timing_ms_per_step": {k: v / steps for k, v in tim.items() if k.endswith("ms")},
                      "iters_mean": float(its.mean()), "iters_max": int(its.max()), "rows_mean": float(rows.mean()),
                      "rows_max": int(rows.max())}), flush=True)
