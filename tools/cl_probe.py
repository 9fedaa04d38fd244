"""K2c phase split (needs a -DKD_PROF_CL build): rank 0's thread-0 cycles per
PADMM iteration in each phase, DR-Legs after settling.  usage: cl_probe.py LIB [worlds]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_16536_b200.loopdyn as L  # noqa: E402
L.LIB_PATH = os.path.abspath(sys.argv[1])
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scenes import dr_legs  # noqa: E402

nw = int(sys.argv[2]) if len(sys.argv) > 2 else 296
sc = dr_legs()
cfg = K.config_for(sc)
m = K.build_model(sc)
b = K.WorldBatch()
for _ in range(nw):
    b.add_world(m)
p, t, tm = b.get_state()
t = K.bench_jitter(t, [m.n_bodies] * nw, seed=1)
b.set_state(p, t, tm)
b.step(cfg, 30)
b.step(cfg, 1)
ph = b.phase_cycles().astype(float)
it = np.array([x.iterations for x in b.diagnostics()[:nw]], float)
names = ["bar_a", "pass1", "combine", "wait_B", "pass2", "cluster_A", "units", "red_rest"]
out = {"iters_mean": float(it.mean()), "kernels": sorted(set(b.kernels()))}
for k, nm in enumerate(names):
    out[nm] = round(float(np.sum(ph[:, k]) / np.sum(it)), 1)
out["total"] = round(sum(out[nm] for nm in names), 1)
print(json.dumps(out))
