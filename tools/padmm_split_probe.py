"""PADMM iteration cost split of the dense kernel (needs the KD_PROF_PADMM
build, tools/libkamino_b200_prof.so): per-world cycles of the solve (incl. its
entry barrier), units + reduction, and the rest, natural steps on DR-Legs.
usage: padmm_split_probe.py [worlds] [lib]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_16536_b200.loopdyn as L  # noqa: E402
L.LIB_PATH = os.path.abspath(sys.argv[2]) if len(sys.argv) > 2 else os.path.join(ROOT, "tools", "libkamino_b200_prof.so")
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
b.step(cfg, 1)
ph = b.phase_cycles().astype(float)
it = np.array([x.iterations for x in b.diagnostics()[:nw]], float)
per = lambda k: float(np.sum(ph[:, k]) / np.sum(it))  # noqa: E731
print(json.dumps({"lib": os.path.basename(L.LIB_PATH), "iters_mean": float(it.mean()), "padmm_per_iter": per(4), "solve_incl_entry_barrier": per(1),
                  "units_and_reduction": per(7), "pass1": per(5), "pass2": per(6),
                  "rest": per(4) - per(1) - per(7), "inverse": float(ph[:, 3].mean()),
                  "scatter": float(ph[:, 0].mean()), "solve_setup": float(ph[:, 2].mean())}))
