"""K2f (hand-off factor kernel) phase split on DR-Legs (thread 0's clock64):
setup + Gram, panel factors (incl. the barrier after them), ancestor updates,
and warp 0's time inside the register panel factor.  usage: k2f_probe.py [worlds]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16536_b200.loopdyn as L  # noqa: E402
if len(sys.argv) > 2:
    L.LIB_PATH = os.path.abspath(sys.argv[2])  # a -DKD_PROF_K2F build: [6] setup, [7] Gram
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
b.step(cfg, 30)
b.step(cfg, 1)
ph = b.phase_cycles().astype(float)
print(json.dumps({"worlds": nw, "setup_gram": ph[:, 5].mean(), "panels_incl_barrier": ph[:, 6].mean(),
                  "ancestor_updates": ph[:, 7].mean(), "warp0_panel_factor": ph[:, 1].mean(),
                  "plan": m.sparse_plan_info()}))
