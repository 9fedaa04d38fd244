"""Per-warp cycles of one explicit-inverse solve pass in the dense kernel
(needs a -DKD_PROF_WARP=1|2 build; run with KD_DENSE_DF=0): mean cycles per
PADMM iteration each warp spends in its pass-1 tile row (1) or pass-2 tile
column (2), excluding the barriers.  usage: warp_probe.py LIB [worlds]"""
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

nw = int(sys.argv[2]) if len(sys.argv) > 2 else 148
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
print(json.dumps({"lib": os.path.basename(sys.argv[1]), "iters_mean": float(it.mean()),
                  "per_warp_per_iter": [round(float(np.sum(ph[:, k]) / np.sum(it)), 1) for k in range(8)]}))
