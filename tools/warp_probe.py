"""Per-warp cycles of the explicit-inverse solve in the dense kernel, mean per
PADMM iteration (needs a -DKD_PROF_WARP=k build):
  1 / 2  pass-1 tile row / pass-2 tile column, barrier version (KD_DENSE_DF=0);
  3      dataflow solve: entry barrier -> the warp's column done;
  4      dataflow solve: time spent waiting for published rows;
  5      dataflow solve: entry barrier -> the warp's row published;
  6      PADMM units: x-complete barrier -> before the residual reduction;
  7      the block residual reduction (warp max, barrier, partials).
usage: warp_probe.py LIB [worlds]"""
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
