"""L^-1 formation phase split of the dense kernel on DR-Legs (needs a
-DKD_PROF_INV build; development tool): thread 0's cycles in phase 1
(X_kk,j = Linv_kk B_kk,j), phase 2 (B_ij -= L_i,kk X_kk,j), phase 3
(B_i,kk = -L_i,kk Linv_kk), each with its barriers, and the final step.
usage: inv_probe.py LIB [worlds]"""
import json
import os
import sys

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
b.step(cfg, 30)
b.step(cfg, 1)
ph = b.phase_cycles().astype(float)
print(json.dumps({"worlds": nw, "phase1": ph[:, 5].mean(), "phase2": ph[:, 6].mean(), "phase3": ph[:, 7].mean(),
                  "final_step": ph[:, 1].mean(), "inverse_total_stamp3": ph[:, 3].mean()}))
