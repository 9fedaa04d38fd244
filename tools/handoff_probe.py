"""Hand-off prologue split of the dense kernel on DR-Legs (needs a
-DKD_PROF_HO build; development tool): kernel start -> zero fill, scatter of
the supernodal factor into tiles, diagonal-tile inverses (thread 0's clock64).
usage: handoff_probe.py LIB [worlds]"""
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
print(json.dumps({"worlds": nw, "start_to_zero_fill": ph[:, 5].mean(), "scatter": ph[:, 6].mean(),
                  "diag_inverses": ph[:, 7].mean(), "stamp0_total": ph[:, 0].mean()}))
