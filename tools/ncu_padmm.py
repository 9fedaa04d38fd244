"""ncu target: DR-Legs, one world per SM (148), settled 50 steps, then steps in
fixed-iteration mode with many PADMM iterations so the dense kernel's PADMM
loop dominates its profile (the per-iteration solve passes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scenes import dr_legs  # noqa: E402

nw = int(sys.argv[1]) if len(sys.argv) > 1 else 148
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
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
c = K.StepConfig(**{**cfg.__dict__})
c.fixed_iteration_mode = True
c.max_iters = iters
for _ in range(3):
    b.step(c, 1)
print("done", nw, iters)
