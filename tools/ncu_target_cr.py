"""Small fixed workload for ncu captures of the matrix-free CR kernel (closed
chain by default; argv[3] = sphere_pile | box_pile)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scenes import box_pile, closed_chain, sphere_pile  # noqa: E402

nw = int(sys.argv[1]) if len(sys.argv) > 1 else 148
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
which = sys.argv[3] if len(sys.argv) > 3 else "closed_chain"
sc = {"closed_chain": lambda: closed_chain(22), "sphere_pile": lambda: sphere_pile(100),
      "box_pile": lambda: box_pile(64)}[which]()
cfg = K.config_for(sc)
m = K.build_model(sc)
b = K.WorldBatch()
for _ in range(nw):
    b.add_world(m)
p, t, tm = b.get_state()
t = K.bench_jitter(t, [m.n_bodies] * nw, seed=1)
b.set_state(p, t, tm)
for _ in range(steps):
    b.step(cfg, 1)
print("done", nw, steps)
