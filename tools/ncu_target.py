"""Small fixed workload for ncu captures (DR-Legs, 148 worlds = one CTA per SM;
argv[3] = fourbar for the bundled four-bar)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scenes import dr_legs  # noqa: E402

nw = int(sys.argv[1]) if len(sys.argv) > 1 else 148
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
if len(sys.argv) > 3 and sys.argv[3] == "fourbar":
    import json
    from paper_2603_16536_b200.scene import parse_scene_obj
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sc = parse_scene_obj(json.load(open(os.path.join(root, "tests", "golden", "scenes_bundle.json")))["fourbar"], "fourbar")
else:
    sc = dr_legs()
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
