"""Hetero-batch probe (diagnostic): per-model step time alone vs the mixed batch."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scene import parse_scene_obj  # noqa: E402
from paper_2603_16536_b200.scenes import dr_legs  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
bundle = json.load(open(os.path.join(ROOT, "tests", "golden", "scenes_bundle.json")))
scenes = [parse_scene_obj(bundle["fourbar"], "fourbar"), dr_legs(), parse_scene_obj(bundle["serial_chain_10"], "serial_chain_10")]
models = [K.build_model(s) for s in scenes]
cfg = K.config_for(scenes[0])


def run(wm, label):
    b = K.WorldBatch()
    for w in wm:
        b.add_world(models[w])
    p, t, tm = b.get_state()
    t = K.bench_jitter(t, [models[w].n_bodies for w in wm], seed=1)
    b.set_state(p, t, tm)
    b.step(cfg, 20)
    b.enable_timing(True)
    t0 = time.perf_counter()
    b.step(cfg, 10)
    dt = (time.perf_counter() - t0) / 10
    tim = b.timing()
    import numpy as np
    its = np.array([d.iterations for d in b.diagnostics()[:len(wm)]])
    print(label, len(wm), "ms/step %.3f" % (1e3 * dt), "iters mean %.1f max %d" % (its.mean(), its.max()), {k: round(v / 10, 3) for k, v in tim.items() if k.endswith("ms")},
          "kernels", {k: b.kernels().count(k) for k in set(b.kernels())}, flush=True)


N = 16384
which = sys.argv[1:] or ["hetero", "0", "1", "2"]
for x in which:
    if x == "hetero":
        run([w % 3 for w in range(N)], "hetero")
    else:
        run([int(x)] * (N // 3), scenes[int(x)].name)
