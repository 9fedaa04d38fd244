"""Two independent half-batches on two streams vs one batch (diagnostic): how
much kernel-tail overlap a library-internal split could buy per workload."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scene import parse_scene_obj  # noqa: E402
from paper_2603_16536_b200.scenes import dr_legs  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
bundle = json.load(open(os.path.join(ROOT, "tests", "golden", "scenes_bundle.json")))
which = sys.argv[1] if len(sys.argv) > 1 else "dr_legs"
if which == "dr_legs":
    scenes, wm, N = [dr_legs()], lambda w: 0, 4096
else:
    scenes = [parse_scene_obj(bundle["fourbar"], "fourbar"), dr_legs(), parse_scene_obj(bundle["serial_chain_10"], "s")]
    wm, N = (lambda w: w % 3), 16384
models = [K.build_model(s) for s in scenes]
cfg = K.config_for(scenes[0])


def mk(lo, hi):
    b = K.WorldBatch()
    for w in range(lo, hi):
        b.add_world(models[wm(w)])
    p, t, tm = b.get_state()
    t = K.bench_jitter(t, [models[wm(w)].n_bodies for w in range(lo, hi)], seed=1)
    b.set_state(p, t, tm)
    b.step(cfg, 20)
    return b


def timeit(bs, steps=10):
    for b in bs:
        b.step_async(cfg, 1)
    for b in bs:
        b.sync()
    t0 = time.perf_counter()
    for _ in range(steps):
        for b in bs:
            b.step_async(cfg, 1)
    for b in bs:
        b.sync()
    return (time.perf_counter() - t0) / steps * 1e3


full = [mk(0, N)]
halves = [mk(0, N // 2), mk(N // 2, N)]
for rep in range(2):
    print(which, "full ms/step %.3f" % timeit(full), "two halves ms/step %.3f" % timeit(halves), flush=True)
