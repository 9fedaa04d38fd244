"""A/B of library builds on one workload (diagnostic): for each .so, a fresh
process settles the batch, times K steps (device-synchronised wall clock) and
prints world-steps/s, mean PADMM iterations and a state checksum (equal
checksums = bitwise-equal trajectories).
usage: lib_ab.py WORKLOAD WORLDS LIB [LIB ...]"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(workload, nw, libpath):
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_2603_16536_b200.loopdyn as L
    L.LIB_PATH = os.path.abspath(libpath)
    import paper_2603_16536_b200 as K
    from paper_2603_16536_b200 import scenes
    def bundled(name):
        from paper_2603_16536_b200.scene import parse_scene_obj
        with open(os.path.join(ROOT, "tests", "golden", "scenes_bundle.json")) as f:
            return parse_scene_obj(json.load(f)[name], name)
    sc = {"fourbar": lambda: bundled("fourbar"), "dr_legs": scenes.dr_legs, "stewart_tower": scenes.stewart_tower,
          "closed_chain": lambda: scenes.closed_chain(22), "sphere_pile": lambda: scenes.sphere_pile(100),
          "box_pile": lambda: scenes.box_pile(64)}[workload]()
    cfg = K.config_for(sc)
    m = K.build_model(sc)
    b = K.WorldBatch()
    for _ in range(nw):
        b.add_world(m)
    p, t, tm = b.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * nw, seed=1)
    b.set_state(p, t, tm)
    b.step(cfg, 30)
    b.get_state()
    res = []
    for _ in range(3):
        t0 = time.perf_counter()
        b.step(cfg, 10)
        p, t, _ = b.get_state()
        res.append(nw * 10 / (time.perf_counter() - t0))
    its = float(np.mean([d.iterations for d in b.diagnostics()]))
    print(json.dumps({"lib": os.path.basename(libpath), "world_steps_s": round(max(res)), "iters": its,
                      "checksum": float(np.sum(np.abs(p)) + np.sum(np.abs(t)))}))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]), sys.argv[4])
    else:
        for lib in sys.argv[3:]:
            subprocess.run([sys.executable, __file__, "--child", sys.argv[1], sys.argv[2], lib], check=False)
