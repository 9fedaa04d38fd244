"""A/B throughput of the fused dense kernel vs the supernodal kernel per model
(diagnostic): python tools/kernel_ab.py  (run twice: KD_SPARSE=0 and default)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle_lib  # noqa: E402
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scenes import dr_legs  # noqa: E402

for name, nw in [("fourbar", 16384), ("double_fourbar", 16384), ("serial_chain_10", 16384), ("dr_legs", 4096)]:
    sc = dr_legs() if name == "dr_legs" else oracle_lib.bundled_scene(name)
    cfg = K.config_for(sc)
    m = K.build_model(sc)
    b = K.WorldBatch()
    for _ in range(nw):
        b.add_world(m)
    p, t, tm = b.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * nw, seed=1)
    b.set_state(p, t, tm)
    b.step(cfg, 20)
    b.enable_timing(True)
    t0 = time.perf_counter()
    b.step(cfg, 10)
    dt = time.perf_counter() - t0
    tim = b.timing()
    its = sum(d.iterations for d in b.diagnostics()) / nw
    print(json.dumps({"model": name, "worlds": nw, "kernel": b.kernels()[0], "ws_per_s": nw * 10 / dt,
                      "solve_ms": tim["dense_ms"] / 10, "iters": its}), flush=True)
