"""GPU-vs-oracle parity probe (diagnostic; the asserted version is
tests/test_parity_gpu.py).  Prints per-scene discrete agreement and float
deviations after N free-running steps."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle_lib  # noqa: E402
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scenes import closed_chain, dr_legs, sphere_pile  # noqa: E402


def run(name, scene, steps, n_worlds=1, cfg=None, jitter=False, every=1):
    cfg = cfg or K.config_for(scene)
    m = K.build_model(scene)
    om = oracle_lib.OracleModel(scene)
    gb = K.WorldBatch()
    for _ in range(n_worlds):
        gb.add_world(m)
    ob = oracle_lib.OracleBatch([om], [0] * n_worlds, n_threads=8)
    if jitter:
        p, t, tm = ob.get_state()
        t = K.bench_jitter(t, [m.n_bodies] * n_worlds, seed=1)
        ob.set_state(p, t, tm)
        gb.set_state(p, t, tm)
    rep = {"name": name, "steps": steps, "worlds": n_worlds, "rows_mismatch": 0, "contacts_mismatch": 0,
           "limits_mismatch": 0, "iter_diff_max": 0, "iter_sum_gpu": 0, "iter_sum_cpu": 0}
    t_g = t_c = 0.0
    worst = 0.0
    for k in range(steps):
        t0 = time.perf_counter()
        gb.step(cfg)
        t1 = time.perf_counter()
        ob.step(cfg)
        t2 = time.perf_counter()
        t_g += t1 - t0
        t_c += t2 - t1
        if (k + 1) % every == 0 or k == steps - 1:
            dg, do = gb.diagnostics(), ob.diagnostics()
            for w in range(n_worlds):
                rep["rows_mismatch"] += dg[w].n_rows != do[w].n_rows
                rep["contacts_mismatch"] += dg[w].contact_count != do[w].contact_count
                rep["limits_mismatch"] += dg[w].n_limits != do[w].n_limits
                rep["iter_diff_max"] = max(rep["iter_diff_max"], abs(dg[w].iterations - do[w].iterations))
                rep["iter_sum_gpu"] += dg[w].iterations
                rep["iter_sum_cpu"] += do[w].iterations
            pg, tg, _ = gb.get_state()
            po, to, _ = ob.get_state()
            worst = max(worst, float(np.abs(pg - po).max()), float(np.abs(tg - to).max()))
    pg, tg, tmg = gb.get_state()
    po, to, tmo = ob.get_state()
    rep["pose_maxdiff"] = float(np.abs(pg - po).max())
    rep["twist_maxdiff"] = float(np.abs(tg - to).max())
    rep["worst_along"] = worst
    rep["time_diff"] = float(np.abs(tmg - tmo).max())
    dg, do = gb.diagnostics(), ob.diagnostics()
    rep["kkt_gpu"] = max(d.kkt_momentum_inf for d in dg[:n_worlds])
    rep["kkt_cpu"] = max(d.kkt_momentum_inf for d in do[:n_worlds])
    rep["gpu_s_per_step"] = t_g / steps
    rep["cpu_s_per_step"] = t_c / steps
    print(json.dumps(rep), flush=True)
    return rep


def one_step_rows(name, scene, cfg=None):
    """Cold-start one-step parity of the assembled rows and solved impulses."""
    cfg = cfg or K.config_for(scene)
    m = K.build_model(scene)
    om = oracle_lib.OracleModel(scene)
    gb = K.WorldBatch()
    gb.add_world(m)
    ob = oracle_lib.OracleBatch([om], [0], n_threads=1)
    ob.set_trace(True)
    gb.step(cfg)
    ob.step(cfg)
    rg, ro = gb.dump_rows(0), ob.dump_rows(0)
    rep = {"name": name, "n": len(rg["kind"])}
    if len(rg["kind"]) == len(ro["kind"]) and len(rg["kind"]):
        rep["body_equal"] = bool((rg["body"] == ro["body"]).all())
        rep["kind_equal"] = bool((rg["kind"] == ro["kind"]).all())
        for key in ("J", "bias", "reg", "scale", "vf", "lambda", "z"):
            a, b = rg[key], ro[key]
            rep[key] = float(np.abs(a - b).max() / max(1e-300, np.abs(b).max()))
    print(json.dumps(rep), flush=True)


if __name__ == "__main__":
    bundle = oracle_lib.load_bundle()
    for name in ["fourbar", "double_fourbar", "serial_chain_10", "pendulum", "sphere_on_plane", "inclined_box",
                 "freefall"]:
        sc = oracle_lib.bundled_scene(name)
        one_step_rows(name, sc)
        run(name, sc, 240)
    one_step_rows("dr_legs", dr_legs())
    run("dr_legs", dr_legs(), 50, n_worlds=4, jitter=True)
    fb = oracle_lib.bundled_scene("fourbar")
    cfg = K.config_for(fb)
    cfg.backend = "sparse"
    cfg.cr_iters = 50
    run("fourbar_cr50", fb, 240, cfg=cfg)
    cfg.cr_iters = 9
    run("fourbar_cr9", fb, 240, cfg=cfg)
    cc = closed_chain(16)
    one_step_rows("closed_chain", cc)
    run("closed_chain", cc, 20)
    sp = sphere_pile(40)
    one_step_rows("sphere_pile", sp)
    run("sphere_pile", sp, 20)
