"""Parity at the bench's scale and trajectory point (GPU box only).

The default bench line steps 4096 DR-Legs worlds for 50 settle + 5 warm-up +
30 timed steps; the C3 line 16384 worlds of the four-bar / DR-Legs /
serial_chain_10 mix.  Here the full batch runs on the device for the same 85
steps and a sample of its worlds (spread over the batch, same global jitter
stream, main.cpp:199-211) runs on the CPU oracle: per step the row, contact
and limit counts match exactly and the PADMM iteration counts match in at
least 99 % of world-steps; at the end the states agree within the trajectory
tolerances of test_parity_gpu.py.  Solo-vs-batch bitwise equality
(test_batch_gpu.py) carries the result to every other world.
"""
import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import dr_legs

pytestmark = pytest.mark.gpu


def _run(scenes, wmodel, n_worlds, sample, steps, seed=1):
    models = [K.build_model(sc) for sc in scenes]
    omodels = [oracle_lib.OracleModel(sc) for sc in scenes]
    cfg = K.config_for(scenes[0])  # one StepConfig from the first scene (main.cpp:194)
    gb = K.WorldBatch()
    for w in range(n_worlds):
        gb.add_world(models[wmodel(w)])
    p, t, tm = gb.get_state()
    nb = [models[wmodel(w)].n_bodies for w in range(n_worlds)]
    t = K.bench_jitter(t, nb, seed=seed)
    gb.set_state(p, t, tm)
    po = np.cumsum([0] + [7 * x for x in nb])
    to = np.cumsum([0] + [6 * x for x in nb])
    ob = oracle_lib.OracleBatch(omodels, [wmodel(w) for w in sample], n_threads=16)
    ob.set_state(np.concatenate([p[po[w]:po[w + 1]] for w in sample]),
                 np.concatenate([t[to[w]:to[w + 1]] for w in sample]), tm[sample])
    same = total = 0
    for _ in range(steps):
        gb.step(cfg)
        ob.step(cfg)
        dg, do = gb.diagnostics(), ob.diagnostics()
        for k, w in enumerate(sample):
            assert (dg[w].n_rows, dg[w].contact_count, dg[w].n_limits) == \
                (do[k].n_rows, do[k].contact_count, do[k].n_limits)
            same += dg[w].iterations == do[k].iterations
            total += 1
    pg, tg, _ = gb.get_state()
    pS, tS, _ = ob.get_state()
    pg = np.concatenate([pg[po[w]:po[w + 1]] for w in sample])
    tg = np.concatenate([tg[to[w]:to[w + 1]] for w in sample])
    return same / total, float(np.abs(pg - pS).max()), float(np.abs(tg - tS).max())


def test_dr_legs_4096_worlds_bench_trajectory_vs_oracle():
    nw = 4096
    sample = list(range(0, nw, 171)) + [nw - 1]  # 25 worlds across the batch
    frac, dp, dt = _run([dr_legs()], lambda w: 0, nw, sample, 85)
    assert frac >= 0.99
    assert dp < 1e-7 and dt < 1e-5


def test_c3_mix_16384_worlds_vs_oracle():
    scenes = [oracle_lib.bundled_scene("fourbar"), dr_legs(), oracle_lib.bundled_scene("serial_chain_10")]
    nw = 16384
    sample = list(range(0, nw, 997)) + [nw - 3, nw - 2, nw - 1]  # all three models
    frac, dp, dt = _run(scenes, lambda w: w % 3, nw, sample, 60)
    assert frac >= 0.99
    assert dp < 1e-7 and dt < 1e-5
