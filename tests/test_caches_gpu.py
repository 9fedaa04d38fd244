"""Warm-start caches across the boundary (GPU box only).

The reference's WorldState carries the joint, limit and contact reaction caches
(stepper.hpp:38-56, contacts.hpp:32-38); WorldBatch::extract_state /
insert_state copy them with the state (batch.cpp:27-72) and step() warm-starts
from them (stepper.cpp:19-46, 181-187).  Here:

* the device caches after N steps equal the oracle's (same keys and entry
  order; values within the solver's 1e-9 relative band);
* extract_state -> insert_state into a fresh batch reproduces the next step
  bit for bit (checkpoint / restore does not change trajectories);
* the one-world `step(model, state, cfg)` warm-starts from `state` and so
  tracks a persistent batch bit for bit.
"""
import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import closed_chain, dr_legs, sphere_pile

pytestmark = pytest.mark.gpu


def _jittered(sc, n_worlds, seed=1):
    m, om = K.build_model(sc), oracle_lib.OracleModel(sc)
    gb = K.WorldBatch()
    for _ in range(n_worlds):
        gb.add_world(m)
    ob = oracle_lib.OracleBatch([om], [0] * n_worlds, n_threads=4)
    p, t, tm = ob.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * n_worlds, seed=seed)
    ob.set_state(p, t, tm)
    gb.set_state(p, t, tm)
    return m, gb, ob


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(1.0, float(np.abs(b).max()))) if b.size else 0.0


@pytest.mark.parametrize("name,steps", [("dr_legs", 60), ("sphere_pile", 15)])
def test_caches_match_oracle(name, steps):
    sc = dr_legs() if name == "dr_legs" else sphere_pile(24)
    cfg = K.config_for(sc)
    m, gb, ob = _jittered(sc, 2)
    seen_limits = seen_contacts = 0
    for k in range(steps):
        gb.step(cfg)
        ob.step(cfg)
        for w in range(2):
            jc, lc, cc = gb.get_caches(w)
            olam, oz, ov, olc, occ = ob.caches(w)
            n = len(jc.lambda_)
            assert jc.valid == ov
            assert _rel(jc.lambda_, olam[:n]) < 1e-9 and _rel(jc.z, oz[:n]) < 1e-9
            assert sorted(lc) == sorted(olc)
            for key in lc:
                assert _rel(lc[key], olc[key]) < 1e-9
            assert [(e.geom_a, e.geom_b) for e in cc] == [(o[0], o[1]) for o in occ]
            for e, o in zip(cc, occ):
                assert np.abs(e.position - o[2]).max() < 1e-12
                assert _rel(e.impulse, o[3]) < 1e-9 and _rel(e.dual, o[4]) < 1e-9
            seen_limits += len(lc)
            seen_contacts += len(cc)
    assert seen_contacts > 0
    if name == "dr_legs":
        assert seen_limits >= 0  # pad limits engage only on some trajectories


@pytest.mark.parametrize("name", ["dr_legs", "sphere_pile", "closed_chain"])
def test_extract_insert_reproduces_next_step_bitwise(name):
    sc = {"dr_legs": dr_legs, "sphere_pile": lambda: sphere_pile(24), "closed_chain": lambda: closed_chain(16)}[name]()
    cfg = K.config_for(sc)
    m, ga, _ = _jittered(sc, 3)
    for _ in range(25):
        ga.step(cfg)
    s = ga.extract_state(1)
    assert s.joint_cache.valid
    gb = K.WorldBatch()
    gb.add_world(m)
    gb.insert_state(0, s)
    for k in range(3):
        ga.step(cfg)
        gb.step(cfg)
        sa, sb = ga.extract_state(1), gb.extract_state(0)
        assert np.array_equal(sa.poses, sb.poses), k
        assert np.array_equal(sa.twists, sb.twists), k
        assert ga.diagnostics()[1].iterations == gb.diagnostics()[0].iterations
        assert ga.diagnostics()[1].cr_iterations == gb.diagnostics()[0].cr_iterations
    # without the caches the restored world cold-starts: a different solve
    cold = K.WorldState(s.poses, s.twists, s.time)
    gc = K.WorldBatch()
    gc.add_world(m, cold)
    gc.step(cfg)
    gd = K.WorldBatch()
    gd.add_world(m, s)
    gd.step(cfg)
    assert gc.diagnostics()[0].iterations != gd.diagnostics()[0].iterations or \
        not np.array_equal(gc.extract_state(0).twists, gd.extract_state(0).twists)


def test_single_world_step_warm_starts_from_state():
    sc = dr_legs()
    cfg = K.config_for(sc)
    m, gb, _ = _jittered(sc, 1)
    state = gb.extract_state(0)
    for k in range(12):
        d = K.step(m, state, cfg)
        gb.step(cfg)
        ref = gb.extract_state(0)
        assert np.array_equal(state.poses, ref.poses), k
        assert np.array_equal(state.twists, ref.twists), k
        assert d.iterations == gb.diagnostics()[0].iterations


def test_set_caches_drops_unmatchable_entries_and_checks_capacity():
    sc = sphere_pile(24)
    m = K.build_model(sc)
    gb = K.WorldBatch()
    gb.add_world(m)
    gb.step(K.config_for(sc))
    jc, lc, cc = gb.get_caches(0)
    bogus = K.ReactionCacheEntry(0, 0, np.zeros(3), np.ones(3), np.ones(3))  # geom 0 with itself: no such pair
    gb.set_caches(0, jc, {(0, 0): (1.0, 1.0)}, cc + [bogus])  # joint 0 does not exist / has no limits
    jc2, lc2, cc2 = gb.get_caches(0)
    assert lc2 == {} and len(cc2) == len(cc)
    too_many = [cc[0]] * (m.info.max_contacts + 1) if cc else []
    if too_many:
        with pytest.raises(K.KaminoError, match="capacity"):
            gb.set_caches(0, jc, {}, too_many)
