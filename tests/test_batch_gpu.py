"""WorldBatch semantics on the device (batch.hpp:14-58, test_batch.cpp) and the
reference acceptance criteria re-run on the device path (acceptance.cpp)."""
import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import dr_legs

pytestmark = pytest.mark.gpu


def load(name):
    sc = oracle_lib.bundled_scene(name)
    return sc, K.build_model(sc)


def test_two_identical_worlds_stay_bitwise_identical():
    _, m = load("fourbar")
    b = K.WorldBatch()
    b.add_world(m)
    b.add_world(m)
    for _ in range(100):
        b.step(K.StepConfig())
    s0, s1 = b.extract_state(0), b.extract_state(1)
    assert np.array_equal(s0.poses, s1.poses) and np.array_equal(s0.twists, s1.twists)


def test_heterogeneous_batch_equals_solo_runs_bitwise():
    names = ["fourbar", "sphere_on_plane", "freefall", "serial_chain_10"]
    models = [load(n)[1] for n in names]
    batch = K.WorldBatch()
    for m in models:
        batch.add_world(m)
    solo = []
    for m in models:
        s = K.WorldBatch()
        s.add_world(m)
        solo.append(s)
    for _ in range(200):
        batch.step(K.StepConfig())
        for s in solo:
            s.step(K.StepConfig())
    for w, s in enumerate(solo):
        a, b = batch.extract_state(w), s.extract_state(0)
        assert np.array_equal(a.poses, b.poses) and np.array_equal(a.twists, b.twists)


def test_mixed_dr_legs_batch_matches_solo_bitwise():
    legs = K.build_model(dr_legs())
    _, fb = load("fourbar")
    batch = K.WorldBatch()
    for m in (legs, fb, legs):
        batch.add_world(m)
    solo = K.WorldBatch()
    solo.add_world(legs)
    cfg = K.config_for(dr_legs())
    for _ in range(20):
        batch.step(cfg)
        solo.step(cfg)
    a, b = batch.extract_state(2), solo.extract_state(0)
    assert np.array_equal(a.poses, b.poses)


def test_inactive_worlds_are_skipped():
    _, m = load("freefall")
    b = K.WorldBatch()
    b.add_world(m)
    b.add_world(m)
    b.set_active(0, False)
    b.step(K.StepConfig())
    assert b.extract_state(0).time == 0.0
    assert abs(b.extract_state(1).time - 1.0 / 240.0) < 1e-15
    assert not b.active(0)
    assert b.converged(1)


def test_offsets_are_prefix_sums():
    _, fb = load("fourbar")
    _, sp = load("sphere_on_plane")
    b = K.WorldBatch()
    for m in (fb, sp, fb):
        b.add_world(m)
    assert [b.pose_offset(w) for w in range(3)] == [0, 21, 28]
    assert [b.twist_offset(w) for w in range(3)] == [0, 18, 24]
    assert len(b.pose_storage()) == 49


def test_insert_extract_roundtrip():
    _, fb = load("fourbar")
    b = K.WorldBatch()
    b.add_world(fb)
    s = b.extract_state(0)
    s.twists[1, 2] = 0.25
    s.time = 3.0
    b.insert_state(0, s)
    s2 = b.extract_state(0)
    assert s2.twists[1, 2] == 0.25 and s2.time == 3.0


# ---------------------------------------------------------------- acceptance
ALL = ["freefall", "pendulum", "sphere_on_plane", "inclined_box", "fourbar", "double_fourbar", "serial_chain_10"]


def test_acc1_kkt_momentum_balance():
    worst = 0.0
    for name in ALL:
        sc, m = load(name)
        b = K.WorldBatch()
        b.add_world(m)
        cfg = K.config_for(sc)
        for _ in range(480):
            b.step(cfg)
            worst = max(worst, b.diagnostics()[0].kkt_momentum_inf)
    assert worst <= 1e-5


def test_acc5_loop_closure():
    for name in ("fourbar", "double_fourbar"):
        sc, m = load(name)
        om = oracle_lib.OracleModel(sc)
        b = K.WorldBatch()
        b.add_world(m)
        cfg = K.config_for(sc)
        worst = 0.0
        for _ in range(2400):
            b.step(cfg)
            worst = max(worst, b.diagnostics()[0].f_inf)
        assert worst < 1e-4


def test_acc7_freefall_closed_form():
    sc, m = load("freefall")
    b = K.WorldBatch()
    b.add_world(m)
    b.add_world(m)
    for _ in range(240):
        b.step(K.StepConfig())
    s = b.extract_state(0)
    n, g, dt = 240, 9.81, 1.0 / 240.0
    assert abs(s.twists[0, 2] + g * n * dt) < 1e-9
    assert abs(s.poses[0, 2] + g * dt * dt * n * (n + 1) / 2) < 1e-9
    assert np.array_equal(s.poses, b.extract_state(1).poses)


def test_acc10_warm_start_halves_iterations():
    sc, m = load("sphere_on_plane")
    warm, cold = K.WorldBatch(), K.WorldBatch()
    warm.add_world(m)
    cold.add_world(m)
    cw = K.StepConfig()
    cc = K.StepConfig(warm_start=False)
    wi = ci = 0
    for _ in range(200):
        warm.step(cw)
        cold.step(cc)
        wi += warm.diagnostics()[0].iterations
        ci += cold.diagnostics()[0].iterations
    assert wi <= 0.5 * ci
    s = warm.extract_state(0)
    assert abs(s.poses[0, 2] - 0.1) < 1e-4


def test_acc3_iteration_budget():
    for name in ("sphere_on_plane", "fourbar"):
        sc, m = load(name)
        b = K.WorldBatch()
        b.add_world(m)
        cfg = K.config_for(sc)
        worst = 0
        for k in range(2400):
            b.step(cfg)
            if k >= 10:
                worst = max(worst, b.diagnostics()[0].iterations)
        assert worst <= 30


def test_dr_legs_kkt_and_convergence_at_scale():
    sc = dr_legs()
    m = K.build_model(sc)
    b = K.WorldBatch()
    for _ in range(256):
        b.add_world(m)
    p, t, tm = b.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * 256, seed=1)
    b.set_state(p, t, tm)
    cfg = K.config_for(sc)
    b.step(cfg, 60)
    d = b.diagnostics()
    assert max(d[w].kkt_momentum_inf for w in range(256)) < 1e-5
    assert np.mean([d[w].converged for w in range(256)]) > 0.9
    assert max(d[w].f_inf for w in range(256)) < 1e-3


@pytest.mark.parametrize("workload,nw,steps", [("dr_legs", 4096, 3), ("closed_chain", 1024, 3)])
def test_full_size_batch_equals_sampled_solo_runs(workload, nw, steps):
    """BASELINE sizes (4096 DR-Legs worlds on the dense path, 1024 closed-chain
    worlds on the matrix-free path): every sampled world of the full batch is
    bitwise equal to the same world stepped in a small batch (no cross-world
    interaction, no dependence on batch size or launch shape), and the momentum
    balance (KKT) holds in every world."""
    from paper_2603_16536_b200.scenes import closed_chain
    sc = dr_legs() if workload == "dr_legs" else closed_chain(22)
    m = K.build_model(sc)
    cfg = K.config_for(sc)
    b = K.WorldBatch()
    for _ in range(nw):
        b.add_world(m)
    p, t, tm = b.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * nw, seed=1)
    b.set_state(p, t, tm)
    sample = [0, nw // 3, nw // 2 + 7, nw - 1]
    s = K.WorldBatch()
    for _ in sample:
        s.add_world(m)
    np_, nt_ = 7 * m.n_bodies, 6 * m.n_bodies
    s.set_state(np.concatenate([p[w * np_:(w + 1) * np_] for w in sample]),
                np.concatenate([t[w * nt_:(w + 1) * nt_] for w in sample]), tm[sample])
    b.step(cfg, steps)
    s.step(cfg, steps)
    pb, tb, _ = b.get_state()
    ps, ts, _ = s.get_state()
    for k, w in enumerate(sample):
        assert (pb[w * np_:(w + 1) * np_] == ps[k * np_:(k + 1) * np_]).all()
        assert (tb[w * nt_:(w + 1) * nt_] == ts[k * nt_:(k + 1) * nt_]).all()
    d = b.diagnostics()
    assert max(d[w].kkt_momentum_inf for w in range(nw)) < 1e-5
    assert len(set(b.kernels())) == 1


def test_empty_batch_steps_and_reports_nothing():
    b = K.WorldBatch()
    cfg = K.StepConfig()
    b.step(cfg, 3)
    p, t, tm = b.get_state()
    assert len(p) == 0 and len(t) == 0 and len(tm) == 0


def test_contact_capacity_overflow_is_reported():
    """A pile whose boxes touch on every side makes more contacts than the
    per-world capacity (8 per geom + 16 with box-box pairs): the step fails
    with KD_ERR_CAPACITY instead of dropping contacts silently."""
    from paper_2603_16536_b200.scenes import box_pile
    sc = box_pile(64, gap=0.0)
    m = K.build_model(sc)
    b = K.WorldBatch()
    b.add_world(m)
    with pytest.raises(K.KaminoError) as e:
        b.step(K.config_for(sc), 1)
    assert "capacity" in str(e.value)
