"""Supernodal sparse-LLT kernel (kd_sparse.cu) on the device (GPU box only).

The kernel factors the same D_{eta,rho} as the reference's Dense backend
(delassus.cpp:59-104) in the model plan's fill-reducing order; the PADMM loop
is padmm.cpp:87-159 unchanged.  Checks: which kernel ran, agreement with the
fused dense kernel (KD_SPARSE=0) from identical states, trajectory parity with
the CPU oracle, and the per-step fallback to the dense kernel when a world
activates a contact outside the plan."""
import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import _Builder, dr_legs

pytestmark = pytest.mark.gpu


def _batch(sc, n, jitter=True):
    m = K.build_model(sc)
    b = K.WorldBatch()
    for _ in range(n):
        b.add_world(m)
    if jitter:
        p, t, tm = b.get_state()
        t = K.bench_jitter(t, [m.n_bodies] * n, seed=1)
        b.set_state(p, t, tm)
    return b


@pytest.fixture
def force_supernodal(monkeypatch):
    """KD_SPARSE=2: the supernodal kernel for every planned model (Auto keeps
    it for small systems only)."""
    monkeypatch.setenv("KD_SPARSE", "2")


def test_auto_kernel_choice():
    small = _batch(oracle_lib.bundled_scene("fourbar"), 4, jitter=False)
    large = _batch(dr_legs(), 4)
    small.step(K.config_for(oracle_lib.bundled_scene("fourbar")), 2)
    large.step(K.config_for(dr_legs()), 2)
    assert small.kernels() == ["supernodal"] * 4
    assert large.kernels() == ["supernodal+dense"] * 4  # plan factor handed to the dense kernel


def test_dr_legs_runs_supernodal_kernel(force_supernodal):
    sc = dr_legs()
    b = _batch(sc, 16)
    b.step(K.config_for(sc), 3)
    assert b.kernels() == ["supernodal"] * 16
    cyc = b.phase_cycles()
    assert (cyc[:, 0] > 0).all() and (cyc[:, 2] > 0).all() and (cyc[:, 4] > 0).all()


def test_supernodal_matches_dense_kernel_from_identical_states(monkeypatch):
    sc = dr_legs()
    cfg = K.config_for(sc)
    monkeypatch.setenv("KD_SPARSE", "2")
    sn = _batch(sc, 16)
    monkeypatch.setenv("KD_SPARSE", "0")
    de = _batch(sc, 16)
    monkeypatch.delenv("KD_SPARSE")
    worst, same, total = 0.0, 0, 0
    for _ in range(40):
        p, t, tm = sn.get_state()
        de.set_state(p, t, tm)
        sn.step(cfg)
        de.step(cfg)
        assert sn.kernels() == ["supernodal"] * 16 and de.kernels() == ["dense"] * 16
        a, d = sn.impulses(), de.impulses()
        worst = max(worst, float(np.abs(a - d).max() / max(1.0, np.abs(d).max())))
        for gs, gd in zip(sn.diagnostics(), de.diagnostics()):
            assert gs.n_rows == gd.n_rows and gs.contact_count == gd.contact_count
            same += gs.iterations == gd.iterations
            total += 1
    assert worst < 1e-8
    assert same >= 0.98 * total


def test_supernodal_dr_legs_trajectory_vs_oracle(force_supernodal):
    """Same protocol and tolerances as the dense kernel's DR-Legs trajectory
    test (test_parity_gpu.py): 8 worlds x 100 steps."""
    sc = dr_legs()
    cfg = K.config_for(sc)
    n = 8
    gb = _batch(sc, n, jitter=False)
    om = oracle_lib.OracleModel(sc)
    ob = oracle_lib.OracleBatch([om], [0] * n, n_threads=8)
    p, t, tm = ob.get_state()
    t = K.bench_jitter(t, [om.n_bodies] * n, seed=1)
    ob.set_state(p, t, tm)
    gb.set_state(p, t, tm)
    same = total = 0
    for _ in range(100):
        gb.step(cfg)
        ob.step(cfg)
        for dg, do in zip(gb.diagnostics(), ob.diagnostics()):
            assert (dg.n_rows, dg.contact_count, dg.n_limits) == (do.n_rows, do.contact_count, do.n_limits)
            same += dg.iterations == do.iterations
            total += 1
    assert gb.kernels() == ["supernodal"] * n
    assert same >= 0.99 * total
    pg, tg, _ = gb.get_state()
    po, to, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-8
    assert np.abs(tg - to).max() < 1e-6


def test_handoff_matches_dense_kernel_from_identical_states(monkeypatch):
    """The supernodal factor handed to the dense kernel (default for DR-Legs)
    against the dense kernel's own blocked Cholesky (KD_SN_HANDOFF=0)."""
    sc = dr_legs()
    cfg = K.config_for(sc)
    ho = _batch(sc, 16)
    monkeypatch.setenv("KD_SN_HANDOFF", "0")
    de = _batch(sc, 16)
    monkeypatch.delenv("KD_SN_HANDOFF")
    worst, same, total = 0.0, 0, 0
    for _ in range(40):
        p, t, tm = ho.get_state()
        de.set_state(p, t, tm)
        ho.step(cfg)
        de.step(cfg)
        assert set(ho.kernels()) <= {"supernodal+dense", "supernodal+cluster"} and de.kernels() == ["dense"] * 16
        a, d = ho.impulses(), de.impulses()
        worst = max(worst, float(np.abs(a - d).max() / max(1.0, np.abs(d).max())))
        for gh, gd in zip(ho.diagnostics(), de.diagnostics()):
            assert gh.n_rows == gd.n_rows and gh.contact_count == gd.contact_count
            same += gh.iterations == gd.iterations
            total += 1
    assert worst < 1e-8
    assert same >= 0.98 * total


def test_dense_kernel_dr_legs_trajectory_vs_oracle(monkeypatch):
    monkeypatch.setenv("KD_SPARSE", "0")
    sc = dr_legs()
    cfg = K.config_for(sc)
    gb = _batch(sc, 4, jitter=False)
    om = oracle_lib.OracleModel(sc)
    ob = oracle_lib.OracleBatch([om], [0] * 4, n_threads=4)
    p, t, tm = ob.get_state()
    t = K.bench_jitter(t, [om.n_bodies] * 4, seed=1)
    ob.set_state(p, t, tm)
    gb.set_state(p, t, tm)
    for _ in range(60):
        gb.step(cfg)
        ob.step(cfg)
    assert gb.kernels() == ["dense"] * 4
    pg, _, _ = gb.get_state()
    po, _, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-8


def _two_spheres():
    """A pendulum bob resting against a free sphere on a plane: one planned
    body-world pair per sphere and one unplanned sphere-sphere pair."""
    b = _Builder("two_spheres")
    b.body("a", 1.0, (0.2, 0.2, 0.2), (0.0, 0.0, 0.1))
    b.body("b", 1.0, (0.2, 0.2, 0.2), (0.195, 0.0, 0.1))
    b.body("c", 0.5, (0.1, 0.1, 0.1), (0.0, 0.0, 0.5))
    b.joint("hinge", "world", "c", (0.0, 0.0, 0.8), (0.0, 1.0, 0.0))
    b.geom(body="a", shape="sphere", radius=0.1, mu=0.5, restitution=0.0)
    b.geom(body="b", shape="sphere", radius=0.1, mu=0.5, restitution=0.0)
    b.geom(body="world", shape="plane", normal=[0.0, 0.0, 1.0], offset=0.0, mu=0.5, restitution=0.0)
    return b.scene()


def test_unplanned_contact_falls_back_to_dense_kernel(force_supernodal):
    sc = _two_spheres()
    m = K.build_model(sc)
    assert m.sparse_plan_info() is not None
    cfg = K.config_for(sc)
    gb = _batch(sc, 1, jitter=False)
    om = oracle_lib.OracleModel(sc)
    ob = oracle_lib.OracleBatch([om], [0], n_threads=1)
    kinds = set()
    for _ in range(30):
        gb.step(cfg)
        ob.step(cfg)
        kinds.add(gb.kernels()[0])
        dg, do = gb.diagnostics()[0], ob.diagnostics()[0]
        assert (dg.n_rows, dg.contact_count, dg.iterations) == (do.n_rows, do.contact_count, do.iterations)
    assert "dense" in kinds  # the sphere-sphere contact is not in the plan
    pg, _, _ = gb.get_state()
    po, _, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-9


def test_heterogeneous_batch_kernels():
    """Config 3 mix: four-bar, DR-Legs and serial chain worlds in one batch
    under Auto: the four-bars take the supernodal kernel, the larger models the
    supernodal factor + dense solve hand-off, all in one step."""
    scs = [oracle_lib.bundled_scene("fourbar"), dr_legs(), oracle_lib.bundled_scene("serial_chain_10")]
    ms = [K.build_model(s) for s in scs]
    oms = [oracle_lib.OracleModel(s) for s in scs]
    wm = [w % 3 for w in range(12)]
    gb = K.WorldBatch()
    for w in wm:
        gb.add_world(ms[w])
    ob = oracle_lib.OracleBatch(oms, wm, n_threads=8)
    cfg = K.config_for(scs[0])
    for _ in range(20):
        gb.step(cfg)
        ob.step(cfg)
        for dg, do in zip(gb.diagnostics(), ob.diagnostics()):
            assert (dg.n_rows, dg.iterations) == (do.n_rows, do.iterations)
    kinds = gb.kernels()
    assert all(kinds[w] == ("supernodal" if wm[w] == 0 else "supernodal+dense") for w in range(12))
    pg, _, _ = gb.get_state()
    po, _, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-9


def test_cr_world_beyond_shared_memory_uses_hbm_scratch():
    """A 200-sphere pile: its row capacity (3738) puts the shared CR kernel's
    vectors beyond one CTA's shared memory, so they live in a per-world HBM
    slab (the reference's matrix-free solve has no size limit).  Parity vs the
    oracle over a few steps: contact order bit-exact, PADMM iteration counts
    equal, positions within 1e-9."""
    import oracle_lib
    from paper_2603_16536_b200.scenes import sphere_pile
    sc = sphere_pile(200)
    cfg = K.config_for(sc)
    m, om = K.build_model(sc), oracle_lib.OracleModel(sc)
    assert m.info.row_capacity > 2500
    gb = K.WorldBatch()
    gb.add_world(m)
    gb.add_world(m)
    ob = oracle_lib.OracleBatch([om], [0, 0], n_threads=8)
    ob.set_trace(True)
    for _ in range(4):
        gb.step(cfg)
        ob.step(cfg)
        dg, do = gb.diagnostics(), ob.diagnostics()
        for w in range(2):
            assert dg[w].n_rows == do[w].n_rows and dg[w].contact_count == do[w].contact_count
            assert dg[w].iterations == do[w].iterations
        cg, _ = gb.dump_contacts(0)
        co, _ = ob.dump_contacts(0)
        assert (cg == co).all()
    assert gb.kernels() == ["cr", "cr"]
    pg, _, _ = gb.get_state()
    po, _, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-9
