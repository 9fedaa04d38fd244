"""K2c, the dense PADMM loop of hand-off worlds on a CTA pair (GPU box only;
opt-in with KD_CLUSTER=1, measured slower than K2 on DR-Legs).

K2 forms X = L^-1 from the supernodal factor and writes its nonzero tiles to
the world's slab; K2c (kd_dense_cl.cu) splits X's tile rows over the two CTAs
of a cluster and runs padmm_solve (padmm.cpp:87-159) with one DSMEM exchange
of pass-2 partials per iteration.  Its sums are grouped per tile, so it is not
bitwise equal to K2's running sums: the checks are the oracle's (iteration
counts, trajectories) and K2c vs K2 from identical states (impulses within
1e-9, iteration counts equal almost everywhere), plus the determinism the
batch API promises (a world's result does not depend on its batch).
"""
import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import dr_legs

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def cluster_on(monkeypatch):
    monkeypatch.setenv("KD_CLUSTER", "1")


def _batch(sc, n, seed=1):
    m = K.build_model(sc)
    b = K.WorldBatch()
    for _ in range(n):
        b.add_world(m)
    p, t, tm = b.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * n, seed=seed)
    b.set_state(p, t, tm)
    b._ensure()
    return b


def test_dr_legs_takes_the_cluster_kernel_and_k2_without_it(monkeypatch):
    sc = dr_legs()
    cfg = K.config_for(sc)
    cl = _batch(sc, 8)
    monkeypatch.setenv("KD_CLUSTER", "0")
    k2 = _batch(sc, 8)
    monkeypatch.setenv("KD_CLUSTER", "1")
    cl.step(cfg, 2)
    k2.step(cfg, 2)
    assert cl.kernels() == ["supernodal+cluster"] * 8
    assert k2.kernels() == ["supernodal+dense"] * 8


def test_cluster_vs_k2_from_identical_states(monkeypatch):
    sc = dr_legs()
    cfg = K.config_for(sc)
    nw = 296  # two waves of CTA pairs
    cl = _batch(sc, nw)
    monkeypatch.setenv("KD_CLUSTER", "0")
    k2 = _batch(sc, nw)
    monkeypatch.setenv("KD_CLUSTER", "1")
    worst, same, total = 0.0, 0, 0
    for _ in range(30):
        p, t, tm = cl.get_state()
        k2.set_state(p, t, tm)
        cl.step(cfg)
        k2.step(cfg)
        a, d = cl.impulses(), k2.impulses()
        worst = max(worst, float(np.abs(a - d).max() / max(1.0, np.abs(d).max())))
        for gc, gk in zip(cl.diagnostics(), k2.diagnostics()):
            assert (gc.n_rows, gc.contact_count) == (gk.n_rows, gk.contact_count)
            assert gc.converged == gk.converged
            same += gc.iterations == gk.iterations
            total += 1
    assert worst < 1e-9
    assert same >= 0.99 * total


def test_cluster_trajectory_vs_oracle():
    sc = dr_legs()
    cfg = K.config_for(sc)
    m, om = K.build_model(sc), oracle_lib.OracleModel(sc)
    gb = K.WorldBatch()
    for _ in range(6):
        gb.add_world(m)
    ob = oracle_lib.OracleBatch([om], [0] * 6, n_threads=6)
    p, t, tm = ob.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * 6, seed=3)
    ob.set_state(p, t, tm)
    gb.set_state(p, t, tm)
    same = total = 0
    for _ in range(60):
        gb.step(cfg)
        ob.step(cfg)
        for dg, do in zip(gb.diagnostics(), ob.diagnostics()):
            assert (dg.n_rows, dg.contact_count, dg.n_limits) == (do.n_rows, do.contact_count, do.n_limits)
            same += dg.iterations == do.iterations
            total += 1
    assert gb.kernels() == ["supernodal+cluster"] * 6
    assert same >= 0.99 * total
    pg, tg, _ = gb.get_state()
    po, to, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-8
    assert np.abs(tg - to).max() < 1e-6


def test_world_result_independent_of_batch():
    """A world steps bit for bit the same alone and inside a larger batch."""
    sc = dr_legs()
    cfg = K.config_for(sc)
    big = _batch(sc, 150, seed=9)
    p, t, tm = big.get_state()
    solo = K.WorldBatch()
    solo.add_world(K.build_model(sc))
    solo.set_state(p[: p.size // 150], t[: t.size // 150], tm[:1])
    big.step(cfg, 5)
    solo.step(cfg, 5)
    pb, tb, _ = big.get_state()
    ps, ts, _ = solo.get_state()
    assert np.array_equal(pb[: ps.size], ps) and np.array_equal(tb[: ts.size], ts)
