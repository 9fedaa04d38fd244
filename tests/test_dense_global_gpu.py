"""Dense backend beyond the shared-memory class (GPU box only).

Worlds whose row capacity exceeds the dense kernel's shared-memory class (232
rows) factor D in a per-world HBM slab (`dense_kernel<256, true>`).  Under
Auto that covers 233..300 rows (build_backend's crossover, delassus.cpp:204-206);
with backend = Dense it covers every n (delassus.cpp:203-216: the reference
factors densely at any size).  The ladder `closed_chain(k)` has 20 k rows, all
bilateral, so k = 14 (280 rows) also has more cone units than the kernel has
threads (256): each thread loops over its units.

Checks, against the CPU oracle on the same inputs: row layout bit-exact, J /
bias / R / P / v_f within 1e-12, lambda / z within 1e-9, equal PADMM iteration
counts every step, trajectories within 1e-8 (1e-7 for the 440-row ladder).
"""
import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import closed_chain

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(a - b).max() / max(1.0, float(np.abs(b).max()))) if len(b) else 0.0


def _pair(sc, n_worlds=2):
    m, om = K.build_model(sc), oracle_lib.OracleModel(sc)
    gb = K.WorldBatch()
    for _ in range(n_worlds):
        gb.add_world(m)
    ob = oracle_lib.OracleBatch([om], [0] * n_worlds, n_threads=4)
    p, t, tm = ob.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * n_worlds, seed=3)
    ob.set_state(p, t, tm)
    gb.set_state(p, t, tm)
    return gb, ob


def _check_rows(gb, ob, w):
    rg, ro = gb.dump_rows(w), ob.dump_rows(w)
    assert len(rg["kind"]) == len(ro["kind"])
    assert (rg["body"] == ro["body"]).all()
    assert (rg["kind"] == ro["kind"]).all()
    for key in ("J", "bias", "reg", "scale", "vf"):
        assert rel(rg[key], ro[key]) < 1e-12, key
    for key in ("lambda", "z"):
        assert rel(rg[key], ro[key]) < 1e-9, key


@pytest.mark.parametrize("cells,backend,steps,tol", [(12, "auto", 120, 1e-8), (14, "auto", 120, 1e-8),
                                                     (22, "dense", 40, 1e-7)])
def test_dense_global_matches_oracle(cells, backend, steps, tol):
    sc = closed_chain(cells)
    cfg = K.config_for(sc)
    cfg.backend = backend
    gb, ob = _pair(sc)
    ob.set_trace(True)
    for k in range(steps):
        gb.step(cfg)
        ob.step(cfg)
        dg, do = gb.diagnostics(), ob.diagnostics()
        for w in range(2):
            assert dg[w].n_rows == do[w].n_rows == 20 * cells
            assert dg[w].iterations == do[w].iterations, (k, w)
            assert dg[w].converged == do[w].converged
        if k < 3 or k == steps - 1:
            for w in range(2):
                _check_rows(gb, ob, w)
    assert gb.kernels() == ["dense", "dense"]
    pg, tg, _ = gb.get_state()
    po, to, _ = ob.get_state()
    assert np.abs(pg - po).max() < tol
    assert np.abs(tg - to).max() < 100 * tol


def test_dense_global_residual_history_fixed_mode():
    """280 rows (> 256 threads): the per-iteration combined residual of the
    unit-looping PADMM equals the oracle's (padmm_solve combined_history)."""
    sc = closed_chain(14)
    cfg = K.config_for(sc)
    cfg.fixed_iteration_mode = True
    cfg.max_iters = 25
    gb, ob = _pair(sc, n_worlds=1)
    gb.set_history_capacity(32)
    ob.set_trace(True)
    for _ in range(3):
        gb.step(cfg)
        ob.step(cfg)
    hg, ho = gb.history()[0], ob.history(32)[0]
    assert (hg[:25] > 0).all() and (hg[25:] == -1).all()
    assert np.abs(hg[:25] - ho[:25]).max() / max(1e-300, np.abs(ho[:25]).max()) < 1e-9


def test_dense_and_matrix_free_agree_above_crossover():
    """The reference compares the two backends on one world
    (test_stepper.cpp:295-316: 480 steps, cr_iters 50, positions within 1e-6);
    here on the 440-row ladder, which needs the dense slab beyond 300 rows."""
    sc = closed_chain(22)
    m = K.build_model(sc)
    dense, sparse = K.config_for(sc), K.config_for(sc)
    dense.backend = "dense"
    sparse.backend = "sparse"
    sparse.cr_iters = 50
    gd, gs = K.WorldBatch(), K.WorldBatch()
    gd.add_world(m)
    gs.add_world(m)
    worst = 0.0
    for _ in range(120):
        gd.step(dense)
        gs.step(sparse)
        pd, _, _ = gd.get_state()
        ps, _, _ = gs.get_state()
        worst = max(worst, float(np.abs(pd - ps).max()))
    assert gd.kernels() == ["dense"] and gs.kernels() == ["cr"]
    assert worst < 1e-6


def test_slab_sweep_kernel_bitwise(monkeypatch):
    """The sweep kernel (one CTA tests 256 worlds' backends and runs the slab
    worlds among them in turn; the default for slab bins of planned models,
    whose worlds land there only as a fallback) gives the per-world slab
    kernel's results bit for bit (KD_SLAB_SWEEP=1 forces it)."""
    import numpy as np
    import paper_2603_16536_b200 as K
    from paper_2603_16536_b200.scenes import closed_chain
    sc = closed_chain(12)
    cfg = K.config_for(sc)
    res = []
    for force in ("0", "1"):
        monkeypatch.setenv("KD_SLAB_SWEEP", force)
        m = K.build_model(sc)
        b = K.WorldBatch()
        for _ in range(300):
            b.add_world(m)
        p, t, tm = b.get_state()
        t = K.bench_jitter(t, [m.n_bodies] * 300, seed=2)
        b.set_state(p, t, tm)
        b.step(cfg, 6)
        p, t, _ = b.get_state()
        res.append((p, t, [d.iterations for d in b.diagnostics()], b.kernels()))
    monkeypatch.delenv("KD_SLAB_SWEEP")
    assert res[0][3] == res[1][3] and "dense" in res[0][3][0]
    assert res[0][2] == res[1][2]
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
