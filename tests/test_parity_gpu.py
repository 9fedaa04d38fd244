"""Device path vs CPU oracle (GPU box only).

Parity protocol: (i) the oracle passes the reference KATs
(test_oracle.py); (ii) one-step parity: same input state -> row count, row
kinds, body ids, limit keys and contact (geom_a, geom_b) order bit-exact; J,
bias, R, P, v_f within 1e-12 relative, solver lambda/z within 1e-9 relative;
(iii) N-step trajectories and PADMM iteration counts; (iv) residual histories
in fixed-iteration mode.  Tolerances: the device uses FMA contraction and a
blocked factorization, the oracle neither, so agreement is ulp-level per step
and grows only as the dynamics amplify it.
"""
import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import closed_chain, dr_legs, sphere_pile

pytestmark = pytest.mark.gpu

BUNDLED = ["fourbar", "double_fourbar", "serial_chain_10", "pendulum", "sphere_on_plane", "inclined_box", "freefall"]


def scene(name):
    if name == "dr_legs":
        return dr_legs()
    if name == "closed_chain":
        return closed_chain(16)
    if name == "sphere_pile":
        return sphere_pile(40)
    return oracle_lib.bundled_scene(name)


def pair(sc, n_worlds=1, jitter=False, threads=8):
    m, om = K.build_model(sc), oracle_lib.OracleModel(sc)
    gb = K.WorldBatch()
    for _ in range(n_worlds):
        gb.add_world(m)
    ob = oracle_lib.OracleBatch([om], [0] * n_worlds, n_threads=threads)
    if jitter:
        p, t, tm = ob.get_state()
        t = K.bench_jitter(t, [m.n_bodies] * n_worlds, seed=1)
        ob.set_state(p, t, tm)
        gb.set_state(p, t, tm)
    return gb, ob


def rel(a, b):
    return float(np.abs(a - b).max() / max(1.0, float(np.abs(b).max()))) if len(b) else 0.0


@pytest.mark.parametrize("name", BUNDLED + ["dr_legs", "closed_chain", "sphere_pile"])
def test_one_step_rows_match_oracle(name):
    sc = scene(name)
    cfg = K.config_for(sc)
    gb, ob = pair(sc, jitter=name == "dr_legs")
    ob.set_trace(True)
    for _ in range(3):  # a few steps so warm-start caches are exercised too
        gb.step(cfg)
        ob.step(cfg)
        rg, ro = gb.dump_rows(0), ob.dump_rows(0)
        assert len(rg["kind"]) == len(ro["kind"])
        assert (rg["body"] == ro["body"]).all()
        assert (rg["kind"] == ro["kind"]).all()
        for key in ("J", "bias", "reg", "scale", "vf"):
            assert rel(rg[key], ro[key]) < 1e-12, key
        for key in ("lambda", "z"):
            assert rel(rg[key], ro[key]) < 1e-9, key
        cg, cdg = gb.dump_contacts(0)
        co, cdo = ob.dump_contacts(0)
        assert (cg == co).all()
        if len(cdo):
            assert np.abs(cdg - cdo).max() < 1e-12
        assert (gb.dump_limits(0) == ob.dump_limits(0)).all()
        dg, do = gb.diagnostics()[0], ob.diagnostics()[0]
        assert (dg.n_rows, dg.contact_count, dg.n_limits, dg.first_contact_row) == \
               (do.n_rows, do.contact_count, do.n_limits, do.first_contact_row)
        assert dg.iterations == do.iterations
        assert dg.converged == do.converged


@pytest.mark.parametrize("name,steps", [("fourbar", 2400), ("double_fourbar", 480), ("serial_chain_10", 480),
                                        ("pendulum", 480), ("sphere_on_plane", 480), ("inclined_box", 480),
                                        ("freefall", 240)])
def test_trajectory_parity(name, steps):
    sc = scene(name)
    cfg = K.config_for(sc)
    gb, ob = pair(sc)
    iters_g = iters_o = 0
    for k in range(steps):
        gb.step(cfg)
        ob.step(cfg)
        dg, do = gb.diagnostics()[0], ob.diagnostics()[0]
        assert dg.n_rows == do.n_rows and dg.contact_count == do.contact_count
        iters_g += dg.iterations
        iters_o += do.iterations
    pg, tg, tmg = gb.get_state()
    po, to, tmo = ob.get_state()
    assert np.abs(pg - po).max() < 1e-9
    assert np.abs(tg - to).max() < 1e-8
    assert np.abs(tmg - tmo).max() < 1e-12
    assert iters_g == iters_o


def test_dr_legs_trajectory_parity():
    sc = dr_legs()
    cfg = K.config_for(sc)
    gb, ob = pair(sc, n_worlds=8, jitter=True)
    same_iters = total = 0
    for k in range(100):
        gb.step(cfg)
        ob.step(cfg)
        dg, do = gb.diagnostics(), ob.diagnostics()
        for w in range(8):
            assert dg[w].n_rows == do[w].n_rows
            assert dg[w].contact_count == do[w].contact_count
            assert dg[w].n_limits == do[w].n_limits
            same_iters += dg[w].iterations == do[w].iterations
            total += 1
    assert same_iters >= 0.99 * total
    pg, tg, _ = gb.get_state()
    po, to, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-8
    assert np.abs(tg - to).max() < 1e-6


@pytest.mark.parametrize("name", ["serial_chain_10", "dr_legs", "sphere_on_plane"])
def test_residual_history_parity_fixed_mode(name):
    sc = scene(name)
    cfg = K.config_for(sc)
    cfg.fixed_iteration_mode = True
    cfg.max_iters = 17
    gb, ob = pair(sc, jitter=name == "dr_legs")
    gb.set_history_capacity(32)
    ob.set_trace(True)
    for _ in range(3):
        gb.step(cfg)
        ob.step(cfg)
        hg, ho = gb.history()[0], ob.history(32)[0]
        assert gb.diagnostics()[0].iterations == 17 == ob.diagnostics()[0].iterations
        assert (hg[17:] == -1).all() and (ho[17:] == -1).all()
        assert np.all(np.abs(hg[:17] - ho[:17]) <= 1e-9 * np.maximum(1e-3, np.abs(ho[:17])) + 1e-13)


@pytest.mark.parametrize("cr_iters", [9, 50])
def test_matrix_free_fourbar_parity(cr_iters):
    sc = scene("fourbar")
    cfg = K.config_for(sc)
    cfg.backend = "sparse"
    cfg.cr_iters = cr_iters
    gb, ob = pair(sc)
    same = 0
    for _ in range(240):
        gb.step(cfg)
        ob.step(cfg)
        dg, do = gb.diagnostics()[0], ob.diagnostics()[0]
        assert dg.iterations == do.iterations
        # the CR breakdown guard (r.Ar <= 1e-30 |rhs|^2, delassus.cpp:166-172) can
        # fire one inner iteration apart once the residual is at rounding level
        assert abs(dg.cr_iterations - do.cr_iterations) <= 2
        same += dg.cr_iterations == do.cr_iterations
    assert same >= 0.95 * 240
    pg, tg, _ = gb.get_state()
    po, to, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-9 and np.abs(tg - to).max() < 1e-8


def test_closed_chain_cr_path_parity():
    sc = closed_chain(16)
    cfg = K.config_for(sc)
    gb, ob = pair(sc)
    for _ in range(20):
        gb.step(cfg)
        ob.step(cfg)
        dg, do = gb.diagnostics()[0], ob.diagnostics()[0]
        assert dg.n_rows == do.n_rows > 300  # Auto -> matrix-free
        assert dg.cr_iterations > 0
    pg, tg, _ = gb.get_state()
    po, to, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-7 and np.abs(tg - to).max() < 1e-5


def test_sphere_pile_contact_indexing():
    sc = sphere_pile(40)
    cfg = K.config_for(sc)
    gb, ob = pair(sc)
    ob.set_trace(True)
    for _ in range(10):
        gb.step(cfg)
        ob.step(cfg)
        cg, _ = gb.dump_contacts(0)
        co, _ = ob.dump_contacts(0)
        assert cg.shape == co.shape and (cg == co).all()
    pg, _, _ = gb.get_state()
    po, _, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-9


def test_dense_vs_matrix_free_on_device():
    """Acceptance #2 (acceptance.cpp:114-135) on the device: same state and
    caches solved both ways, impulses within 1e-6 relative."""
    sc = scene("fourbar")
    cfg = K.config_for(sc)
    m = K.build_model(sc)
    dense, sparse = K.WorldBatch(), K.WorldBatch()
    dense.add_world(m)
    sparse.add_world(m)
    cd = K.StepConfig(**{**cfg.__dict__, "backend": "dense"})
    cs = K.StepConfig(**{**cfg.__dict__, "backend": "sparse", "cr_iters": 50})
    worst = 0.0
    for _ in range(100):
        p, t, tm = dense.get_state()
        sparse.set_state(p, t, tm)
        sparse.reset_caches()
        dense.reset_caches()
        dense.step(cd)
        sparse.step(cs)
        a = dense.impulses()[:21]
        b = sparse.impulses()[:21]
        worst = max(worst, float(np.abs(a - b).max() / max(1e-9, np.abs(a).max())))
    assert worst <= 1e-6


@pytest.mark.parametrize("cells,steps", [(16, 20), (22, 12)])
def test_cr_kernel_paths_vs_oracle(cells, steps):
    """Every matrix-free kernel path (incidence owners, row owners; selected by
    the world's size and body degrees) against the oracle: same row counts and
    PADMM iterations per step, CR counts within +-2, poses after N steps."""
    sc = closed_chain(cells)
    cfg = K.config_for(sc)
    gb, ob = pair(sc, n_worlds=2, jitter=True)
    paths = set()
    for _ in range(steps):
        gb.step(cfg)
        ob.step(cfg)
        paths.update(gb.cr_paths())
        for dg, do in zip(gb.diagnostics()[:2], ob.diagnostics()[:2]):
            assert dg.n_rows == do.n_rows > 300
            assert dg.iterations == do.iterations
            assert abs(dg.cr_iterations - do.cr_iterations) <= 2
    assert paths <= {"incidence", "rows"} and paths, paths
    if cells == 22:  # 440 rows, rails of degree 15 -> 3 lanes of 5: fits 256 lanes
        assert paths == {"incidence"}
    pg, tg, _ = gb.get_state()
    po, to, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-7 and np.abs(tg - to).max() < 1e-5


@pytest.mark.parametrize("scene_expr", ["closed_chain(22)", "sphere_pile(100)"])
def test_cr_incidence_vs_rows_kernels(scene_expr):
    """The incidence-owner and row-owner kernels on the same states (the
    second via KD_CR_REG=3 in a subprocess): impulses within 1e-9 relative.
    closed_chain(22): 440 rows, 256 x 2 launch; sphere_pile(100): 780 rows,
    256 x 4 launch with pieces of up to 8 incidences."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import closed_chain, sphere_pile
sc = eval(sys.argv[2])
cfg = K.config_for(sc)
m = K.build_model(sc)
b = K.WorldBatch()
for _ in range(4):
    b.add_world(m)
p, t, tm = b.get_state()
t = K.bench_jitter(t, [m.n_bodies] * 4, seed=3)
b.set_state(p, t, tm)
b.step(cfg, 5)
print(json.dumps({"paths": b.cr_paths(), "imp": b.impulses().tolist(),
                  "it": [d.iterations for d in b.diagnostics()[:4]]}))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("1", "3"):
        env = dict(os.environ, KD_CR_REG=mode)
        r = subprocess.run([sys.executable, "-c", code, root, scene_expr], env=env, capture_output=True, text=True,
                           check=True)
        out[mode] = json.loads(r.stdout.strip().splitlines()[-1])
    assert set(out["1"]["paths"]) == {"incidence"} and set(out["3"]["paths"]) == {"rows"}
    assert out["1"]["it"] == out["3"]["it"]
    a, b = np.array(out["1"]["imp"]), np.array(out["3"]["imp"])
    assert np.abs(a - b).max() <= 1e-9 * max(1.0, np.abs(b).max())


def test_sphere_pile_768_row_path_vs_oracle():
    """The 513..1024-row CR launch (incidence owners, 256 x 4) on the full
    100-sphere pile against the oracle: contact order bit-exact, the same row
    counts and PADMM iteration counts, poses after 3 steps within 1e-9."""
    sc = sphere_pile(100)
    cfg = K.config_for(sc)
    gb, ob = pair(sc)
    ob.set_trace(True)
    for _ in range(3):
        gb.step(cfg)
        ob.step(cfg)
        cg, _ = gb.dump_contacts(0)
        co, _ = ob.dump_contacts(0)
        assert cg.shape == co.shape and (cg == co).all()
        dg, do = gb.diagnostics()[0], ob.diagnostics()[0]
        assert dg.n_rows == do.n_rows > 512
        assert dg.iterations == do.iterations
    assert gb.cr_paths() == ["incidence"]
    pg, _, _ = gb.get_state()
    po, _, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-9
