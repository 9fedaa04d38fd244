"""Every joint type and joint-dynamics row on the device (GPU box only).

`mixed_joints()` holds fixed, spherical, revolute and prismatic joints; PD,
armature (R = 1/m_a, v* = rate u) and damping (R = 1/(dt d), v* = 0) rows; a
revolute limit and two prismatic limits inside the 0.001 m linear margin
(constraints.cpp:90-108, 160-187, 218-229, 256-274).  It runs through each
device kernel that can solve it -- the Auto choice (supernodal factor handed to
the dense kernel), the dense kernel alone (KD_SPARSE=0), the supernodal kernel
end to end (KD_SPARSE=2) and the matrix-free CR kernel (backend = sparse) --
against the CPU oracle: row layout, body ids and limit keys bit-exact; J, bias,
R, P, v_f within 1e-12; lambda / z within 1e-9; PADMM iteration counts equal;
240-step trajectories within 1e-9.

`stewart_tower()` is BASELINE config 4 as SURVEY §8d specifies it (a spatial
parallel manipulator: 156 bodies, spherical + prismatic legs, n = 942): CR
path parity vs the oracle.
"""
import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import mixed_joints, stewart_tower

pytestmark = pytest.mark.gpu

MODES = {  # name -> (env KD_SPARSE, backend, expected kernel)
    "auto": (None, "auto", "supernodal+dense"),
    "dense": ("0", "auto", "dense"),
    "supernodal": ("2", "auto", "supernodal"),
    "cr": (None, "sparse", "cr"),
}


def rel(a, b):
    return float(np.abs(a - b).max() / max(1.0, float(np.abs(b).max()))) if len(b) else 0.0


def _pair(sc, n_worlds, monkeypatch, sparse_env=None, seed=5):
    if sparse_env is not None:
        monkeypatch.setenv("KD_SPARSE", sparse_env)
    m, om = K.build_model(sc), oracle_lib.OracleModel(sc)
    gb = K.WorldBatch()
    for _ in range(n_worlds):
        gb.add_world(m)
    ob = oracle_lib.OracleBatch([om], [0] * n_worlds, n_threads=4)
    p, t, tm = ob.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * n_worlds, seed=seed)
    ob.set_state(p, t, tm)
    gb.set_state(p, t, tm)
    gb._ensure()  # created under the env setting
    monkeypatch.delenv("KD_SPARSE", raising=False)
    return gb, ob


def _rows_match(gb, ob, w, tol=1e-12):
    rg, ro = gb.dump_rows(w), ob.dump_rows(w)
    assert len(rg["kind"]) == len(ro["kind"])
    assert (rg["body"] == ro["body"]).all()
    assert (rg["kind"] == ro["kind"]).all()
    for key in ("J", "bias", "reg", "scale", "vf"):
        assert rel(rg[key], ro[key]) < tol, key
    for key in ("lambda", "z"):
        assert rel(rg[key], ro[key]) < 1e-9, key
    assert (gb.dump_limits(w) == ob.dump_limits(w)).all()
    return rg


@pytest.mark.parametrize("mode", list(MODES))
def test_mixed_joints_match_oracle(mode, monkeypatch):
    env, backend, kernel = MODES[mode]
    sc = mixed_joints()
    cfg = K.config_for(sc)
    cfg.backend = backend
    gb, ob = _pair(sc, 2, monkeypatch, env)
    ob.set_trace(True)
    kinds_seen = set()
    for k in range(240):
        gb.step(cfg)
        ob.step(cfg)
        dg, do = gb.diagnostics(), ob.diagnostics()
        for w in range(2):
            assert (dg[w].n_rows, dg[w].n_limits) == (do[w].n_rows, do[w].n_limits)
            assert dg[w].iterations == do[w].iterations, (k, w)
            if backend == "sparse":
                assert abs(dg[w].cr_iterations - do[w].cr_iterations) <= 2
        if k < 4 or k % 60 == 0:
            for w in range(2):
                rg = _rows_match(gb, ob, w)
                kinds_seen.update(int(x) for x in rg["kind"])
    assert gb.kernels() == [kernel, kernel]
    assert kinds_seen == {0, 1}  # bilateral/joint-dynamics and limit rows
    pg, tg, _ = gb.get_state()
    po, to, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-9
    assert np.abs(tg - to).max() < 1e-8


def test_mixed_joints_row_values():
    """Known answers of the joint-dynamics rows (test_constraints.cpp:132-183):
    PD R = 1/(dt (dt kp + kd)), armature R = 1/m_a, damping R = 1/(dt d); the
    active prismatic limits carry keys (joint, 0) and gap-driven bias."""
    sc = mixed_joints()
    cfg = K.config_for(sc)
    m = K.build_model(sc)
    gb = K.WorldBatch()
    gb.add_world(m)
    gb.step(cfg)
    rg = gb.dump_rows(0)
    dt = cfg.dt
    reg = rg["reg"][m.n_bilateral_rows: m.n_bilateral_rows + m.n_dynamics_rows]
    expect = [1.0 / (dt * (dt * 20.0 + 1.0)), 1.0 / 0.05, 1.0 / (dt * 0.1), 1.0 / 0.2, 1.0 / (dt * 0.5)]
    assert np.allclose(reg, expect, rtol=1e-14, atol=0)
    keys = gb.dump_limits(0)
    assert [tuple(k) for k in keys] == [(4, 0), (5, 0)]  # plunge and slide_y lower bounds


def test_stewart_tower_cr_parity(monkeypatch):
    sc = stewart_tower()
    cfg = K.config_for(sc)
    gb, ob = _pair(sc, 2, monkeypatch)
    ob.set_trace(True)
    for k in range(8):
        gb.step(cfg)
        ob.step(cfg)
        dg, do = gb.diagnostics(), ob.diagnostics()
        for w in range(2):
            assert dg[w].n_rows == do[w].n_rows and dg[w].n_limits == do[w].n_limits
            assert dg[w].iterations == do[w].iterations, (k, w)
            assert abs(dg[w].cr_iterations - do[w].cr_iterations) <= 2
        if k < 2:  # identical inputs at k = 0; after one step the states differ at rounding level
            _rows_match(gb, ob, 0, 1e-12 if k == 0 else 1e-9)
    assert gb.kernels() == ["cr", "cr"]
    pg, tg, _ = gb.get_state()
    po, to, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-8
    assert np.abs(tg - to).max() < 1e-6
