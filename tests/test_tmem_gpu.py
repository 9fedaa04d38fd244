"""K2's tensor-memory solve tiles (GPU box only).

The dense kernel parks the dataflow solve's tiles of X = L^-1 in TMEM
(tcgen05.alloc/st/ld, kd_dense.cu tm_load / tm_dot_*) and reads them with the
same dot-product order as the shared-memory and register tiles, so a batch
stepped with KD_TMEM=0 (tiles from shared memory only) or KD_DENSE_DF=0 (the
barrier version of the passes) must give the same states, impulses and
iteration counts as the default path, bit for bit (up to the sign of exact
zeros, which == ignores).  Covers the supernodal hand-off (DR-Legs, T = 7
tile rows, a structured X mask) and plain dense worlds (the capacity-class K2
with contacts, full X mask).
"""
import numpy as np
import pytest

import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import dr_legs

pytestmark = pytest.mark.gpu


def _batch(sc, n, seed=3):
    m = K.build_model(sc)
    b = K.WorldBatch()
    for _ in range(n):
        b.add_world(m)
    p, t, tm = b.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * n, seed=seed)
    b.set_state(p, t, tm)
    b._ensure()
    return b


def _run(monkeypatch, sc, n, steps, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    b = _batch(sc, n)
    for k in env:
        monkeypatch.delenv(k)
    cfg = K.config_for(sc)
    its = []
    for _ in range(steps):
        b.step(cfg, 1)
        its.append([d.iterations for d in b.diagnostics()])
    p, t, _ = b.get_state()
    return p, t, np.array(its), b.kernels()


@pytest.mark.parametrize("env", [{"KD_TMEM": "0"}, {"KD_DENSE_DF": "0"}])
def test_dr_legs_handoff_tmem_tiles_bitwise(monkeypatch, env):
    sc = dr_legs()
    p0, t0, i0, k0 = _run(monkeypatch, sc, 300, 12, {})
    p1, t1, i1, k1 = _run(monkeypatch, sc, 300, 12, env)
    assert k0 == k1 == ["supernodal+dense"] * 300
    assert np.array_equal(i0, i1)
    assert np.array_equal(p0, p1) and np.array_equal(t0, t1)


def test_plain_dense_worlds_tmem_tiles_bitwise(monkeypatch):
    # KD_SPARSE=0: DR-Legs without its supernodal plan runs the plain K2
    # (Gram + blocked Cholesky in the kernel; n ~ 214 -> the 256-thread
    # class, full X mask, T from the step's rows incl. foot contacts)
    sc = dr_legs()
    p0, t0, i0, k0 = _run(monkeypatch, sc, 300, 12, {"KD_SPARSE": "0"})
    p1, t1, i1, k1 = _run(monkeypatch, sc, 300, 12, {"KD_SPARSE": "0", "KD_TMEM": "0"})
    assert k0 == k1 == ["dense"] * 300
    assert np.array_equal(i0, i1)
    assert np.array_equal(p0, p1) and np.array_equal(t0, t1)
