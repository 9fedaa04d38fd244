"""Box-box narrow phase on the device (KD_EXT_BOX_BOX extension) against the
oracle's restatement of the same algorithm (parity unpinned: the reference
rejects box-box pairs, model.cpp:56-62)."""
import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import box_pile
from test_box_box import CASES

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", sorted(CASES))
def test_device_box_box_contacts_match_oracle(name):
    sc = CASES[name][0]
    m, om = K.build_model(sc), oracle_lib.OracleModel(sc)
    gb = K.WorldBatch()
    gb.add_world(m)
    ob = oracle_lib.OracleBatch([om], [0], n_threads=1)
    ob.set_trace(True)
    cfg = K.config_for(sc)
    gb.step(cfg)
    ob.step(cfg)
    cg, dg = gb.dump_contacts(0)
    co, do = ob.dump_contacts(0)
    assert cg.shape == co.shape and (cg == co).all()
    if len(co):
        np.testing.assert_allclose(dg, do, rtol=0, atol=1e-12)
    pg, tg, _ = gb.get_state()
    po, to, _ = ob.get_state()
    assert np.abs(pg - po).max() < 1e-12 and np.abs(tg - to).max() < 1e-10


def test_box_pile_vs_oracle():
    """64-box pile: contact (geom_a, geom_b) order bit-exact every step, the
    first step's state to 1e-12; later steps within 1e-6 (a stacked pile is
    chaotic: a PADMM run that converges one iteration apart, as rounding
    decides, moves the impulses by ~eps)."""
    sc = box_pile(64)
    cfg = K.config_for(sc)
    m, om = K.build_model(sc), oracle_lib.OracleModel(sc)
    gb = K.WorldBatch()
    gb.add_world(m)
    ob = oracle_lib.OracleBatch([om], [0], n_threads=1)
    ob.set_trace(True)
    for k in range(5):
        gb.step(cfg)
        ob.step(cfg)
        cg, dg = gb.dump_contacts(0)
        co, do = ob.dump_contacts(0)
        assert cg.shape == co.shape and (cg == co).all()
        assert len(co) >= 4 * 64
        pg, _, _ = gb.get_state()
        po, _, _ = ob.get_state()
        assert np.abs(pg - po).max() < (1e-12 if k == 0 else 1e-6)
    assert gb.kernels() == ["cr"]


def test_box_pile_batch_equals_solo_bitwise():
    sc = box_pile(64)
    cfg = K.config_for(sc)
    m = K.build_model(sc)
    nw = 296
    b = K.WorldBatch()
    for _ in range(nw):
        b.add_world(m)
    p, t, tm = b.get_state()
    t = K.bench_jitter(t, [m.n_bodies] * nw, seed=1)
    b.set_state(p, t, tm)
    w = nw - 3
    s = K.WorldBatch()
    s.add_world(m)
    np_, nt_ = 7 * m.n_bodies, 6 * m.n_bodies
    s.set_state(p[w * np_:(w + 1) * np_], t[w * nt_:(w + 1) * nt_], tm[w:w + 1])
    b.step(cfg, 3)
    s.step(cfg, 3)
    pb, tb, _ = b.get_state()
    ps, ts, _ = s.get_state()
    assert (pb[w * np_:(w + 1) * np_] == ps).all() and (tb[w * nt_:(w + 1) * nt_] == ts).all()
    d = b.diagnostics()
    assert max(d[i].kkt_momentum_inf for i in range(nw)) < 1e-5
