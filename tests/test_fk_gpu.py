"""Batched forward kinematics on the device (kd_fk.cu; fk_solve, fk.cpp) vs the
CPU oracle's restatement, which is pinned by the reference's four FK tests
(test_fk.cpp:33-153, restated in oracle/oracle_tests.cpp)."""
import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import dr_legs

pytestmark = pytest.mark.gpu


def _run(scene, joints, values_per_world):
    m, om = K.build_model(scene), oracle_lib.OracleModel(scene)
    nw = len(values_per_world)
    b = K.WorldBatch()
    for _ in range(nw):
        b.add_world(m)
    p0, _, _ = b.get_state()
    it, res, conv = b.fk(np.tile(joints, (nw, 1)), np.asarray(values_per_world))
    pg, _, _ = b.get_state()
    nb = m.n_bodies
    out = []
    for w in range(nw):
        po, ito, reso, convo = om.fk(joints, values_per_world[w], p0[7 * nb * w: 7 * nb * (w + 1)])
        out.append((pg[7 * nb * w: 7 * nb * (w + 1)], it[w], res[w], conv[w], po, ito, reso, convo))
    return out


def test_fourbar_cranks_match_oracle():
    sc = oracle_lib.bundled_scene("fourbar")
    cranks = [[np.pi / 2 + d] for d in (0.1, 0.4, -0.3, 0.9)]
    for pg, it, res, conv, po, ito, reso, convo in _run(sc, [0], cranks):
        assert conv and convo and res < 1e-8
        assert it == ito
        assert np.abs(pg - po).max() < 1e-9


def test_consistent_input_is_untouched():
    sc = oracle_lib.bundled_scene("fourbar")
    m = K.build_model(sc)
    b = K.WorldBatch()
    b.add_world(m)
    p0, _, _ = b.get_state()
    q0 = m.joint_coordinate(0, p0.reshape(-1, 7))
    it, res, conv = b.fk([0], [q0])
    assert it[0] == 0 and conv[0]
    assert np.array_equal(b.get_state()[0], p0)


def test_dr_legs_random_actuator_targets():
    """Resets of the config-2 biped: the 12 PD joints get random offsets from
    their build-time coordinates (PAPER §5.3); loops close within 1e-8."""
    sc = dr_legs()
    m = K.build_model(sc)
    p0 = np.asarray(m.initial_state().poses).reshape(-1)
    pd = [j for j, js in enumerate(sc.joints) if js.kp > 0]
    base = np.array([m.joint_coordinate(j, p0.reshape(-1, 7)) for j in pd])
    rng = np.random.default_rng(3)
    vals = [base + rng.uniform(-0.15, 0.15, size=len(pd)) for _ in range(6)]
    same = 0
    for pg, it, res, conv, po, ito, reso, convo in _run(sc, pd, vals):
        assert conv == convo
        assert conv and res < 1e-8
        assert np.abs(pg - po).max() < 1e-7
        same += it == ito
    assert same >= 5


def test_loop_that_cannot_close_is_flagged():
    from paper_2603_16536_b200.scene import parse_scene
    sc = parse_scene("""{"name": "fourbar_long_crank", "gravity": [0, -9.81, 0],
      "bodies": [
        {"name": "crank", "mass": 1.0, "inertia": [1e-4, 0.2, 0.2], "position": [0.0, 0.75, 0.0],
         "orientation": [0.7071067811865476, 0, 0, 0.7071067811865476]},
        {"name": "coupler", "mass": 1.0, "inertia": [1e-4, 0.1, 0.1],
         "position": [0.43014417303072305, 1.2450961153538151, 0.0],
         "orientation": [0.964439823436757, 0.0, 0.0, -0.26430252925251585]},
        {"name": "rocker", "mass": 1.0, "inertia": [1e-4, 0.1, 0.1],
         "position": [0.930144173030723, 0.49509611535381526, 0.0],
         "orientation": [0.6558537741224968, 0.0, 0.0, 0.7548879565665867]}],
      "joints": [
        {"name": "crank_pivot", "type": "revolute", "parent": "world", "child": "crank",
         "parent_position": [0, 0, 0], "child_position": [-0.75, 0, 0], "axis": [0, 0, 1]},
        {"name": "crank_coupler", "type": "revolute", "parent": "crank", "child": "coupler",
         "parent_position": [0.75, 0, 0], "child_position": [-0.5, 0, 0], "axis": [0, 0, 1]},
        {"name": "coupler_rocker", "type": "revolute", "parent": "coupler", "child": "rocker",
         "parent_position": [0.5, 0, 0], "child_position": [0.5, 0, 0], "axis": [0, 0, 1]},
        {"name": "rocker_ground", "type": "revolute", "parent": "world", "child": "rocker",
         "parent_position": [1, 0, 0], "child_position": [-0.5, 0, 0], "axis": [0, 0, 1]}],
      "geoms": []}""")
    (pg, it, res, conv, po, ito, reso, convo), = _run(sc, [0], [[np.pi]])
    assert not conv and not convo
    assert res > 1e-3 and reso > 1e-3


def test_fk_rejects_non_scalar_joint():
    sc = oracle_lib.bundled_scene("fourbar")
    b = K.WorldBatch()
    b.add_world(K.build_model(sc))
    with pytest.raises(Exception):
        b.fk([99], [0.0])


def test_fk_large_model_uses_hbm_scratch():
    """156 bodies (normal matrix 936 x 936, beyond one CTA's shared memory):
    the kernel works in a per-world HBM slab; fk_solve has no size cap
    (fk.cpp:65-106).  Extend the bottom Stewart legs by 5 / 10 mm."""
    from paper_2603_16536_b200.scenes import stewart_tower
    sc = stewart_tower()
    m = K.build_model(sc)
    legs = [j for j, name in enumerate(m.joint_names) if name.startswith("p0_")]
    assert len(legs) == 6
    for pg, it, res, conv, po, ito, reso, convo in _run(sc, legs, [[0.005] * 6, [0.01] * 6]):
        assert conv and convo and res < 1e-8
        assert it == ito
        assert np.abs(pg - po).max() < 1e-8
