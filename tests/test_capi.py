"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/kamino_b200.h declares, and the host model build agrees with
the oracle (row layout, loop count, PD targets, ModelError codes/messages)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200 import _capi
from paper_2603_16536_b200.scene import ModelError, SceneBody, SceneDescription, SceneGeom, SceneJoint
from paper_2603_16536_b200.scenes import box_pile, closed_chain, dr_legs, sphere_pile

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "kamino_b200.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(kd_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = C.CDLL(K.LIB_PATH)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(header_symbols()) >= 25


def test_struct_layouts_match_compiled_abi():
    lib = C.CDLL(K.LIB_PATH)
    out = (C.c_int32 * 10)()
    assert lib.kd_abi_sizes(out, 10) == 10
    mine = [C.sizeof(t) for t in (_capi.kd_body_desc, _capi.kd_joint_desc, _capi.kd_geom_desc,
                                   _capi.kd_scene_desc, _capi.kd_step_config, _capi.kd_step_diag,
                                   _capi.kd_model_info, _capi.kd_row_dump, _capi.kd_limit_cache_entry,
                                   _capi.kd_contact_cache_entry)]
    assert list(out) == mine


def test_no_device_fails_loudly():
    pytest.importorskip("torch")
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    m = K.build_model(oracle_lib.bundled_scene("fourbar"))
    b = K.WorldBatch()
    b.add_world(m)
    with pytest.raises(K.KaminoError, match="no CPU fallback"):
        b.step(K.StepConfig())


ALL = ["fourbar", "double_fourbar", "serial_chain_10", "pendulum", "sphere_on_plane", "inclined_box", "freefall"]


@pytest.mark.parametrize("name", ALL)
def test_model_build_matches_oracle(name):
    sc = oracle_lib.bundled_scene(name)
    m, o = K.build_model(sc), oracle_lib.OracleModel(sc)
    for f, _ in m.info._fields_:
        assert getattr(m.info, f) == getattr(o.info, f), f
    for a, b in zip(m.joint_layout(), o.joint_layout()):
        assert (a == b).all()


def test_synthetic_models_match_oracle():
    for sc in (dr_legs(), closed_chain(16), sphere_pile(20), box_pile(8)):
        m, o = K.build_model(sc), oracle_lib.OracleModel(sc)
        for f, _ in m.info._fields_:
            assert getattr(m.info, f) == getattr(o.info, f), (sc.name, f)
    m = K.build_model(dr_legs())
    assert (m.info.n_bodies, m.info.n_joints, m.n_loops, m.n_bilateral_rows, m.n_dynamics_rows) == (31, 36, 6, 180, 12)


def test_joint_coordinate_matches_oracle():
    sc = oracle_lib.bundled_scene("fourbar")
    m, o = K.build_model(sc), oracle_lib.OracleModel(sc)
    rng = np.random.default_rng(3)
    for _ in range(20):
        p = np.zeros((3, 7))
        p[:, :3] = rng.normal(size=(3, 3))
        q = rng.normal(size=(3, 4))
        p[:, 3:] = q / np.linalg.norm(q, axis=1, keepdims=True)
        for j in range(4):
            assert abs(m.joint_coordinate(j, p) - o.joint_coordinate(j, p)) < 1e-14


def _minimal():
    return SceneDescription(name="m", bodies=[SceneBody("a", 1.0, [[0.1, 0, 0], [0, 0.1, 0], [0, 0, 0.1]])])


def _bad_scenes():
    out = []
    s = _minimal(); s.joints.append(SceneJoint("j", "revolute", "a", "nosuch")); out.append(s)
    s = _minimal(); s.joints.append(SceneJoint("j", "revolute", "world", "a", axis=[0, 0, 2])); out.append(s)
    s = _minimal(); s.bodies[0].inertia = [[-1, 0, 0], [0, -1, 0], [0, 0, -1]]; out.append(s)
    s = _minimal(); s.bodies[0].inertia = [[1, 0, 0], [0, 0.1, 0], [0, 0, 0.1]]; out.append(s)
    s = _minimal(); s.joints.append(SceneJoint("j", "spherical", "world", "a", limits=[-1, 1])); out.append(s)
    s = _minimal(); s.joints.append(SceneJoint("j", "revolute", "world", "a", limits=[1, -1])); out.append(s)
    s = _minimal(); s.joints.append(SceneJoint("j", "revolute", "a", "a")); out.append(s)
    s = _minimal(); s.bodies.append(s.bodies[0]); out.append(s)
    s = _minimal(); s.geoms.append(SceneGeom("a", "plane")); out.append(s)
    s = _minimal(); s.bodies.append(SceneBody("b", 1.0, [[0.1, 0, 0], [0, 0.1, 0], [0, 0, 0.1]]))
    s.geoms += [SceneGeom("a", "box", half_extents=[0.1] * 3), SceneGeom("b", "sphere", radius=0.1)]; out.append(s)
    s = _minimal(); s.joints.append(SceneJoint("j", "hinge", "world", "a")); out.append(s)
    s = _minimal(); s.geoms.append(SceneGeom("a", "sphere", radius=-1)); out.append(s)
    s = _minimal(); s.joints.append(SceneJoint("j", "spherical", "world", "a", kp=1.0)); out.append(s)
    return out


@pytest.mark.parametrize("k", range(13))
def test_model_errors_match_oracle(k):
    sc = _bad_scenes()[k]
    with pytest.raises(ModelError) as e1:
        K.build_model(sc)
    with pytest.raises(ModelError) as e2:
        oracle_lib.OracleModel(sc)
    assert e1.value.code == e2.value.code
    assert str(e1.value) == str(e2.value)
