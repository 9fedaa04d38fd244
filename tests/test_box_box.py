"""Box-box narrow phase (opt-in extension KD_EXT_BOX_BOX).

The reference rejects box-box pairs (model.cpp:56-62), so there is no reference
behaviour to pin: the oracle's restatement (oracle.cpp box_box) is checked here
against hand-derived contact sets, and the device narrow phase against the
oracle (tests/test_box_gpu.py).  Parity for this path is therefore unpinned."""
import json
import math

import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scene import parse_scene

C8, S8 = math.cos(math.pi / 8), math.sin(math.pi / 8)
R2 = math.sqrt(0.5)


def two_boxes(pos_a, quat_a=(1, 0, 0, 0), quat_b=(1, 0, 0, 0), ext=True):
    root = {"name": "bb", "gravity": [0, 0, 0],
            "bodies": [{"name": "B", "mass": 1, "inertia": [0.1, 0.1, 0.1], "position": [0, 0, 0],
                        "orientation": list(quat_b)},
                       {"name": "A", "mass": 1, "inertia": [0.1, 0.1, 0.1], "position": list(pos_a),
                        "orientation": list(quat_a)}],
            "joints": [],
            "geoms": [{"body": "B", "shape": "box", "half_extents": [0.5, 0.5, 0.5], "mu": 0.5},
                      {"body": "A", "shape": "box", "half_extents": [0.5, 0.5, 0.5], "mu": 0.5}]}
    if ext:
        root["extensions"] = ["box_box"]
    return parse_scene(json.dumps(root))


# name -> (scene, expected contact rows [x, y, z, nx, ny, nz, depth, mu, e]); geom 0 is
# the lower box B, so the normal (b -> a) points down, -z
CASES = {
    "face": (two_boxes((0.1, 0.05, 0.95)),
             [[-0.4, 0.5, 0.475], [-0.4, -0.45, 0.475], [0.5, -0.45, 0.475], [0.5, 0.5, 0.475]]),
    "rotated_face": (two_boxes((0.0, 0.0, 0.95), (C8, 0, 0, S8)), None),  # see the octagon test
    "edge_edge": (two_boxes((0, 0, 2 * R2 - 0.02), (C8, S8, 0, 0), (C8, 0, S8, 0)), [[0.0, 0.0, R2 - 0.01]]),
    "edge_face": (two_boxes((0.1, 0, 0.5 + R2 - 0.02), (C8, S8, 0, 0)), [[-0.4, 0.0, 0.49], [0.5, 0.0, 0.49]]),
    "separated": (two_boxes((0, 0, 1.05)), []),
}


def oracle_contacts(sc):
    om = oracle_lib.OracleModel(sc)
    ob = oracle_lib.OracleBatch([om], [0], n_threads=1)
    ob.set_trace(True)
    ob.step(K.config_for(sc))
    return ob.dump_contacts(0)


def test_box_box_rejected_without_the_extension():
    with pytest.raises(oracle_lib.ModelError):
        oracle_lib.OracleModel(two_boxes((0, 0, 0.9), ext=False))
    with pytest.raises(Exception):
        K.build_model(two_boxes((0, 0, 0.9), ext=False))


def test_unknown_extension_is_rejected():
    with pytest.raises(ValueError):
        parse_scene(json.dumps({"name": "x", "bodies": [], "joints": [], "geoms": [], "extensions": ["nope"]}))


@pytest.mark.parametrize("name", ["face", "edge_edge", "edge_face", "separated"])
def test_oracle_box_box_contact_sets(name):
    sc, expect = CASES[name]
    g, d = oracle_contacts(sc)
    assert len(g) == len(expect)
    if not expect:
        return
    assert (g == [[0, 1]] * len(expect)).all()
    np.testing.assert_allclose(d[:, 0:3], np.array(expect), atol=1e-12)
    np.testing.assert_allclose(d[:, 3:6], [[0, 0, -1]] * len(expect), atol=1e-12)
    depth = {"face": 0.05, "edge_edge": 0.02, "edge_face": 0.02}[name]
    np.testing.assert_allclose(d[:, 6], depth, atol=1e-12)
    np.testing.assert_allclose(d[:, 7], 0.5, atol=1e-15)


def test_oracle_octagon_keeps_four_spread_points():
    """A box yawed 45 degrees on another: the clipped overlap is an octagon of
    equal-depth points; the kept four are pairwise far apart (every quadrant
    of the support polygon), not four neighbours."""
    g, d = oracle_contacts(CASES["rotated_face"][0])
    assert len(g) == 4
    np.testing.assert_allclose(d[:, 6], 0.05, atol=1e-12)
    xy = d[:, 0:2]
    assert abs(xy.mean(axis=0)).max() < 1e-12  # symmetric about the centre
    dmin = min(np.linalg.norm(xy[i] - xy[j]) for i in range(4) for j in range(i + 1, 4))
    assert dmin > 0.75
