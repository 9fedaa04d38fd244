"""Golden scene bundle and the scene parser (scene.cpp:86-241)."""
import json
import os

import pytest

import oracle_lib
from paper_2603_16536_b200.scene import (SceneError, parse_scene, parse_scene_obj, serialize_scene,
                                         config_for)

REF = "/root/reference/proj/scenes"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present (GPU box)")
def test_bundle_matches_reference_scenes():
    bundle = oracle_lib.load_bundle()
    names = sorted(f[:-5] for f in os.listdir(REF) if f.endswith(".json"))
    assert sorted(bundle) == names
    for n in names:
        with open(os.path.join(REF, n + ".json")) as f:
            assert json.load(f) == bundle[n]


def test_bundle_has_the_seven_spec_scenes():
    assert sorted(oracle_lib.load_bundle()) == ["double_fourbar", "fourbar", "freefall", "inclined_box",
                                                  "pendulum", "serial_chain_10", "sphere_on_plane"]


def test_scene_config_block():
    fb = oracle_lib.bundled_scene("fourbar")
    cfg = config_for(fb)
    assert cfg.integrator == "moreau" and cfg.dt == 1.0 / 240.0 and cfg.rho == 0.1


def test_scene_errors_carry_context():
    with pytest.raises(SceneError, match="bodies\\[0\\]: missing field 'mass'"):
        parse_scene('{"bodies":[{"name":"a","inertia":[1,1,1]}]}', "x.json")
    with pytest.raises(SceneError, match="not a unit quaternion"):
        parse_scene('{"bodies":[{"name":"a","mass":1,"inertia":[1,1,1],"orientation":[2,0,0,0]}]}')
    with pytest.raises(SceneError, match="unknown shape"):
        parse_scene('{"geoms":[{"body":"world","shape":"cone"}]}')
    with pytest.raises(SceneError):
        parse_scene("{not json")


def test_serialize_roundtrip():
    for name, obj in oracle_lib.load_bundle().items():
        s = parse_scene_obj(obj, name)
        s2 = parse_scene(serialize_scene(s), name)
        assert [b.position for b in s.bodies] == [b.position for b in s2.bodies]
        assert [j.axis for j in s.joints] == [j.axis for j in s2.joints]
        assert len(s.geoms) == len(s2.geoms)
