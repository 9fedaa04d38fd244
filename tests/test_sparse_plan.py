"""Supernodal sparse-LLT plans (paper_2603_16536_b200/csrc/kd_snplan.cpp), host only.

The device factors the reference's Dense-backend system D = L L^T
(DenseDelassus, delassus.cpp:59-65) with a per-model plan: a fill-reducing
order of the static row-capacity pattern plus level-scheduled factor/solve
programs.  These tests run the plan's programs through the host interpreter
on random SPD systems with the plan's pattern and random inactive slots, and
compare with a dense Cholesky solve of the active subsystem."""
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import closed_chain, dr_legs, sphere_pile

SCENES = ["fourbar", "double_fourbar", "serial_chain_10", "pendulum", "sphere_on_plane", "inclined_box"]


def _scene(name):
    if name == "dr_legs":
        return dr_legs()
    if name == "closed_chain":
        return closed_chain()
    return oracle_lib.bundled_scene(name)


@pytest.mark.parametrize("name", SCENES + ["dr_legs", "closed_chain"])
def test_plan_solves_random_spd_systems(name):
    m = K.build_model(_scene(name))
    info = m.sparse_plan_info()
    assert info is not None
    for seed in range(1, 6):
        assert m.sparse_plan_selftest(seed) < 1e-11


def test_dr_legs_plan_is_sparse():
    """DR-Legs (config 2): 192 static rows + 12 limit slots + 6 pad-ground
    contact triples = 222 planned slots; the pad-pad sphere pairs are left
    out of the plan (a world that activates one takes the dense kernel)."""
    info = K.build_model(dr_legs()).sparse_plan_info()
    assert info["slots"] == 222
    assert info["nnz_L"] < 0.2 * 222 * 223 / 2          # vs the dense factor
    assert info["factor_fma"] < 0.03 * info["dense_factor_fma"]
    assert info["solve_levels"] <= 20
    assert info["smem_doubles_per_world"] * 8 < 56 * 1024  # three worlds + the solve program per CTA


def test_fourbar_plan_counts():
    info = K.build_model(oracle_lib.bundled_scene("fourbar")).sparse_plan_info()
    assert info["slots"] == 21                             # 20 bilateral + 1 PD row (test_constraints.cpp:98-110)


def test_large_pile_has_no_plan():
    assert K.build_model(sphere_pile(100)).sparse_plan_info() is None
