"""The device-backed simulate/bench harness (paper_2603_16536_b200/cli.py) and
its JSONL wire format (the reference CLI's tools/main.cpp:90-244)."""
import io
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle_lib
from paper_2603_16536_b200 import cli
from paper_2603_16536_b200 import loopdyn as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _scene_file(tmp_path, name):
    path = tmp_path / f"{name}.json"
    path.write_text(json.dumps(oracle_lib.load_bundle()[name]))
    return str(path)


def test_help_lists_both_subcommands():
    out = subprocess.run([sys.executable, "-m", "paper_2603_16536_b200.cli", "--help"], capture_output=True,
                         text=True, cwd=ROOT).stdout
    assert "simulate" in out and "bench" in out


def test_solver_flags_override_scene_config(tmp_path):
    """make_config (main.cpp:68-85): the scene's config block, then flags."""
    path = _scene_file(tmp_path, "fourbar")
    a = argparse_ns(["simulate", path, "--rho", "0.5", "--max-iters", "17", "--fixed-iters", "--backend", "sparse"])
    cfg = cli.make_config(cli.load_scene_file(path), a)
    assert cfg.integrator == "moreau"          # fourbar.json config block
    assert (cfg.rho, cfg.max_iters, cfg.fixed_iteration_mode, cfg.backend) == (0.5, 17, True, "sparse")


def argparse_ns(argv):
    import argparse
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd")
    s = sub.add_parser("simulate")
    s.add_argument("scene")
    cli.add_solver_flags(s)
    return ap.parse_args(argv)


def test_memory_estimate_formula():
    """main.cpp:219-231 for the four-bar: 21 rows (20 bilateral + 1 PD), dense."""
    m = L.build_model(oracle_lib.bundled_scene("fourbar"))
    est = cli.per_world_mem_estimate(m, cli.StepConfig())
    assert est == 8.0 * (13.0 * 3 + 24.0 * 21 + 21 * 21 + 10.0 * 21)


def test_records_are_compact_sorted_json():
    s = cli.dumps({"type": "bench", "b": [1.0, 2], "a": True})
    assert s == '{"a":true,"b":[1.0,2],"type":"bench"}'


@pytest.mark.gpu
def test_simulate_fourbar_matches_oracle(tmp_path):
    path = _scene_file(tmp_path, "fourbar")
    buf = io.StringIO()
    import argparse
    ns = argparse.Namespace(scene=path, duration=0.25, output="", emit_every=12, seed=0, dt=None, integrator=None,
                            backend=None, beta=None, rho=None, eta=None, eps=None, max_iters=None, cr_iters=None,
                            fixed_iters=False)
    assert cli.run_simulate(ns, buf) == 0
    recs = [json.loads(x) for x in buf.getvalue().splitlines()]
    steps = [r for r in recs if r["type"] == "step"]
    summary = recs[-1]
    assert summary["type"] == "summary" and summary["steps"] == 60 and len(steps) == 5
    assert set(steps[0]) == {"type", "time", "bodies", "joints", "f_inf", "contacts", "solver"}
    assert set(steps[0]["solver"]) == {"iterations", "r_p", "r_d", "r_c", "restarts", "converged", "cr_iterations"}
    sc = oracle_lib.bundled_scene("fourbar")
    om = oracle_lib.OracleModel(sc)
    ob = oracle_lib.OracleBatch([om], [0], n_threads=1)
    cfg = cli.make_config(sc, ns)
    for k, r in enumerate(steps):
        ob.step(cfg, 12)
        p, _, tm = ob.get_state()
        got = np.array([b["position"] + b["orientation"] for b in r["bodies"]]).reshape(-1)
        assert np.abs(got - p).max() < 1e-9
        assert abs(r["time"] - tm[0]) < 1e-12
        assert r["solver"]["iterations"] == ob.diagnostics()[0].iterations


@pytest.mark.gpu
def test_bench_rows(tmp_path):
    path = _scene_file(tmp_path, "double_fourbar")
    import argparse
    ns = argparse.Namespace(scenes=[path], worlds=[1, 64], steps=5, threads=0, seed=1, dt=None, integrator=None,
                            backend=None, beta=None, rho=None, eta=None, eps=None, max_iters=None, cr_iters=None,
                            fixed_iters=False)
    buf = io.StringIO()
    assert cli.run_bench(ns, buf) == 0
    rows = [json.loads(x) for x in buf.getvalue().splitlines()]
    assert [r["worlds"] for r in rows] == [1, 64]
    assert all(r["type"] == "bench" and r["throughput_steps_per_s"] > 0 for r in rows)
