"""bench.py's one-line JSON contract on a short run (GPU box only): the keys
the driver reads, the end-to-end figure with its copy sizes, the roofline and
CPU-baseline objects, clocks and the kernel-launch count, and the reference
arm's line on the same metric and config."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_product_line_contract():
    d = _run(["--steps", "3", "--warmup", "3", "--settle", "2", "--worlds-per-gpu", "1184"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "clocks", "gpu_launches", "e2e"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["config"]["workload"] == "dr_legs" and d["config"]["global_worlds"] == 1184
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "smem" and r["achieved"] > 0 and r["peak"] > 0 and 0 < r["frac"] < 1
    assert r["kernel"].startswith("dense_kernel")
    c = d["cpu_baseline"]
    assert c["value"] > 0 and c["kind"] == "port" and c["cores"] >= 1
    assert d["gpu_launches"] > 0
    assert d["clocks"].get("sm_max_mhz")


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "3", "--settle", "2", "--worlds-per-gpu", "64"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["metric"] == "world-steps/sec (DR Legs worlds, dense PADMM step)"
