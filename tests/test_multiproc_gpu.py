"""The N-rank bench path end to end on a GPU box (GPU box only).

`bench.py --gpus 2` re-launches itself under torch.distributed.run; with
KD_BENCH_SHARE_GPU=1 both ranks step their dealt worlds on the box's GPU(s)
and reduce over gloo, so the launcher, the deal of the global batch, the
per-rank stepping and the end-of-run reductions all run on hardware even on a
one-GPU box (the reported rate is then not a 2-GPU throughput).
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_rank_bench_runs_end_to_end():
    env = dict(os.environ, KD_BENCH_SHARE_GPU="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup",
                          "3", "--settle", "2", "--worlds-per-gpu", "296", "--no-e2e", "--no-cpu"],
                         capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_worlds"] == 2 * 296
    assert d["run_stats"]["worlds"] == 2 * 296  # both ranks' statistics reduced
    assert d["value"] > 0 and d["run_stats"]["max_kkt"] < 1e-5
