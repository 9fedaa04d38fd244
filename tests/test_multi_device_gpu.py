"""One process driving several batches / devices (GPU box).

The >48 KB shared-memory opt-in of every kernel is a per-device attribute; the
library caches it per device ordinal with a compare-exchange, so batches on
different GPUs in one process, or host threads stepping their own batches at
once, all launch correctly.  Worlds are independent, so every batch must give
the bitwise result of a lone batch.
"""
import threading

import numpy as np
import pytest

import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import closed_chain, dr_legs

pytestmark = pytest.mark.gpu


def _run(model, cfg, device, steps, out, key):
    b = K.WorldBatch(device=device)
    for _ in range(64):
        b.add_world(model)
    p, t, tm = b.get_state()
    t = K.bench_jitter(t, [model.n_bodies] * 64, seed=7)
    b.set_state(p, t, tm)
    b.step(cfg, steps)
    out[key] = b.get_state()


def test_host_threads_step_own_batches_concurrently():
    sc = dr_legs()
    m, cfg = K.build_model(sc), K.config_for(sc)
    ref = {}
    _run(m, cfg, 0, 20, ref, "solo")
    out = {}
    th = [threading.Thread(target=_run, args=(m, cfg, 0, 20, out, k)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for k in range(4):
        for a, b in zip(out[k], ref["solo"]):
            assert np.array_equal(a, b)


def test_batches_on_two_devices_in_one_process():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    sc = closed_chain(12)  # the dense HBM-slab kernel needs the > 48 KB opt-in on each device
    m, cfg = K.build_model(sc), K.config_for(sc)
    out = {}
    th = [threading.Thread(target=_run, args=(m, cfg, d, 10, out, d)) for d in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)
