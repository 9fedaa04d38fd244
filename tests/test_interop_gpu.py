"""Zero-copy device state for PyTorch (kd_batch_device_state)."""
import numpy as np
import pytest

import oracle_lib
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import dr_legs

pytestmark = pytest.mark.gpu


def test_device_state_views_alias_the_batch():
    import torch
    sc = dr_legs()
    m = K.build_model(sc)
    b = K.WorldBatch()
    for _ in range(4):
        b.add_world(m)
    b.step(K.config_for(sc), 2)
    p, t, tm = b.device_state()
    hp, ht, htm = b.get_state()
    assert p.dtype == torch.float64 and p.is_cuda and p.numel() == b.pose_len
    assert np.array_equal(p.cpu().numpy(), hp) and np.array_equal(t.cpu().numpy(), ht)
    assert np.array_equal(tm.cpu().numpy(), htm)
    # a write through the view is the batch's state (ordered on the batch stream)
    s = torch.cuda.ExternalStream(b.stream())
    with torch.cuda.stream(s):
        t.zero_()
    b.sync()
    assert not b.get_state()[1].any()


def test_device_state_step_sees_torch_writes():
    import torch
    sc = oracle_lib.bundled_scene("freefall")
    m = K.build_model(sc)
    b = K.WorldBatch()
    b.add_world(m)
    cfg = K.config_for(sc)
    p, t, _ = b.device_state()
    s = torch.cuda.ExternalStream(b.stream())
    with torch.cuda.stream(s):
        t[2] = 1.0  # upward linear velocity
    b.step(cfg, 1)
    vz = b.get_state()[1][2]
    assert abs(vz - (1.0 - 9.81 * cfg.dt)) < 1e-12
