"""Per-family device time of one step at the bench's configuration (CUDA
events on the solver streams, kd_batch_get_timing): K1 assemble, dense family
(K2f + K2), matrix-free, K3 recover, and the step's wall time on the device.
usage: family_probe.py [workload] [worlds]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_16536_b200 as K  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "dr_legs"
wl = bench.workloads()[name]
W = int(sys.argv[2]) if len(sys.argv) > 2 else wl[2]
scenes = [f() for f in wl[0]]
cfg = K.config_for(scenes[0])
keys, mine = bench.global_plan((wl[0], wl[1], W, wl[3]), W, 1, 0)
b, _ = bench.build_world_batch(K, scenes, keys, mine, 1, 0)
b.step(cfg, 55)
b.get_state()
b.enable_timing(True)
t0 = time.perf_counter()
b.step(cfg, 20)
b.get_state()
wall = (time.perf_counter() - t0) / 20 * 1e3
tim = b.timing()
print(json.dumps({"workload": name, "worlds": W, "wall_ms_per_step": wall,
                  **{k: v / 20 for k, v in tim.items() if k.endswith("_ms")}}))
