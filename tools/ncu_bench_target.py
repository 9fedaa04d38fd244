"""ncu target at the bench's timed configuration: WORKLOAD (default dr_legs)
worlds as bench.py builds them (reference jitter), `settle` untimed steps,
then 2 steps.  Run with KD_SPLIT=1 KD_GRAPHS=0 so every kernel of a step is
one direct launch over the whole batch (launch counting for -s is then
steps x kernels).  usage: ncu_bench_target.py [workload] [worlds] [settle]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2603_16536_b200 as K  # noqa: E402

wl_name = sys.argv[1] if len(sys.argv) > 1 else "dr_legs"
wl = bench.workloads()[wl_name]
W = int(sys.argv[2]) if len(sys.argv) > 2 else wl[2]
settle = int(sys.argv[3]) if len(sys.argv) > 3 else 50
scenes = [f() for f in wl[0]]
cfg = K.config_for(scenes[0])
keys, mine = bench.global_plan((wl[0], wl[1], W, wl[3]), W, 1, 0)
b, _ = bench.build_world_batch(K, scenes, keys, mine, 1, 0)
for _ in range(settle):
    b.step(cfg, 1)
b.step(cfg, 2)
print("done", wl_name, W, settle)
