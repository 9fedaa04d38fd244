"""Per-world PADMM iteration distribution (diagnostic) and a greedy list-schedule
estimate of the K2 tail: natural world order vs longest-first."""
import heapq
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scenes import closed_chain, dr_legs  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "dr_legs"
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
slots = int(sys.argv[3]) if len(sys.argv) > 3 else 148
fixed = float(sys.argv[4]) if len(sys.argv) > 4 else 10.0
sc = dr_legs() if which == "dr_legs" else closed_chain(22)
cfg = K.config_for(sc)
m = K.build_model(sc)
b = K.WorldBatch()
for _ in range(nw):
    b.add_world(m)
p, t, tm = b.get_state()
t = K.bench_jitter(t, [m.n_bodies] * nw, seed=1)
b.set_state(p, t, tm)
b.step(cfg, 55)


def makespan(costs):
    h = [0.0] * slots
    for c in costs:
        s = heapq.heappop(h)
        heapq.heappush(h, s + c)
    return max(h)


rows = []
for k in range(5):
    b.step(cfg, 1)
    it = np.array([d.iterations for d in b.diagnostics()[:nw]], dtype=float)
    prev = it if k == 0 else prev_it
    cost = it + fixed
    nat = makespan(cost)
    srt = makespan(cost[np.argsort(-(prev + fixed), kind="stable")])
    ideal = cost.sum() / slots
    rows.append({"step": k, "iters_mean": it.mean(), "iters_max": it.max(), "n_200": int((it >= 200).sum()),
                 "natural_over_ideal": nat / ideal, "sorted_by_prev_over_ideal": srt / ideal,
                 "corr_prev": float(np.corrcoef(prev, it)[0, 1]) if k else 1.0})
    prev_it = it
print(json.dumps(rows))
