"""CR-kernel phase probe (diagnostic only): run with KD_CR_REG=2 to get thread
0's clock64 split of cr_reg_kernel per world; prints cycles per CR apply."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scenes import closed_chain, sphere_pile, stewart_tower  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "closed_chain"
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 296
sc = {"closed_chain": lambda: closed_chain(22), "stewart_tower": stewart_tower}.get(which, sphere_pile)()
cfg = K.config_for(sc)
m = K.build_model(sc)
b = K.WorldBatch()
for _ in range(nw):
    b.add_world(m)
p, t, tm = b.get_state()
t = K.bench_jitter(t, [m.n_bodies] * nw, seed=1)
b.set_state(p, t, tm)
b.step(cfg, 10)
b.step(cfg, 1)
pc = b.phase_cycles().astype(np.float64)
d = b.diagnostics()
its = np.array([x.iterations for x in d], dtype=np.float64)
cri = np.array([x.cr_iterations for x in d], dtype=np.float64)
applies = cri + 2 * its
names = ["A products+bar", "B body sums+bar", "C gather", "CR reductions", "PADMM reduction", "rest", "total"]
out = {"workload": which, "worlds": nw, "padmm_iters_mean": its.mean(), "cr_iters_mean": cri.mean(),
       "rows": d[0].n_rows}
for k, nm in enumerate(names):
    out[nm + " /apply"] = float((pc[:, k] / np.maximum(applies, 1)).mean())
print(json.dumps(out))
