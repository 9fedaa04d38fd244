"""Box-pile probe (diagnostic): device vs oracle contacts and states over a few
steps, kernel/CR-path mix and row counts."""
import collections
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle_lib  # noqa: E402
import paper_2603_16536_b200 as K  # noqa: E402
from paper_2603_16536_b200.scenes import box_pile  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
sc = box_pile(n)
cfg = K.config_for(sc)
m, om = K.build_model(sc), oracle_lib.OracleModel(sc)
gb = K.WorldBatch()
gb.add_world(m)
ob = oracle_lib.OracleBatch([om], [0], n_threads=1)
ob.set_trace(True)
for k in range(steps):
    gb.step(cfg)
    ob.step(cfg)
    cg, dg_ = gb.dump_contacts(0)
    co, do_ = ob.dump_contacts(0)
    dg, do = gb.diagnostics()[0], ob.diagnostics()[0]
    pg, _, _ = gb.get_state()
    po, _, _ = ob.get_state()
    same = cg.shape == co.shape and (cg == co).all()
    print(k, "rows", dg.n_rows, do.n_rows, "contacts", len(cg), len(co), "same_idx", same,
          "it", dg.iterations, do.iterations, "pose_err %.2e" % float(np.abs(pg - po).max()),
          "path", collections.Counter(gb.cr_paths()), gb.kernels()[0], flush=True)
