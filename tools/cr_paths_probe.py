import sys, collections
sys.path.insert(0, '/root/repo')
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import sphere_pile, closed_chain
for name, sc, nw in (("sphere_pile", sphere_pile(), 296), ("closed_chain", closed_chain(22), 64)):
    cfg = K.config_for(sc); m = K.build_model(sc)
    b = K.WorldBatch()
    for _ in range(nw): b.add_world(m)
    p, t, tm = b.get_state(); t = K.bench_jitter(t, [m.n_bodies] * nw, seed=1); b.set_state(p, t, tm)
    for k in range(20):
        b.step(cfg, 1)
        if k % 5 == 4:
            d = b.diagnostics()
            print(name, k, dict(collections.Counter(b.cr_paths())), "rows", min(x.n_rows for x in d[:nw]), max(x.n_rows for x in d[:nw]))
