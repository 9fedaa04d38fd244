import sys, collections
sys.path.insert(0, '/root/repo')
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import box_pile
sc = box_pile(64); cfg = K.config_for(sc); m = K.build_model(sc)
b = K.WorldBatch()
for _ in range(296): b.add_world(m)
p, t, tm = b.get_state(); t = K.bench_jitter(t, [m.n_bodies] * 296, seed=1); b.set_state(p, t, tm)
b.step(cfg, 12)
print(dict(collections.Counter(b.cr_paths())))
