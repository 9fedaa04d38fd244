import sys, os, time, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2603_16536_b200 as K
from paper_2603_16536_b200.scenes import dr_legs
sc = dr_legs(); cfg = K.config_for(sc); m = K.build_model(sc)
def mk(nw):
    b = K.WorldBatch(device=0)
    for _ in range(nw): b.add_world(m)
    p, t, tm = b.get_state(); t = K.bench_jitter(t, [m.n_bodies]*nw, seed=1); b.set_state(p, t, tm)
    b.step(cfg, 50); return b
def timeit(fn, steps=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps * 1e3
full = mk(4096)
print("full step_async ms", timeit(lambda: (full.step_async(cfg, 1), full.sync())))
print("full step(cfg,10)/10 ms", timeit(lambda: full.step(cfg, 10), 3) / 10)
hs = [mk(2048), mk(2048)]
def both():
    for h in hs: h.step_async(cfg, 1)
    for h in hs: h.sync()
print("two halves concurrent ms", timeit(both))
def serial():
    for h in hs: h.step_async(cfg, 1); h.sync()
print("two halves serial ms", timeit(serial))
q = [mk(1024) for _ in range(4)]
def four():
    for h in q: h.step_async(cfg, 1)
    for h in q: h.sync()
print("four quarters concurrent ms", timeit(four))
# copies
def pinned(n):
    return torch.empty(n, dtype=torch.float64).pin_memory().numpy()
bufs = []
for h in hs:
    ph, th = pinned(h.pose_len), pinned(h.twist_len)
    h.get_state_async(ph, th); h.sync(); bufs.append((ph, th))
def copies_only():
    for h, (ph, th) in zip(hs, bufs): h.set_state_async(ph, th); h.get_state_async(ph, th)
    for h in hs: h.sync()
print("copies only (both halves, H2D+D2H) ms", timeit(copies_only))
def e2e():
    for h, (ph, th) in zip(hs, bufs):
        h.set_state_async(ph, th); h.step_async(cfg, 1); h.get_state_async(ph, th)
    for h in hs: h.sync()
print("e2e halves (sync every step) ms", timeit(e2e))
def e2e_nosync():
    for h, (ph, th) in zip(hs, bufs):
        h.set_state_async(ph, th); h.step_async(cfg, 1); h.get_state_async(ph, th)
t0 = time.perf_counter()
for _ in range(20): e2e_nosync()
for h in hs: h.sync()
print("e2e halves (no sync) ms", (time.perf_counter() - t0) / 20 * 1e3)
print("pose+twist MB per step", 8 * sum(h.pose_len + h.twist_len for h in hs) / 1e6)
def h2d_only():
    for h, (ph, th) in zip(hs, bufs):
        h.set_state_async(ph, th); h.step_async(cfg, 1)
    for h in hs: h.sync()
print("halves H2D+step ms", timeit(h2d_only))
def d2h_only():
    for h, (ph, th) in zip(hs, bufs):
        h.step_async(cfg, 1); h.get_state_async(ph, th)
    for h in hs: h.sync()
print("halves step+D2H ms", timeit(d2h_only))
def d2h_only1():
    for h, (ph, th) in zip(hs, bufs):
        h.step_async(cfg, 1); h.get_state_async(ph, None)
    for h in hs: h.sync()
print("halves step+D2H poses only ms", timeit(d2h_only1))
print("two halves concurrent again ms", timeit(both))
