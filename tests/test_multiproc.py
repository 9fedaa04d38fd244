"""Multi-GPU host logic on CPU (gloo, world_size 2): world sharding, the global
jitter stream sliced per rank, and the end-of-run statistics reduction."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_16536_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    nb, per = 31, 5
    init = np.zeros(6 * nb)
    worlds = sharding.world_range(per, rank)
    twists = sharding.jitter_slice(init, nb, worlds, seed=1)
    gathered = [None] * ws
    dist.all_gather_object(gathered, twists.tolist())

    class D:
        def __init__(self, it, kkt):
            self.iterations, self.converged, self.kkt_momentum_inf = it, 1, kkt
            self.r_p = self.r_d = self.r_c = 1e-7 * (rank + 1)

    diags = [D(10 * (rank + 1) + w, 1e-9 * (rank + 1)) for w in range(per)]
    st = sharding.reduce_stats(dist, sharding.local_stats(diags, per))
    if rank == 0:
        out.put((gathered, st))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_jitter_and_stats_two_ranks():
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    gathered, st = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the concatenated rank slices equal the single-process global stream
    full = sharding.jitter_slice(np.zeros(6 * 31), 31, range(0, 10), seed=1)
    assert np.array_equal(np.concatenate([np.asarray(g) for g in gathered]), full)
    assert st["worlds"] == 10
    assert st["iterations"] == sum(10 + w for w in range(5)) + sum(20 + w for w in range(5))
    assert abs(st["max_kkt"] - 2e-9) < 1e-20
    assert abs(st["max_r"] - 2e-7) < 1e-20


def test_split_range_partitions():
    for n in (1, 7, 4096, 4097):
        for ws in (1, 2, 3, 8):
            rs = [sharding.split_range(n, r, ws) for r in range(ws)]
            assert rs[0].start == 0 and rs[-1].stop == n
            assert all(a.stop == b.start for a, b in zip(rs, rs[1:]))
            assert max(len(r) for r in rs) - min(len(r) for r in rs) <= 1


def test_bench_launcher_two_gloo_ranks():
    """The real multi-GPU launcher of bench.py (`--gpus 2` outside torchrun ->
    torch.distributed.run, 2 ranks; gloo on this CPU host) in --plan-only mode:
    the global heterogeneous batch is dealt by model, every world appears on
    exactly one rank, each rank's jittered initial twists equal the slices of
    the single-process global stream, and the statistics reduce over ranks."""
    import json
    import subprocess
    import sys

    import oracle_lib
    from paper_2603_16536_b200.scenes import dr_legs

    root = oracle_lib.ROOT
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--plan-only",
                        "--worlds-per-gpu", "7", "--workload", "hetero"], capture_output=True, text=True,
                       timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    out = json.loads(line)
    assert out["n_gpus"] == 2 and len(out["ranks"]) == 2
    worlds = [w for rk in out["ranks"] for w in rk["worlds"]]
    assert sorted(worlds) == list(range(14))  # W x ranks global worlds, each on one rank
    for rk in out["ranks"]:  # the deal keeps the w % 3 mix balanced (counts differ by at most 1 per model)
        assert all(abs(c - 14 / 3 / 2) <= 1 for c in rk["models"])
    # per-rank twists == the single-process global stream's slices
    scenes = [oracle_lib.bundled_scene("fourbar"), dr_legs(), oracle_lib.bundled_scene("serial_chain_10")]
    init = [oracle_lib.OracleBatch([oracle_lib.OracleModel(s)], [0], n_threads=1).get_state()[1].copy()
            for s in scenes]
    keys = [w % 3 for w in range(14)]
    full = oracle_lib.bench_jitter(np.concatenate([init[k] for k in keys]), [init[k].size // 6 for k in keys], seed=1)
    off = np.concatenate([[0], np.cumsum([init[k].size for k in keys])])
    for rk in out["ranks"]:
        mine = np.concatenate([full[off[w]: off[w + 1]] for w in rk["worlds"]])
        assert rk["twist_len"] == mine.size
        assert abs(rk["twist_sum"] - float(mine.sum())) < 1e-12
    st = out["run_stats"]
    assert st["worlds"] == 14 and st["iterations"] == sum(w % 7 for w in range(14))
    assert st["converged"] == sum(1 for w in range(14) if w % 2 == 0)
    assert abs(st["max_kkt"] - 4e-9) < 1e-20


def test_deal_balances_every_bin():
    keys = [w % 3 for w in range(3 * 4096)]
    for ws in (1, 2, 3, 4, 6, 8):
        ranks = [sharding.deal(keys, ws, r) for r in range(ws)]
        assert sorted(w for rk in ranks for w in rk) == list(range(len(keys)))
        for rk in ranks:
            counts = [sum(1 for w in rk if keys[w] == k) for k in range(3)]
            assert max(counts) - min(counts) <= 1
