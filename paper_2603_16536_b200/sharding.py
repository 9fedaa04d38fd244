"""World sharding across GPUs (one process per GPU) — SURVEY.md §8e.

Worlds are independent, so the data path has no collective.  The global world
list is built in the reference order (main.cpp:199-211: one jitter stream,
world-major over the whole batch), so every world's initial state is
independent of the GPU count.  `deal` bins the global worlds by a key (the
model, i.e. the device capacity class) and deals every bin round-robin over
the ranks, so each GPU gets the same mix of world sizes (for the
heterogeneous config, a contiguous block would depend on where the block
boundary falls in the w % 3 cycle; a plain w % ranks deal would give rank r
only model r % 3 when the rank count is a multiple of 3).  The only
collective is the end-of-run reduction of a few statistics (`reduce_stats`).
"""
from __future__ import annotations

import numpy as np


def world_range(n_per_rank: int, rank: int) -> range:
    """Weak scaling: every rank owns `n_per_rank` consecutive global worlds."""
    return range(rank * n_per_rank, (rank + 1) * n_per_rank)


def split_range(n_global: int, rank: int, world_size: int) -> range:
    """Strong scaling: `n_global` worlds split into near-equal contiguous blocks."""
    base, extra = divmod(n_global, world_size)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def deal(keys, world_size: int, rank: int) -> list:
    """Global world ids of `rank`: worlds grouped by keys[w] (bins in order of
    first appearance), each bin dealt round-robin over the ranks.  Every rank
    gets floor or ceil of |bin| / world_size worlds of every bin; the ids are
    returned ascending (the rank's batch keeps the global order)."""
    bins = {}
    for w, k in enumerate(keys):
        bins.setdefault(k, []).append(w)
    mine = []
    for ids in bins.values():
        mine.extend(ids[rank::world_size])
    return sorted(mine)


def jitter_worlds(world_twists, worlds, seed: int = 1, sigma: float = 1e-3, jitter=None):
    """Twists of the global worlds `worlds` (any ascending id list) after the
    reference bench jitter (main.cpp:199-211): the stream runs world-major over
    global worlds [0, max id] and each listed world keeps its own block.
    `world_twists(w)` gives global world w's initial twists; `jitter` is the
    stream implementation (default: the product library's kd_bench_jitter)."""
    if jitter is None:
        from .loopdyn import bench_jitter as jitter
    worlds = list(worlds)
    if not worlds:
        return np.zeros(0)
    top = max(worlds) + 1
    per = [np.asarray(world_twists(w), dtype=np.float64).reshape(-1) for w in range(top)]
    nb = [p.size // 6 for p in per]
    full = jitter(np.concatenate(per), nb, seed=seed, sigma=sigma)
    off = np.concatenate([[0], np.cumsum([6 * n for n in nb])])
    return np.concatenate([full[off[w]: off[w + 1]] for w in worlds])


def jitter_slice(initial_twists: np.ndarray, n_bodies: int, worlds: range, seed: int = 1, sigma: float = 1e-3):
    """Twist storage of global worlds `worlds` after the reference bench jitter:
    the stream is drawn for worlds [0, worlds.stop) and this block is kept."""
    from .loopdyn import bench_jitter
    per = np.asarray(initial_twists, dtype=np.float64).reshape(-1)
    assert per.size == 6 * n_bodies
    full = np.tile(per, worlds.stop)
    full = bench_jitter(full, [n_bodies] * worlds.stop, seed=seed, sigma=sigma)
    return full[6 * n_bodies * worlds.start:].copy()


def jitter_slice_mixed(world_twists, worlds: range, seed: int = 1, sigma: float = 1e-3):
    """Heterogeneous batches: `world_twists(w)` gives global world w's initial
    twists (6 per body); the stream runs over worlds [0, worlds.stop) in world
    order (main.cpp:199-211) and the block `worlds` is kept."""
    from .loopdyn import bench_jitter
    per = [np.asarray(world_twists(w), dtype=np.float64).reshape(-1) for w in range(worlds.stop)]
    nb = [p.size // 6 for p in per]
    full = bench_jitter(np.concatenate(per), nb, seed=seed, sigma=sigma)
    off = 6 * sum(nb[:worlds.start])
    return full[off:].copy()


def local_stats(diags, n_worlds: int) -> dict:
    """Per-step statistics of one rank's worlds (kd_step_diag array)."""
    its = [diags[w].iterations for w in range(n_worlds)]
    return {"worlds": float(n_worlds), "iterations": float(sum(its)),
            "converged": float(sum(diags[w].converged for w in range(n_worlds))),
            "max_kkt": max((diags[w].kkt_momentum_inf for w in range(n_worlds)), default=0.0),
            "max_r": max((max(diags[w].r_p, diags[w].r_d, diags[w].r_c) for w in range(n_worlds)), default=0.0)}


def reduce_stats(dist, stats: dict, device="cpu") -> dict:
    """One all-reduce of the run statistics (sums for counts, max for residuals)."""
    import torch
    sums = torch.tensor([stats["worlds"], stats["iterations"], stats["converged"]], dtype=torch.float64,
                        device=device)
    maxs = torch.tensor([stats["max_kkt"], stats["max_r"]], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized():
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        dist.all_reduce(maxs, op=dist.ReduceOp.MAX)
    s, m = sums.tolist(), maxs.tolist()
    return {"worlds": s[0], "iterations": s[1], "converged": s[2], "max_kkt": m[0], "max_r": m[1],
            "mean_iterations": s[1] / max(1.0, s[0])}
