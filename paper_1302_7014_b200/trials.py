"""Trial sweeps sharded across ranks (BASELINE.json configs[4] "per-GPU-
sharded sweep of 10^4 independent trials over c").

The paper's protocol: many independent G^r_{n,cn} trials, report rounds and
whether the k-core is empty.  Trials are independent, so rank p of P takes the contiguous
index range [p T / P, (p+1) T / P): no data-path collective; one gather of the fixed-size
per-trial records at the end.  Trial t of the paper-shaped sweep uses
c_j = 0.700 + 0.002 j with j = t div 100, m_t = 700,000 + 2,000 j (an exact integer, never
derived from float) and seed 1000 + t.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def paper_trials(T: int = 10_000, n: int = 1_000_000, base_seed: int = 1000, per_c: int = 100):
    """(m[t], seed[t]) of the C5s sweep: 100 values of c from 0.700 in steps of 0.002."""
    t = np.arange(T, dtype=np.uint64)
    j = t // per_c
    m = (700 * n // 1000 + (2 * n // 1000) * j).astype(np.uint64)
    seeds = (base_seed + t).astype(np.uint64)
    return m, seeds


def shard(T: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous trial range of `rank`: [rank T / world, (rank+1) T / world)."""
    return rank * T // world, (rank + 1) * T // world


def run_sweep(runner, m: np.ndarray, seeds: np.ndarray, group=None, device=None):
    """Run this rank's shard with runner(m_slice, seed_slice) -> (rounds u32[], core u64[]) and
    all-gather the per-trial records.  Returns (rounds[T], core[T]) on every rank."""
    T = int(m.size)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard(T, world, rank)
    rounds, core = runner(m[lo:hi], seeds[lo:hi])
    if world == 1:
        return np.asarray(rounds, dtype=np.uint32), np.asarray(core, dtype=np.uint64)
    # fixed-size records: pad every shard to the largest shard length
    maxlen = max(shard(T, world, p)[1] - shard(T, world, p)[0] for p in range(world))
    dev = device if device is not None else torch.device("cpu")
    rec = torch.zeros((maxlen, 2), dtype=torch.int64, device=dev)
    rec[: hi - lo, 0] = torch.from_numpy(np.asarray(rounds, dtype=np.int64))
    rec[: hi - lo, 1] = torch.from_numpy(np.asarray(core, dtype=np.uint64).astype(np.int64))
    out = [torch.zeros_like(rec) for _ in range(world)]
    dist.all_gather(out, rec, group=group)
    R = np.zeros(T, dtype=np.uint32)
    C = np.zeros(T, dtype=np.uint64)
    for p in range(world):
        a, b = shard(T, world, p)
        o = out[p].cpu().numpy()
        R[a:b] = o[: b - a, 0]
        C[a:b] = o[: b - a, 1]
    return R, C


def gpu_runner(n: int, r: int, k: int, batch: int = 128, device=None):
    """runner for run_sweep backed by peel_sweep on this rank's GPU."""
    import paper_1302_7014_b200 as pk

    def run(m, seeds):
        return pk.sweep(n, r, k, m, seeds, batch=batch, device=device)

    return run
