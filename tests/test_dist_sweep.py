"""Multi-process (gloo, world_size 2, CPU) test of the sharded trial sweep's host logic:
every trial runs exactly once, on the rank its index maps to, and the gathered
per-trial records equal a single-process run.  Trials run on the oracle here."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1302_7014_b200 import trials as S


def _oracle_runner(n, r, k):
    from oracle import oracle as O

    def run(m, seeds):
        rounds, core = [], []
        for mm, sd in zip(m, seeds):
            res = O.sync_peel(O.gen_hypergraph(n, int(mm), r, int(sd)), n, k)
            rounds.append(res.rounds)
            core.append(int(res.core_mask.sum()))
        return np.array(rounds, dtype=np.uint32), np.array(core, dtype=np.uint64)

    return run


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, n, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, seeds = S.paper_trials(T, n=n, per_c=5)
    R, C = S.run_sweep(_oracle_runner(n, 3, 2), m, seeds)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.stack([R.astype(np.int64), C.astype(np.int64)]))
    dist.destroy_process_group()


def test_shard_covers_every_trial_once():
    for T in (0, 1, 7, 100, 10_000):
        for world in (1, 2, 3, 8):
            seen = np.zeros(T, dtype=int)
            for p in range(world):
                a, b = S.shard(T, world, p)
                seen[a:b] += 1
            assert np.all(seen == 1)


def test_paper_trials_exact_integers():
    m, seeds = S.paper_trials(10_000)
    assert m[0] == 700_000 and m[99] == 700_000 and m[100] == 702_000 and m[-1] == 898_000
    assert seeds[0] == 1000 and seeds[-1] == 10_999


def test_gloo_two_ranks_match_single_process(tmp_path):
    T, n = 20, 20_000
    port = _free_port()
    mp.spawn(_worker, args=(2, port, T, n, str(tmp_path)), nprocs=2, join=True)
    a = np.load(tmp_path / "r0.npy")
    b = np.load(tmp_path / "r1.npy")
    assert np.array_equal(a, b)
    m, seeds = S.paper_trials(T, n=n, per_c=5)
    R, C = S.run_sweep(_oracle_runner(n, 3, 2), m, seeds)  # world 1
    assert np.array_equal(a[0], R.astype(np.int64)) and np.array_equal(a[1], C.astype(np.int64))
    # c from 0.70 to 0.708 (below c*_{2,3} = 0.818): every core empty
    assert np.all(C == 0) and np.all(R > 0)
