"""Multi-rank execution of the partitioned calls: world sizes 2 and 3, one
process per rank, all on one GPU, over the host transport (peel_comm_init_host driven by
torch.distributed gloo).  This runs the real per-rank protocol -- the count allgather, the
per-peer payload exchange, the allreduce and the error word -- that the NCCL communicator
runs on several GPUs; results are compared bit-exactly with the oracle.  Error protocol:
one rank rejecting its arguments, and one rank failing mid-round (PEEL_FAULT), must make
every rank leave the call (no rank blocked in a collective)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth
from oracle import oracle as O
from peeltest_util import cells_to_dev_layout, forge_foreign_cells, honest_cells

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
PEEL_OK, PEEL_ENOMEM, PEEL_ECUDA, PEEL_EPEER = 0, 2, 3, 7


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_ranks(tmp_path, world, case, env_extra=None, timeout=600, **kw):
    port = free_port()
    procs, outs = [], []
    for rank in range(world):
        out = str(tmp_path / f"{case}_{world}_{rank}.npz")
        cmd = [sys.executable, os.path.join(HERE, "multirank_worker.py"), "--rank", str(rank), "--world",
               str(world), "--port", str(port), "--case", case, "--out", out]
        for k, v in kw.items():
            cmd += [f"--{k}", str(v)]
        env = dict(os.environ)
        env.update(env_extra or {})
        procs.append(subprocess.Popen(cmd, env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
        outs.append(out)
    logs = []
    try:
        for p in procs:
            o, _ = p.communicate(timeout=timeout)
            logs.append(o.decode(errors="replace"))
    except subprocess.TimeoutExpired:
        for p in procs:
            p.kill()
        pytest.fail(f"{case} world {world}: a rank did not finish (blocked in a collective?)")
    for p, lg in zip(procs, logs):
        assert p.returncode == 0, lg[-3000:]
    return [dict(np.load(o)) for o in outs]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("n,m,r", [(200003, 150000, 3), (100001, 80000, 4), (99991, 42000, 2)])
def test_kcore_dist_ranks(tmp_path, world, n, m, r):
    seed = 7 + world
    res = run_ranks(tmp_path, world, "kcore", n=n, m=m, r=r, seed=seed)
    ref = O.sync_peel(O.gen_hypergraph(n, m, r, seed), n, 2)
    mask = np.concatenate([x["mask"] for x in res])
    for x in res:
        assert int(x["status"]) == PEEL_OK
        assert int(x["rounds"]) == ref.rounds
        assert x["survivors"].tolist() == ref.survivors.tolist() and x["killed"].tolist() == ref.killed.tolist()
    assert np.array_equal(mask, ref.core_mask)


@pytest.mark.parametrize("world", [2, 3])
def test_kcore_dist_ranks_binned_shards(tmp_path, world):
    # shards of > 2^23 vertices take the binned build and binned rounds on every rank
    n, m, r, seed = (1 << 24) + 3 * 12345 + world, int(0.75 * ((1 << 24) + 3 * 12345)), 3, 5
    res = run_ranks(tmp_path, world, "kcore", n=n, m=m, r=r, seed=seed, timeout=900)
    ref = O.sync_peel(O.gen_hypergraph(n, m, r, seed), n, 2)
    mask = np.concatenate([x["mask"] for x in res])
    for x in res:
        assert int(x["rounds"]) == ref.rounds
        assert x["survivors"].tolist() == ref.survivors.tolist() and x["killed"].tolist() == ref.killed.tolist()
    assert np.array_equal(mask, ref.core_mask)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("blog", [0, 10])
def test_iblt_dist_ranks(tmp_path, world, blog):
    C, N, r, seed = 3 * 65536, 140000, 3, 3 + world
    res = run_ranks(tmp_path, world, "iblt", n=C, m=N, r=r, seed=seed, blog=blog)
    keys = O.gen_keys(N, seed)
    o = O.Iblt(C, r, seed, blog=blog)
    o.insert(keys)
    ref = o.peel()
    got = np.sort(np.concatenate([x["keys"] for x in res]))
    assert np.array_equal(got, np.sort(ref.keys))
    for x in res:
        assert int(x["status"]) == PEEL_OK and int(x["rounds"]) == ref.rounds
        assert x["per_round"].tolist() == ref.per_round.tolist() and bool(x["complete"]) == ref.complete


@pytest.mark.parametrize("world", [2, 3])
def test_iblt_dist_ranks_forged_cells(tmp_path, world):
    C, r, seed = 3 * 8192, 3, 61
    keys = synth.random_keys(16000, 5)
    cells = honest_cells(O, keys, C, r, seed, "plain")
    forge_foreign_cells(O, cells, C, r, seed, "plain", 50, 23)
    path = str(tmp_path / "cells.npy")
    np.save(path, cells_to_dev_layout(cells))
    res = run_ranks(tmp_path, world, "iblt_cells", n=C, r=r, seed=seed, cells=path)
    o = O.Iblt(C, r, seed)
    o.load_cells(*cells)
    ref = o.peel()
    got = np.sort(np.concatenate([x["keys"] for x in res]))
    assert np.array_equal(got, np.sort(ref.keys)) and np.array_equal(got, np.sort(keys))
    for x in res:
        assert int(x["rounds"]) == ref.rounds and x["per_round"].tolist() == ref.per_round.tolist()
        assert not bool(x["complete"]) and not ref.complete


@pytest.mark.parametrize("world", [2, 3])
def test_error_bad_workspace_on_one_rank(tmp_path, world):
    res = run_ranks(tmp_path, world, "kcore", n=50000, m=35000, r=3, seed=2, shrink_ws_rank=1, timeout=300)
    st = [int(x["status"]) for x in res]
    assert st[1] == PEEL_ENOMEM and all(s == PEEL_EPEER for i, s in enumerate(st) if i != 1)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", ["kcore", "iblt"])
def test_error_mid_round_fault(tmp_path, world, case):
    # rank world-1 fails in round 3: every rank leaves at the next exchange
    kw = dict(n=200003, m=150000, r=3, seed=4) if case == "kcore" else dict(n=3 * 65536, m=140000, r=3, seed=4)
    res = run_ranks(tmp_path, world, case, env_extra={"PEEL_FAULT": f"{world - 1}:3"}, timeout=300, **kw)
    st = [int(x["status"]) for x in res]
    assert st[world - 1] == PEEL_ECUDA and all(s == PEEL_EPEER for s in st[:world - 1])
