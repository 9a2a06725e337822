"""GPU parity of the vertex-partitioned instance (peel_kcore_dist) in virtual-shard mode:
P shards in one process on one GPU, exchanging killed-edge ids through the same send /
receive buffers and kernels the NCCL transport uses.  Bit-exact against the oracle and
against the single-GPU peel for P in {1, 2, 3, 8} (SURVEY §4 layer 5)."""
import numpy as np
import pytest
import torch

import paper_1302_7014_b200 as pk
import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def to_dev(e):
    return torch.from_numpy(np.ascontiguousarray(e, dtype=np.uint32).view(np.int32)).to(DEV)


def check(e_np, n, k, P):
    ref = O.sync_peel(e_np, n, k)
    comm = pk.Comm.virtual_shards(P)
    res = pk.peel_kcore_dist(comm, to_dev(e_np), n, k)
    assert res.rounds == ref.rounds, (P, res.rounds, ref.rounds)
    assert res.survivors.tolist() == ref.survivors.tolist()
    assert res.killed.tolist() == ref.killed.tolist()
    assert np.array_equal(res.core_mask.cpu().numpy(), ref.core_mask)


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_examples_and_degenerate(P):
    check(np.array([[0, 1, 2], [0, 1, 3], [0, 1, 4], [2, 3, 4]], dtype=np.uint32), 8, 2, P)
    check(np.array([[0, 1, 2], [2, 3, 4], [4, 5, 6]], dtype=np.uint32), 9, 2, P)
    e, n = synth.chain(101, 2)
    check(e, n, 2, P)
    check(np.array([[0, 5, 7], [0, 5, 7]], dtype=np.uint32), 8, 2, P)  # duplicate edge
    check(np.zeros((0, 3), dtype=np.uint32), 16, 2, P)
    check(synth.star(2001, 3), 2001, 1, P)


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("r,c", [(3, 0.75), (3, 0.85), (4, 0.8), (2, 0.45)])
def test_random_vs_oracle(P, r, c):
    n = 100003
    e = O.gen_hypergraph(n, int(c * n), r, seed=17 + P)
    check(e, n, 2, P)


def test_full_c3_shape_matches_single_gpu(oracle_goldens):
    g = oracle_goldens["C4a"]
    e = pk.gen_hypergraph(g["n"], g["m"], g["r"], g["seed"], device=DEV)
    res = pk.peel_kcore_dist(pk.Comm.virtual_shards(4), e, g["n"], 2)
    assert res.rounds == g["rounds"] and int(res.core_mask.sum().item()) == g["core"]
    assert res.survivors.tolist() == g["survivors"] and res.killed.tolist() == g["killed"]
    pk._ws_cache.clear()
    torch.cuda.empty_cache()


NCCL_WORLD1 = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["REPO"]); sys.path.insert(0, os.path.join(os.environ["REPO"], "tests"))
import paper_1302_7014_b200 as pk
from oracle import oracle as O
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%s" % os.environ["PORT"], rank=0, world_size=1,
                        device_id=torch.device("cuda:0"))
comm = pk.Comm.from_process_group()
for (n, c, r, seed) in [(100003, 0.75, 3, 5), (50021, 0.85, 3, 6), (40009, 0.8, 4, 7),
                        ((1 << 24) + 12345, 0.75, 3, 8)]:  # the last one: binned build and rounds
    e = O.gen_hypergraph(n, int(c * n), r, seed)
    ref = O.sync_peel(e, n, 2)
    res = pk.peel_kcore_dist(comm, torch.from_numpy(e.view(np.int32)).cuda(), n, 2)
    assert res.rounds == ref.rounds and res.survivors.tolist() == ref.survivors.tolist()
    assert res.killed.tolist() == ref.killed.tolist()
    assert np.array_equal(res.core_mask.cpu().numpy(), ref.core_mask)
for (C, r, load, blog) in [(100003, 3, 0.75, 0), (1 << 18, 3, 0.8, 12)]:
    keys = O.gen_keys(int(load * C), 5)
    o = O.Iblt(C, r, 3, blog=blog)
    o.insert(keys)
    ref = o.peel(cap_keys=keys.size + 1)
    res = pk.iblt_dist_recover(comm, C, r, 3, torch.from_numpy(keys.view(np.int64)).cuda(), blog=blog)
    assert res.rounds == ref.rounds and res.per_round.tolist() == ref.per_round.tolist()
    assert res.complete == ref.complete
    assert np.array_equal(np.sort(res.keys.cpu().numpy().view(np.uint64)), np.sort(ref.keys))
del comm
dist.destroy_process_group()
print("NCCL_OK")
"""


def test_nccl_transport_world1():
    """The real NCCL transport (unique id broadcast over a torch.distributed NCCL group,
    ncclCommInitRank, the per-round allgather / allreduce / grouped send-recv) at world
    size 1: the only size one GPU allows.  Same results as the oracle."""
    import os
    import socket
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    env = dict(os.environ, REPO=repo, PORT=str(port))
    out = subprocess.run([sys.executable, "-c", NCCL_WORLD1], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "NCCL_OK" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]


NCCL_WATCHDOG = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["REPO"])
import paper_1302_7014_b200 as pk
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%s" % os.environ["PORT"], rank=0, world_size=1,
                        device_id=torch.device("cuda:0"))
comm = pk.Comm.from_process_group()
n = (1 << 24) + 12345
e = pk.gen_hypergraph(n, int(0.75 * n), 3, 8, device=torch.device("cuda:0"))
os.environ["PEEL_NCCL_TIMEOUT_S"] = "1e-9"  # every sync after NCCL work "times out"
codes = []
for _ in range(2):
    try:
        pk.peel_kcore_dist(comm, e, n, 2)
        codes.append(0)
    except pk.PeelError as ex:
        codes.append(ex.status)
assert codes == [pk.PEEL_ENCCL, pk.PEEL_ENCCL], codes  # aborted, and stays aborted
del comm
print("WATCHDOG_OK")
"""


def test_nccl_watchdog_aborts():
    """The NCCL watchdog sync (comm_sync): past PEEL_NCCL_TIMEOUT_S it aborts the communicator
    and the call fails with PEEL_ENCCL instead of hanging on a dead peer; later calls on the
    aborted communicator fail the same way."""
    import os
    import socket
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    env = dict(os.environ, REPO=repo, PORT=str(port))
    out = subprocess.run([sys.executable, "-c", NCCL_WATCHDOG], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "WATCHDOG_OK" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]


@pytest.mark.parametrize("P", [1, 2, 3])
def test_binned_shard_build_vs_oracle(P):
    """Shards larger than 2^23 vertices use the binned build restricted to their endpoints
    (shard.h): bit-exact against the oracle, with a ragged n; then the same graph with a hub
    that overflows a bin (direct-build fallback)."""
    n = (1 << 24) + 12345
    m = int(0.75 * n)
    e = O.gen_hypergraph(n, m, 3, seed=31 + P)
    check(e, n, 2, P)
    hub = e[: 400000].copy()
    hub[:, 0] = 7                      # vertex 7 is in 400k edges: its bin overflows
    hub[:, 1] = np.where(hub[:, 1] == 7, 8, hub[:, 1])
    hub[:, 2] = np.where(hub[:, 2] == 7, 9, hub[:, 2])
    ok = (hub[:, 1] != hub[:, 2]) & (hub[:, 1] != 7) & (hub[:, 2] != 7)
    check(np.concatenate([hub[ok], e[400000:]]), n, 2, P)


@pytest.mark.parametrize("P", [4, 5])
def test_narrow_shard_filter_build_vs_oracle(P, monkeypatch):
    """Shards of > 2^23 vertices that are at most n/4 wide take the filter build (a streaming
    pass keeps the shard's endpoints in per-block regions, a second bins them): bit-exact
    against the oracle -- and so are the region-overflow fallback to the chunked partition
    (regions forced small) and the chunked partition itself (PEEL_SHARD_FILTER=0)."""
    n = P * ((1 << 23) + 4099) + 17
    m = int(0.78 * n)
    e = O.gen_hypergraph(n, m, 3, seed=60 + P)
    ref = O.sync_peel(e, n, 2)
    ed = torch.from_numpy(e.view(np.int32)).to(DEV)
    for env in ({}, {"PEEL_SHARD_FILTER_CAP": "5000"}, {"PEEL_SHARD_FILTER": "0"}):
        for name in ("PEEL_SHARD_FILTER_CAP", "PEEL_SHARD_FILTER"):
            if name in env:
                monkeypatch.setenv(name, env[name])
            else:
                monkeypatch.delenv(name, raising=False)
        res = pk.peel_kcore_dist(pk.Comm.virtual_shards(P), ed, n, 2)
        assert res.rounds == ref.rounds, env
        assert res.survivors.tolist() == ref.survivors.tolist() and res.killed.tolist() == ref.killed.tolist(), env
        assert np.array_equal(res.core_mask.cpu().numpy(), ref.core_mask), env
    del ed, res
    pk._ws_cache.clear()
    torch.cuda.empty_cache()


# ---- cell-partitioned IBLT -------------------------------------------------
def iblt_check(C, r, seed, keys_np, P, blog=0):
    o = O.Iblt(C, r, seed, blog=blog)
    o.insert(keys_np)
    ref = o.peel(cap_keys=keys_np.size + 1)
    comm = pk.Comm.virtual_shards(P)
    kd = torch.from_numpy(np.ascontiguousarray(keys_np).view(np.int64)).to(DEV)
    res = pk.iblt_dist_recover(comm, C, r, seed, kd, blog=blog)
    assert res.rounds == ref.rounds, (P, res.rounds, ref.rounds)
    assert res.per_round.tolist() == ref.per_round.tolist()
    assert res.complete == ref.complete
    assert np.array_equal(np.sort(res.keys.cpu().numpy().view(np.uint64)), np.sort(ref.keys))


@pytest.mark.parametrize("P", [1, 2, 3, 8])
@pytest.mark.parametrize("r,load", [(3, 0.75), (3, 0.85), (4, 0.7), (2, 0.4)])
def test_iblt_dist_vs_oracle(P, r, load):
    C = 100003
    keys = synth.random_keys(int(load * C), 40 + P + r)
    iblt_check(C, r, 5 + r, keys, P)


@pytest.mark.parametrize("P", [2, 5])
def test_iblt_dist_blocked_and_edges(P):
    iblt_check(1 << 16, 3, 9, synth.random_keys(int(0.8 * (1 << 16)), 3), P, blog=12)
    iblt_check(64, 3, 1, synth.random_keys(40, 4), P)       # shards of 32 cells, some empty
    iblt_check(1000, 3, 1, np.zeros(0, dtype=np.uint64), P)  # no keys
    iblt_check(1000, 3, 1, np.array([0, 7], dtype=np.uint64), P)
