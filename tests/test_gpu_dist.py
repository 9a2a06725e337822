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


def test_full_c3_shape_matches_single_gpu(goldens):
    g = goldens["C4a"]
    e = pk.gen_hypergraph(g["n"], g["m"], g["r"], g["seed"], device=DEV)
    res = pk.peel_kcore_dist(pk.Comm.virtual_shards(4), e, g["n"], 2)
    assert res.rounds == g["rounds"] and int(res.core_mask.sum().item()) == g["core"]
    assert res.survivors[:4].tolist() == g["survivors_head"] and res.killed[-4:].tolist() == g["killed_tail"]
    pk._ws_cache.clear()
    torch.cuda.empty_cache()
