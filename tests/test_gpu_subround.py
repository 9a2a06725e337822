"""GPU parity of the subround (subtable) variant, PEEL_FLAG_SUBROUNDS,
against the oracle's literal subround peel: flattened subround count, survivors
after every subround, core mask; the partitioned generator; Table 4 on the GPU."""
import numpy as np
import pytest
import torch

import paper_1302_7014_b200 as pk
import synth
from oracle import oracle as O
from peeltest_util import load_table

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def to_dev(e):
    return torch.from_numpy(np.ascontiguousarray(e, dtype=np.uint32).view(np.int32)).to(DEV)


def check(e_np, n, k):
    ref = O.subround_peel(e_np, n, k)
    res = pk.peel_kcore(to_dev(e_np) if len(e_np) else torch.zeros((0, e_np.shape[1]), dtype=torch.int32, device=DEV),
                        n, k, flags=pk.PEEL_FLAG_SUBROUNDS, want_peel_round=True)
    assert res.rounds == ref.subrounds, (res.rounds, ref.subrounds)
    assert res.survivors.tolist() == ref.survivors.tolist()
    assert np.array_equal(res.core_mask.cpu().numpy(), ref.core_mask)
    # every removed vertex's flattened subround is one of its class: (s - 1) % r == class
    pr = res.peel_round.cpu().numpy().view(np.uint32).astype(np.int64)
    r = e_np.shape[1]
    rem = pr > 0
    cls = np.arange(n) // (n // r)
    assert np.all((pr[rem] - 1) % r == cls[rem])
    assert np.array_equal(np.bincount(pr[rem], minlength=res.rounds + 1)[1:],
                          -np.diff(np.concatenate([[n], res.survivors]).astype(np.int64)))
    return ref


@pytest.mark.parametrize("n,m,r,seed", [(12, 200, 3, 5), (1000, 5000, 4, 1), (4096 * 3, 9000, 3, 2), (10, 3, 2, 0)])
def test_generator_matches_oracle(n, m, r, seed):
    got = pk.gen_partitioned(n, m, r, seed, device=DEV).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, O.gen_partitioned(n, m, r, seed))


@pytest.mark.parametrize("r", [2, 3, 4, 5])
@pytest.mark.parametrize("c", [0.45, 0.7, 0.8, 0.95])
def test_partitioned_vs_oracle(r, c):
    n = r * 20011
    e = O.gen_partitioned(n, int(c * n), r, seed=int(100 * c) + r)
    check(e, n, 2)
    check(e, n, 1)


@pytest.mark.parametrize("r", [3, 4])
def test_general_graph_same_class_crossings(r):
    # non-partitioned edges: a class-j vertex can cross during subround j itself
    for s in range(4):
        n = r * 3001
        e = synth.random_hypergraph(n, int(0.7 * n), r, seed=s)
        check(e, n, 2)
    e, n = synth.chain(300, 3)
    n2 = n + (-n) % 3
    check(e, n2, 2)


def test_binned_build_size():
    n = 4 * (1 << 21) + 4 * 1000  # > 2^23: binned build, then the subround loop
    e = O.gen_partitioned(n, int(0.7 * n), 4, 7)
    check(e, n, 2)


def test_rejects_bad_arguments():
    e = to_dev(np.array([[0, 1, 2]], dtype=np.uint32))
    with pytest.raises(pk.PeelError):
        pk.peel_kcore(e, 7, 2, flags=pk.PEEL_FLAG_SUBROUNDS)  # 3 does not divide 7
    with pytest.raises(pk.PeelError):
        pk.peel_kcore(e, 9, 3, flags=pk.PEEL_FLAG_SUBROUNDS)  # k >= 3 not supported in this mode


def test_table4_first_row_on_gpu():
    # Table 4: r=4, k=2, n=10^4, c=0.7 -> 26.018 subrounds; c=0.75 -> 47.732
    rows = load_table("paper_table4.txt")
    n = 10_000
    for c, col in ((0.7, 2), (0.75, 4)):
        subs = []
        for s in range(300):
            e = pk.gen_partitioned(n, int(c * n), 4, 20_000 + s, device=DEV)
            res = pk.peel_kcore(e, n, 2, flags=pk.PEEL_FLAG_SUBROUNDS)
            assert int(res.core_mask.sum().item()) == 0
            subs.append(res.rounds)
        se = np.std(subs, ddof=1) / np.sqrt(len(subs))
        assert abs(np.mean(subs) - float(rows[0][col])) < 4 * se + 0.02
