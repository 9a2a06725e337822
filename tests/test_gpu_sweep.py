"""GPU parity for peel_sweep: per-trial rounds and core size equal the oracle's on
every trial -- on the per-trial group path (k = 2, r <= 4: one trial per group of CTAs,
32-bit states in L2, rows regenerated from the seed), on the union path (batched
trials as one disjoint union; k = 3, or PEEL_SWEEP_GROUPS=0), and through the group
path's overflow fallback -- and the paper's Table 1 protocol reproduced on the GPU."""
import numpy as np
import pytest
import torch

import paper_1302_7014_b200 as pk
from oracle import oracle as O
from paper_1302_7014_b200 import trials as S
from peeltest_util import load_table

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.mark.parametrize("r,k", [(3, 2), (4, 2), (3, 3)])
@pytest.mark.parametrize("batch", [1, 5, 24])
def test_sweep_matches_oracle_per_trial(r, k, batch):
    n = 30011
    cs = np.linspace(0.70, 0.90, 12) if k == 2 else np.linspace(1.45, 1.65, 12)
    m = np.array([int(c * n) for c in cs] * 2, dtype=np.uint64)
    seeds = np.arange(500, 500 + m.size, dtype=np.uint64)
    rounds, core = pk.sweep(n, r, k, m, seeds, batch=batch, device=DEV)
    for t in range(m.size):
        ref = O.sync_peel(O.gen_hypergraph(n, int(m[t]), r, int(seeds[t])), n, k)
        assert rounds[t] == ref.rounds and core[t] == int(ref.core_mask.sum()), t


@pytest.mark.parametrize("path", ["groups", "union"])
def test_sweep_c5s_shape(path, monkeypatch):
    # union: batch * n > 2^23, the union takes the binned build path; groups: the C5s path
    if path == "union":
        monkeypatch.setenv("PEEL_SWEEP_GROUPS", "0")
    n, r, k = 1_000_000, 3, 2
    m, seeds = S.paper_trials(12, n=n, per_c=1)
    rounds, core = pk.sweep(n, r, k, m, seeds, batch=12, device=DEV)
    for t in (0, 5, 11):
        ref = O.sync_peel(O.gen_hypergraph(n, int(m[t]), r, int(seeds[t])), n, k)
        assert rounds[t] == ref.rounds and core[t] == int(ref.core_mask.sum())
    # and every trial equals a standalone peel_kcore on the GPU
    for t in range(12):
        e = pk.gen_hypergraph(n, int(m[t]), r, int(seeds[t]), device=DEV)
        res = pk.peel_kcore(e, n, k)
        assert res.rounds == rounds[t] and int(res.core_mask.sum().item()) == core[t]


def test_table1_first_row_on_gpu():
    # Table 1: r=4, k=2, n=10^4, 1000 trials: c=0.7 -> Failed 0, rounds 12.504;
    # c=0.85 -> Failed 1000, rounds 10.773.  Tolerance: 4 standard errors.
    rows = load_table("paper_table1.txt")
    n = 10_000
    for c, col in ((0.7, 1), (0.85, 7)):
        m = np.full(1000, int(c * n), dtype=np.uint64)
        seeds = np.arange(1000, dtype=np.uint64) + 77
        rounds, core = pk.sweep(n, 4, 2, m, seeds, batch=250, device=DEV)
        failed = int((core > 0).sum())
        assert failed == int(rows[0][col])
        se = rounds.std(ddof=1) / np.sqrt(rounds.size)
        assert abs(rounds.mean() - float(rows[0][col + 1])) < 4 * se + 0.02


@pytest.mark.parametrize("groups", ["1", "7", None])
def test_sweep_group_counts(groups, monkeypatch):
    # one group (every trial in turn on the whole grid), a few, and the default (more groups
    # than trials): identical per-trial results; near-threshold trials run long tails
    if groups:
        monkeypatch.setenv("PEEL_SWEEP_GROUPS", groups)
    n, r, k = 50_000, 3, 2
    cs = np.linspace(0.80, 0.84, 9)
    m = np.array([int(c * n) for c in cs], dtype=np.uint64)
    seeds = np.arange(900, 900 + m.size, dtype=np.uint64)
    rounds, core = pk.sweep(n, r, k, m, seeds, batch=4, device=DEV)
    for t in range(m.size):
        ref = O.sync_peel(O.gen_hypergraph(n, int(m[t]), r, int(seeds[t])), n, k)
        assert rounds[t] == ref.rounds and core[t] == int(ref.core_mask.sum()), t


def test_sweep_group_overflow_falls_back(monkeypatch):
    # a 3-bit count field overflows at degree 8 (present at n = 20011, c = 0.9, r = 4): the
    # scan's sum check flags those trials and the host peels them on the union path
    monkeypatch.setenv("PEEL_SWEEP_CB", "3")
    n, r, k = 20011, 4, 2
    m = np.array([int(c * n) for c in (0.5, 0.7, 0.9, 1.2)], dtype=np.uint64)
    seeds = np.arange(41, 41 + m.size, dtype=np.uint64)
    rounds, core = pk.sweep(n, r, k, m, seeds, batch=2, device=DEV)
    for t in range(m.size):
        ref = O.sync_peel(O.gen_hypergraph(n, int(m[t]), r, int(seeds[t])), n, k)
        assert rounds[t] == ref.rounds and core[t] == int(ref.core_mask.sum()), t


def test_sweep_group_edge_cases():
    # m = 0 (every vertex in F_1, nothing to kill), r = 2 with m above the threshold, a trial
    # with n = r, and m = 1
    for n, r, m in ((1000, 3, 0), (4096, 2, 3000), (3, 3, 5), (10, 4, 1)):
        mm = np.array([m, m], dtype=np.uint64)
        seeds = np.array([5, 6], dtype=np.uint64)
        rounds, core = pk.sweep(n, r, 2, mm, seeds, batch=1, device=DEV)
        for t in range(2):
            ref = O.sync_peel(O.gen_hypergraph(n, m, r, int(seeds[t])), n, 2)
            assert rounds[t] == ref.rounds and core[t] == int(ref.core_mask.sum()), (n, r, m)
