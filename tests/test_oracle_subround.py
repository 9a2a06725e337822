"""Pins for the oracle's subtable model and subround peel:
the k-core is unchanged (brute force, plain peel), Table 4's mean subrounds,
Table 5's per-subround survivors, and the subround-vs-round bound."""
import numpy as np
import pytest

import synth
from oracle import oracle as O
from oracle.brute import kcore_bruteforce
from peeltest_util import load_table


def test_partitioned_generator_model():
    # one vertex per class; S:53 example: per-class degree sums equal m
    n, m, r = 12, 200, 3
    e = O.gen_partitioned(n, m, r, 5)
    cls = e // (n // r)
    assert np.all(cls == np.arange(r))
    assert np.all(np.bincount(e.ravel(), minlength=n).reshape(r, -1).sum(axis=1) == m)
    # uniform within each class
    n, m = 4000, 200000
    e = O.gen_partitioned(n, m, 4, 9)
    for j in range(4):
        c = np.bincount(e[:, j] - j * (n // 4), minlength=n // 4)
        assert c.size == n // 4 and abs(c.mean() - m / (n // 4)) < 1e-9
        assert c.std() < 2 * np.sqrt(m / (n // 4))
    with pytest.raises(ValueError):
        O.gen_partitioned(10, 5, 3, 1)  # r must divide n


@pytest.mark.parametrize("r,k", [(2, 2), (3, 2), (3, 3), (4, 2)])
def test_subround_core_is_the_kcore(r, k):
    rng = np.random.default_rng(r * 10 + k)
    for trial in range(30):
        n = r * int(rng.integers(1, 12 // r + 1))
        m = int(rng.integers(0, 3 * n))
        if trial % 2:
            e = O.gen_partitioned(n, m, r, trial)
        else:
            e = synth.random_hypergraph(n, m, r, seed=trial)  # classes still defined for any graph
        sr = O.subround_peel(e, n, k)
        assert np.array_equal(sr.core_mask, kcore_bruteforce(e, n, k))


@pytest.mark.parametrize("c", [0.7, 0.75, 0.85])
def test_subround_vs_plain_on_paper_shapes(c):
    n, r = 40000, 4
    for s in range(4):
        e = O.gen_partitioned(n, int(c * n), r, 100 + s)
        sr = O.subround_peel(e, n, 2)
        pl = O.sync_peel(e, n, 2)
        assert np.array_equal(sr.core_mask, pl.core_mask)          # S:140 core uniqueness
        assert sr.subrounds <= r * pl.rounds
        assert sr.rounds == -(-sr.subrounds // r)
        s_ = np.concatenate([[n], sr.survivors])
        assert np.all(np.diff(s_.astype(np.int64)) <= 0)
        assert s_[-1] == sr.core_mask.sum()


@pytest.mark.parametrize("c,col", [(0.7, 2), (0.75, 4)])
def test_table4_first_row(c, col):
    # Table 4: r=4, k=2, n=10^4, 1000 trials: mean subrounds 26.018 / 47.732, no failures
    rows = load_table("paper_table4.txt")
    n = 10_000
    subs, fails = [], 0
    for s in range(300):
        sr = O.subround_peel(O.gen_partitioned(n, int(c * n), 4, 9000 + s), n, 2)
        subs.append(sr.subrounds)
        fails += int(sr.core_mask.any())
    se = np.std(subs, ddof=1) / np.sqrt(len(subs))
    assert fails == int(rows[0][col - 1])
    assert abs(np.mean(subs) - float(rows[0][col])) < 4 * se + 0.02


def test_table5_experiment_column():
    # Table 5: per-subround survivors, r=4, k=2, c=0.7, n=10^6
    rows = load_table("paper_table5.txt")
    n = 10**6
    runs = []
    for s in range(4):
        sr = O.subround_peel(O.gen_partitioned(n, 700000, 4, 500 + s), n, 2)
        sv = np.zeros(28)
        L = min(sr.subrounds, 28)
        sv[:L] = sr.survivors[:L]
        runs.append(sv)
    runs = np.array(runs)
    mean, se = runs.mean(0), runs.std(0, ddof=1) / 2
    for i, row in enumerate(rows[:22]):
        exp = float(row[3])
        assert abs(mean[i] - exp) < max(0.004 * exp, 4 * se[i] + 0.002 * exp), (row, mean[i])
