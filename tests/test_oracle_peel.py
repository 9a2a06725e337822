"""Pins for the oracle's round-synchronous k-core peel (a3-a7): worked examples,
brute force, an independent serial algorithm, invariants, and goldens."""
import numpy as np
import pytest

import synth
from oracle import oracle as O
from oracle.brute import kcore_bruteforce


def core_ok(edges, n, k, core):
    """every core vertex has >= k edges lying wholly inside the core."""
    if len(edges) == 0:
        return not core.any() if k > 0 else True
    inside = core[edges].all(axis=1)
    deg = np.bincount(edges[inside].ravel(), minlength=n)
    return bool(np.all(deg[core.astype(bool)] >= k))


# ---- worked examples ----------------------------------------------------
def test_single_edge():
    res = O.sync_peel(np.array([[0, 1, 2]], dtype=np.uint32), 3, 2)
    assert res.rounds == 1 and res.survivors.tolist() == [0] and res.core_mask.sum() == 0


def test_spec_n6_example():
    e = np.array([[0, 1, 2], [0, 1, 3], [0, 1, 4], [2, 3, 4]], dtype=np.uint32)
    res = O.sync_peel(e, 6, 2)
    assert res.core_mask.tolist() == [1, 1, 1, 1, 1, 0]
    assert res.rounds == 1 and res.survivors.tolist() == [5]


def test_spec_chain_example():
    e = np.array([[0, 1, 2], [2, 3, 4], [4, 5, 6]], dtype=np.uint32)
    res = O.sync_peel(e, 7, 2, want_peel_round=True)
    assert res.rounds == 2 and res.survivors.tolist() == [2, 0]
    assert res.peel_round.tolist() == [1, 1, 2, 1, 2, 1, 1]
    assert res.killed.tolist() == [3, 0]


def test_empty_graph_and_zero_vertices():
    res = O.sync_peel(np.zeros((0, 3), dtype=np.uint32), 10, 2)
    assert res.rounds == 1 and res.survivors.tolist() == [0]
    res = O.sync_peel(np.zeros((0, 3), dtype=np.uint32), 0, 2)
    assert res.rounds == 0
    res = O.sync_peel(np.zeros((0, 3), dtype=np.uint32), 10, 0)  # k=0: nothing has deg < 0
    assert res.rounds == 0 and res.core_mask.all()


def test_long_chain_needs_linear_rounds():
    # chains need O(length) rounds (adversarial input; no round cap, P:14-19 hold for random graphs only)
    # a 2-uniform path of 41 edges loses its two end vertices per round
    e, n = synth.chain(41, 2)
    res = O.sync_peel(e, n, 2)
    assert n == 42 and res.rounds == 21 and res.core_mask.sum() == 0
    # a 3-uniform chain (S:118 shape) dies in 2 rounds: every edge has a degree-1 middle
    e, n = synth.chain(41, 3)
    res = O.sync_peel(e, n, 2)
    assert res.rounds == 2


def test_duplicate_edge_forms_2core():
    # k identical edges form a non-empty k-core
    e = np.array([[0, 1, 2], [0, 1, 2], [2, 3, 4]], dtype=np.uint32)
    res = O.sync_peel(e, 6, 2)
    assert res.core_mask.tolist() == [1, 1, 1, 0, 0, 0]
    assert res.rounds == 1


# ---- brute force and the serial algorithm ------------------------------------------------
@pytest.mark.parametrize("r", [2, 3, 4])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_bruteforce_tiny(r, k):
    rng = np.random.default_rng(100 * r + k)
    for trial in range(25):
        n = int(rng.integers(r, 12))
        m = int(rng.integers(0, 2 * n))
        e = synth.random_hypergraph(n, m, r, seed=1000 * r + 10 * k + trial)
        if trial % 5 == 0 and m > 0:
            e = np.concatenate([e, e[:1]])
        bf = kcore_bruteforce(e, n, k)
        sp = O.sync_peel(e, n, k)
        qp = O.queue_peel(e, n, k)
        assert np.array_equal(bf, sp.core_mask), (n, e.tolist(), k)
        assert np.array_equal(bf, qp)


@pytest.mark.parametrize("r,k,c", [(3, 2, 0.75), (3, 2, 0.9), (4, 2, 0.8), (3, 3, 1.6), (4, 3, 1.2)])
def test_sync_equals_queue_and_invariants(r, k, c):
    n = 30000
    m = int(c * n)
    e = O.gen_hypergraph(n, m, r, seed=int(c * 100) + r)
    sp = O.sync_peel(e, n, k, want_peel_round=True)
    qp = O.queue_peel(e, n, k)
    assert np.array_equal(sp.core_mask, qp)
    assert core_ok(e, n, k, sp.core_mask)
    # survivors non-increasing, strictly decreasing each counted round
    s = np.concatenate([[n], sp.survivors])
    assert np.all(np.diff(s.astype(np.int64)) < 0)
    assert s[-1] == sp.core_mask.sum()
    # |F_t| == #vertices with peel_round == t
    hist = np.bincount(sp.peel_round, minlength=sp.rounds + 1)
    assert np.array_equal(hist[1:], -np.diff(s.astype(np.int64)))
    # killed edges total == edges not wholly inside the core
    inside = sp.core_mask[e].all(axis=1)
    assert sp.killed.sum() == m - inside.sum()


def schedule_certificate(edges, n, k, peel_round):
    """Local certificate that peel_round is exactly the synchronous schedule
    (P:48-50): with p(v) the removal round (0 = never) and d(e) = min_{v in e} p(v)
    the edge's death round, deg_t(v) = #{e ni v : d(e) >= t}; v in F_t iff
    deg_t(v) < k and v alive at round t."""
    INF = np.iinfo(np.int64).max
    p = peel_round.astype(np.int64)
    p[p == 0] = INF
    d = p[edges].min(axis=1)
    # for each vertex: deg at start of its removal round < k, and deg at start of round p-1 >= k
    def deg_at(t_per_vertex):
        # number of incident edges with d(e) >= t(v) for each vertex v
        ok = d[:, None] >= t_per_vertex[edges]
        return np.bincount(edges[ok], minlength=n)

    removed = p != INF
    t_rm = np.where(removed, p, 1)
    deg_rm = deg_at(t_rm)
    assert np.all(deg_rm[removed] < k)
    t_prev = np.where(removed, np.maximum(p - 1, 1), 1)
    deg_prev = deg_at(t_prev)
    late = removed & (p >= 2)
    assert np.all(deg_prev[late] >= k)
    core = ~removed
    big = np.full(n, INF)
    deg_core = deg_at(np.where(core, big, 1))
    assert np.all(deg_core[core] >= k)


@pytest.mark.parametrize("r,k,c", [(3, 2, 0.8), (3, 2, 0.85), (4, 3, 1.3)])
def test_schedule_certificate_holds_for_oracle(r, k, c):
    n = 20000
    e = O.gen_hypergraph(n, int(c * n), r, seed=99)
    sp = O.sync_peel(e, n, k, want_peel_round=True)
    schedule_certificate(e, n, k, sp.peel_round)
    # and it rejects a perturbed schedule
    bad = sp.peel_round.copy()
    i = int(np.flatnonzero(bad >= 2)[0])
    bad[i] -= 1
    with pytest.raises(AssertionError):
        schedule_certificate(e, n, k, bad)


# ---- goldens from an independent implementation ----------------------------------------
def test_c1_golden(goldens):
    g = goldens["C1"]
    e = O.gen_hypergraph(g["n"], g["m"], g["r"], g["seed"])
    sp = O.sync_peel(e, g["n"], g["k"])
    assert sp.rounds == g["rounds"]
    assert sp.survivors.tolist() == g["survivors"]
    assert sp.killed.tolist() == g["killed"]
    assert sp.core_mask.sum() == g["core"]


@pytest.mark.parametrize("name", ["C4a_small", "C4b_small"])
def test_reduced_c4_golden(goldens, name):
    g = goldens[name]
    e = O.gen_hypergraph(g["n"], g["m"], g["r"], g["seed"])
    sp = O.sync_peel(e, g["n"], g["k"])
    assert sp.rounds == g["rounds"]
    assert sp.core_mask.sum() == g["core"]
    assert sp.survivors[:5].tolist() == g["survivors_head"]
    assert sp.killed[:3].tolist() == g["killed_head"]
