"""Pins for the oracle's generator and hashes (a1), against published KATs and
an independent implementation's goldens (tests/golden/)."""
import hashlib
import math

import numpy as np
import pytest

from oracle import oracle as O
from peeltest_util import load_table


def test_philox_random123_kats():
    for row in load_table("kat_philox4x32_10.txt"):
        v = [int(x, 16) for x in row]
        assert O.philox4x32_10(v[0:4], v[4:6]) == tuple(v[6:10])


def test_splitmix64_reference_stream():
    expect = [int(x[0], 16) for x in load_table("kat_splitmix64.txt")]
    got = [int(k) for k in O.gen_keys(3, 0)]
    assert got == expect


def test_c1_edges_golden(goldens):
    g = goldens["C1"]
    e = O.gen_hypergraph(g["n"], g["m"], g["r"], g["seed"])
    assert e[:3].tolist() == g["edges_head"]
    assert hashlib.sha256(e.tobytes()).hexdigest() == g["sha256"]


@pytest.mark.parametrize("name", ["C4a_small", "C4b_small"])
def test_reduced_c4_edges_golden(goldens, name):
    g = goldens[name]
    e = O.gen_hypergraph(g["n"], g["m"], g["r"], g["seed"])
    assert e[:1].tolist() == g["edges_head"]
    assert hashlib.sha256(e.tobytes()).hexdigest() == g["sha256"]


@pytest.mark.parametrize("name", ["C3", "C4a", "C4b", "C5"])
def test_full_scale_first_edge(goldens, name):
    # the generator is counter-based: any edge can be computed on its own
    g = goldens[name]
    assert O.gen_edge(g["seed"], g["n"], g["r"], 0).tolist() == g["edges_head"][0]


def test_c2_hashes_golden(goldens):
    g = goldens["C2"]
    assert O.seed_h(g["seed"]) == int(g["seed_h"], 16)
    assert O.seed_c(g["seed"]) == int(g["seed_c"], 16)
    k0 = int(O.gen_keys(1, g["seed"])[0])
    assert k0 == int(g["key0"], 16)
    assert O.cells_of(k0, g["cells"], g["r"], g["seed"]).tolist() == g["key0_cells"]
    assert O.checksum(k0, g["seed"]) == int(g["key0_checksum"], 16)


def test_generator_model_properties():
    # P:89-91 r distinct vertices; handshake sum deg = r m;
    # degrees ~ Poisson(rc)
    n, m, r = 200000, 150000, 3
    e = O.gen_hypergraph(n, m, r, 11)
    assert e.max() < n
    s = np.sort(e, axis=1)
    assert np.all(s[:, 1:] != s[:, :-1])
    deg = np.bincount(e.ravel(), minlength=n)
    assert deg.sum() == r * m
    lam = r * m / n
    hist = np.bincount(deg) / n
    pois = np.array([math.exp(-lam) * lam ** i / math.factorial(i) for i in range(len(hist))])
    tv = 0.5 * np.abs(hist - pois).sum() + 0.5 * (1 - pois.sum())
    assert tv < 0.02
    # uniform over vertices: every slot is uniform (chi-square-ish on 10 buckets)
    for j in range(r):
        b = np.bincount((e[:, j].astype(np.uint64) * 10 // n).astype(np.int64), minlength=10)
        assert np.all(np.abs(b - m / 10) < 5 * math.sqrt(m / 10))


def test_generator_determinism_and_seed_separation():
    a = O.gen_hypergraph(1000, 500, 4, 7)
    b = O.gen_hypergraph(1000, 500, 4, 7)
    c = O.gen_hypergraph(1000, 500, 4, 8)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)


def test_small_n_equals_r_gives_permutations():
    # n == r: every edge must be a permutation of [0, r)
    e = O.gen_hypergraph(4, 100, 4, 3)
    assert np.all(np.sort(e, axis=1) == np.arange(4))


def test_iblt_cells_distinct_and_uniform():
    C, r = 1000, 4
    keys = O.gen_keys(20000, 5)
    cells = np.array([O.cells_of(int(x), C, r, 5) for x in keys[:2000]])
    s = np.sort(cells, axis=1)
    assert np.all(s[:, 1:] != s[:, :-1])
    assert cells.max() < C
    # keys are distinct (SplitMix64 increments a bijection)
    assert np.unique(keys).size == keys.size
