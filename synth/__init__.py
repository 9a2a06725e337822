"""Seeded synthetic INPUTS shared by the oracle tests and the GPU parity tests.

Holds none of the method's arithmetic: it only produces edge lists / key lists
as plain numpy arrays (numpy PCG64 streams), which both sides then consume.
The paper-shaped workloads themselves (G^r_{n,cn}, IBLT keys) come from the
counter-based generator that each side implements independently
(oracle/peel_oracle.c and the CUDA generator); this module is for the small
structured and adversarial cases: ragged sizes, chains, duplicates, stars,
isolated vertices, degenerate k.
"""
from __future__ import annotations

import numpy as np


def random_hypergraph(n: int, m: int, r: int, seed: int) -> np.ndarray:
    """m independent edges, each r distinct vertices uniform over [0,n)."""
    rng = np.random.default_rng(seed)
    if m == 0:
        return np.zeros((0, r), dtype=np.uint32)
    keys = rng.random((m, n)) if n <= 64 else None
    if keys is not None:
        return np.argsort(keys, axis=1)[:, :r].astype(np.uint32)
    out = np.empty((m, r), dtype=np.uint32)
    for e in range(m):
        out[e] = rng.choice(n, size=r, replace=False)
    return out


def chain(length: int, r: int = 3) -> tuple[np.ndarray, int]:
    """Path of `length` r-edges, consecutive edges sharing one vertex
    (S:118's example for r=3, length=3).  Needs ~length rounds for k=2."""
    edges = []
    v = 0
    for _ in range(length):
        edges.append(list(range(v, v + r)))
        v += r - 1
    n = v + 1
    return np.array(edges, dtype=np.uint32).reshape(-1, r), n


def with_duplicates(n: int, m: int, r: int, seed: int, ndup: int = 2) -> np.ndarray:
    """A random hypergraph whose first edge is repeated ndup times (P:296-301:
    k identical edges form a non-empty k-core)."""
    e = random_hypergraph(n, m, r, seed)
    if m == 0:
        return e
    return np.concatenate([e, np.repeat(e[:1], ndup - 1, axis=0)], axis=0)


def star(n: int, r: int = 3) -> np.ndarray:
    """Edges {0, 1+i(r-1), ..., (i+1)(r-1)}: vertex 0 has high degree, leaves degree 1."""
    m = (n - 1) // (r - 1)
    rows = [[0] + list(range(1 + i * (r - 1), 1 + (i + 1) * (r - 1))) for i in range(m)]
    return np.array(rows, dtype=np.uint32).reshape(-1, r)


def complete_r_graph(n: int, r: int) -> np.ndarray:
    """Every r-subset of [0,n) once (dense core)."""
    from itertools import combinations
    return np.array(list(combinations(range(n), r)), dtype=np.uint32).reshape(-1, r)


def random_keys(nkeys: int, seed: int) -> np.ndarray:
    """nkeys distinct uniform 64-bit keys (numpy PCG64 stream, deduplicated)."""
    rng = np.random.default_rng(seed)
    keys = np.unique(rng.integers(0, 2**64 - 1, size=int(nkeys * 1.01) + 8, dtype=np.uint64,
                                  endpoint=True))
    rng.shuffle(keys)
    return keys[:nkeys].copy()
