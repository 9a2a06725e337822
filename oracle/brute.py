"""Brute-force k-core on tiny hypergraphs (TEST INFRASTRUCTURE ONLY).

Definition: the k-core is the maximal sub-hypergraph in
which every vertex has degree at least k.  For a vertex set S, the induced
sub-hypergraph keeps the edges whose endpoints all lie in S.  The union of two
sets with the property has it too, so the k-core's vertex set is the union of
ALL subsets S of [0, n) in which every vertex has >= k induced edges.  This
enumerates all 2^n subsets -- pure Python, n <= 14.
"""
from __future__ import annotations

import numpy as np


def kcore_bruteforce(edges, n: int, k: int) -> np.ndarray:
    if n > 16:
        raise ValueError("brute force is for n <= 16")
    emasks = []
    for e in np.asarray(edges).reshape(-1, np.asarray(edges).shape[-1] if len(edges) else 1):
        mask = 0
        for u in e:
            mask |= 1 << int(u)
        emasks.append(mask)
    union = 0
    for S in range(1, 1 << n):
        deg = [0] * n
        for em in emasks:
            if em & S == em:
                v = em
                while v:
                    low = v & -v
                    deg[low.bit_length() - 1] += 1
                    v ^= low
        ok = True
        s = S
        while s:
            low = s & -s
            if deg[low.bit_length() - 1] < k:
                ok = False
                break
            s ^= low
        if ok:
            union |= S
    return np.array([(union >> v) & 1 for v in range(n)], dtype=np.uint8)
