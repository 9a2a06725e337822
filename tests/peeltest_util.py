"""Shared test helpers (fixture loading).  Imported by tests as `peeltest_util`."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_table(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(line.split())
    return rows


def load_goldens():
    """The independent implementation's goldens quoted by SURVEY.md §8 c3 (pins for the oracle)."""
    with open(os.path.join(GOLDEN, "survey_c3_goldens.json")) as f:
        return json.load(f)


def load_oracle_goldens():
    """Full-size results written by tools/make_oracle_goldens.py from oracle/ alone (the
    expected values of the GPU tests; checked against load_goldens() on CPU)."""
    with open(os.path.join(GOLDEN, "oracle_goldens.json")) as f:
        return json.load(f)


# ---------------------------------------------------------------------------
# forged IBLT tables (R28): cell arrays built here, loaded into both the oracle
# table and the device table, so both sides start from the same bytes
# ---------------------------------------------------------------------------
def key_cells(O, x, C, r, seed, mode, blog=0):
    """x's r cells under the table's hashing mode ('plain', 'subtables', 'blocked')."""
    if mode == "subtables":
        return [int(c) for c in O.cells_of_subtable(x, C, r, seed)]
    if mode == "blocked":
        return [int(c) for c in O.cells_of_blocked(x, C, r, seed, blog)]
    return [int(c) for c in O.cells_of(x, C, r, seed)]


def honest_cells(O, keys, C, r, seed, mode, blog=0):
    """(count int64, keySum uint64, hashSum uint32) of the insert-only table of `keys`."""
    import numpy as np
    count = np.zeros(C, dtype=np.int64)
    ks = np.zeros(C, dtype=np.uint64)
    hs = np.zeros(C, dtype=np.uint32)
    for x in keys.tolist():
        h = O.checksum(x, seed)
        for c in key_cells(O, x, C, r, seed, mode, blog):
            count[c] += 1
            ks[c] ^= np.uint64(x)
            hs[c] ^= np.uint32(h)
    return count, ks, hs


def forge_foreign_cells(O, cells, C, r, seed, mode, nforge, rng_seed, blog=0):
    """Overwrite `nforge` EMPTY cells c with (count 1, checkSum(x), x) for fresh keys x that
    do NOT hash to c: count and checksum say "pure", but c is not one of x's cells (R28).
    Returns the forged cell ids."""
    import numpy as np
    count, ks, hs = cells
    rng = np.random.default_rng(rng_seed)
    empty = np.flatnonzero(count == 0)
    rng.shuffle(empty)
    forged = []
    for c in empty.tolist():
        if len(forged) == nforge:
            break
        while True:
            x = int(rng.integers(0, 2**63))
            if c not in key_cells(O, x, C, r, seed, mode, blog):
                break
        count[c] = 1
        ks[c] = np.uint64(x)
        hs[c] = np.uint32(O.checksum(x, seed))
        forged.append(c)
    return forged


def forge_sign_cycle(O, C, r, seed):
    """A signed table that cycles (R28): key x with cells a < b < d (r = 3);
    a = (+1, x), b = (-1, x), everything else empty.  Round 1 recovers (x, +1) from the
    owner a, which leaves d = (-1, x); round 2 recovers (x, -1) from d, which restores
    a = (+1, x), b = (-1, x); and so on, forever: the 65536-round limit truncates it."""
    import numpy as np
    x = 0x0123456789ABCDEF
    a, b, _d = sorted(key_cells(O, x, C, r, seed, "plain"))
    count = np.zeros(C, dtype=np.int64)
    ks = np.zeros(C, dtype=np.uint64)
    hs = np.zeros(C, dtype=np.uint32)
    h = O.checksum(x, seed)
    count[a], ks[a], hs[a] = 1, x, h
    count[b], ks[b], hs[b] = -1, x, h
    return x, (count, ks, hs)


def cells_to_dev_layout(cells):
    """(count, keySum, hashSum) -> [C, 4] int32 (count, hashSum, keySum_lo, keySum_hi), the
    device cell layout (Iblt.cells())."""
    import numpy as np
    count, ks, hs = cells
    C = count.size
    out = np.zeros((C, 4), dtype=np.uint32)
    out[:, 0] = (count.astype(np.int64) & 0xFFFFFFFF).astype(np.uint32)
    out[:, 1] = hs.astype(np.uint32)
    out[:, 2:4] = np.ascontiguousarray(ks, dtype=np.uint64).view(np.uint32).reshape(C, 2)
    return out.view(np.int32)
