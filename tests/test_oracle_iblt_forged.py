"""Pins for the pure-cell reading R28 ("cells that only contain one
item"): pure <=> count = +-1, hashSum = checkSum(keySum) AND the cell is one of
keySum's own cells.  A cell holding one item x is necessarily one of x's cells, so a cell
failing the last test holds several items whatever its count and checksum say.

Pinned against what the definition fixes, not against the oracle itself:
  * a forged foreign cell (count 1, matching checksum, key not hashing there) is never
    recovered, recovery terminates, every inserted key is recovered, and the forged cell is
    the only non-zero cell left -- for plain, subtable and blocked hashing, round-
    synchronous and serial recovery;
  * a signed table recovers a key found in two pure cells once per round, with the sign of
    the lower cell; the hand-traced two-round cycle of forge_sign_cycle is reproduced and
    truncated at the round limit."""
import numpy as np
import pytest

import synth
from oracle import oracle as O
from peeltest_util import forge_foreign_cells, forge_sign_cycle, honest_cells

MODES = [("plain", 0), ("subtables", 0), ("blocked", 8)]


def _table(C, r, seed, mode, blog):
    return O.Iblt(C, r, seed, subtables=(mode == "subtables"), blog=blog)


@pytest.mark.parametrize("mode,blog", MODES)
@pytest.mark.parametrize("r", [3, 4])
def test_foreign_cells_never_pure(mode, blog, r):
    C = 2048 * r  # divisible by r (subtables) and by 2^blog (blocked)
    seed = 11 + r
    keys = synth.random_keys(int(0.6 * C), 100 + r)
    cells = honest_cells(O, keys, C, r, seed, mode, blog)
    forged = forge_foreign_cells(O, cells, C, r, seed, mode, 20, 7, blog)
    assert len(forged) == 20
    t = _table(C, r, seed, mode, blog)
    t.load_cells(*cells)
    res = t.peel_subtables() if mode == "subtables" else t.peel()
    # every inserted key recovered, nothing else; the forged cells untouched and the only
    # non-zero cells left (recovery never deletes a forged "key")
    assert sorted(res.keys.tolist()) == sorted(keys.tolist())
    assert not res.complete
    c, k, h = t.cells()
    nz = np.flatnonzero((c != 0) | (k != 0) | (h != 0)).tolist()
    assert nz == sorted(forged)
    assert (c[forged] == 1).all()


@pytest.mark.parametrize("mode,blog", MODES)
def test_foreign_cells_serial(mode, blog):
    C, r, seed = 3 * 1024, 3, 5
    keys = synth.random_keys(1500, 9)
    cells = honest_cells(O, keys, C, r, seed, mode, blog)
    forged = forge_foreign_cells(O, cells, C, r, seed, mode, 10, 3, blog)
    t = _table(C, r, seed, mode, blog)
    t.load_cells(*cells)
    got, complete = t.serial_recover()
    assert sorted(got.tolist()) == sorted(keys.tolist()) and not complete


def test_foreign_cells_signed():
    # A \ B and B \ A plus forged cells: the signed recovery returns exactly the two
    # differences, with their signs, and stops
    C, r, seed = 4096, 3, 21
    a = synth.random_keys(900, 1)
    b = np.concatenate([a[:600], synth.random_keys(300, 2)])
    ca = honest_cells(O, a, C, r, seed, "plain")
    cb = honest_cells(O, b, C, r, seed, "plain")
    diff = (ca[0] - cb[0], ca[1] ^ cb[1], ca[2] ^ cb[2])
    forged = forge_foreign_cells(O, diff, C, r, seed, "plain", 12, 4)
    t = O.Iblt(C, r, seed)
    t.load_cells(*diff)
    res, sg = t.peel_signed()
    got = dict(zip(res.keys.tolist(), sg.tolist()))
    want = {x: 1 for x in a[600:].tolist()}
    want.update({x: -1 for x in b[600:].tolist()})
    assert got == want and not res.complete
    c, _, _ = t.cells()
    assert np.flatnonzero(c).tolist() == sorted(forged)


def test_sign_cycle_owner_rule_and_limit():
    C, r, seed = 64, 3, 8
    x, cells = forge_sign_cycle(O, C, r, seed)
    t = O.Iblt(C, r, seed)
    t.load_cells(*cells)
    res, sg = t.peel_signed(cap_keys=70000, cap=65536, allow_trunc=True)
    # hand trace (peeltest_util.forge_sign_cycle): one key per round, signs +1, -1, +1, ...
    assert res.truncated and res.rounds == 65536
    assert (res.per_round == 1).all() and res.per_round.size == 65536
    assert (res.keys == np.uint64(x)).all() and res.keys.size == 65536
    assert sg[0::2].tolist() == [1] * 32768 and sg[1::2].tolist() == [-1] * 32768
