"""GPU parity for the pure-cell reading R28: tables with
forged cells -- count and checksum say "pure" but the key does not hash to the cell -- and
the signed two-cell cycle, loaded byte-for-byte into the device table and into the oracle.
Both sides must terminate and agree bit-exactly (recovered keys and signs, rounds, per-round
counts, completeness, remaining cells), for plain, subtable, blocked and cell-partitioned
recovery."""
import numpy as np
import pytest
import torch

import paper_1302_7014_b200 as pk
import synth
from oracle import oracle as O
from peeltest_util import cells_to_dev_layout, forge_foreign_cells, forge_sign_cycle, honest_cells

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")

MODES = [("plain", 0), ("subtables", 0), ("blocked", 10)]


def dev_table(C, r, seed, mode, blog, cells):
    t = pk.Iblt(C, r, seed, device=DEV, subtables=(mode == "subtables"), blog=blog)
    t.load_cells(torch.from_numpy(cells_to_dev_layout(cells)).to(DEV))
    return t


def ora_table(C, r, seed, mode, blog, cells):
    o = O.Iblt(C, r, seed, subtables=(mode == "subtables"), blog=blog)
    o.load_cells(*cells)
    return o


def remaining(t):
    c = t.cells().cpu().numpy()
    return c[:, 0].astype(np.int64), c[:, 2:4].copy().view(np.uint64).ravel(), c[:, 1].view(np.uint32)


@pytest.mark.parametrize("mode,blog", MODES)
@pytest.mark.parametrize("r", [3, 4])
def test_foreign_cells(mode, blog, r):
    C, seed = 4096 * r, 31 + r
    keys = synth.random_keys(int(0.6 * C), 200 + r)  # below the blocked threshold at 2^10 cells too
    cells = honest_cells(O, keys, C, r, seed, mode, blog)
    forged = forge_foreign_cells(O, cells, C, r, seed, mode, 40, 9, blog)
    t = dev_table(C, r, seed, mode, blog, cells)
    o = ora_table(C, r, seed, mode, blog, cells)
    res = t.peel()
    ref = o.peel_subtables() if mode == "subtables" else o.peel()
    got = np.sort(res.keys.cpu().numpy().view(np.uint64))
    assert np.array_equal(got, np.sort(ref.keys)) and np.array_equal(got, np.sort(keys))
    assert res.rounds == ref.rounds and res.per_round.tolist() == ref.per_round.tolist()
    assert res.complete == ref.complete is False
    rc, rk, rh = remaining(t)
    oc, ok_, oh = o.cells()
    assert np.array_equal(rc.astype(np.int32), oc.astype(np.int32)) and np.array_equal(rk, ok_)
    assert np.array_equal(rh, oh)
    assert np.flatnonzero(oc).tolist() == sorted(forged)


def test_foreign_cells_signed():
    C, r, seed = 8192, 3, 41
    a = synth.random_keys(2000, 11)
    b = np.concatenate([a[:1200], synth.random_keys(700, 12)])
    ca = honest_cells(O, a, C, r, seed, "plain")
    cb = honest_cells(O, b, C, r, seed, "plain")
    diff = (ca[0] - cb[0], ca[1] ^ cb[1], ca[2] ^ cb[2])
    forge_foreign_cells(O, diff, C, r, seed, "plain", 25, 13)
    t = dev_table(C, r, seed, "plain", 0, diff)
    o = ora_table(C, r, seed, "plain", 0, diff)
    res, sg = t.peel_signed()
    ref, rsg = o.peel_signed()
    got = dict(zip(res.keys.cpu().numpy().view(np.uint64).tolist(), sg.cpu().numpy().tolist()))
    want = dict(zip(ref.keys.tolist(), rsg.tolist()))
    assert got == want and len(got) == 1500
    assert res.rounds == ref.rounds and res.per_round.tolist() == ref.per_round.tolist()
    assert res.complete == ref.complete is False


def test_sign_cycle_truncates_identically():
    C, r, seed = 64, 3, 8
    x, cells = forge_sign_cycle(O, C, r, seed)
    t = dev_table(C, r, seed, "plain", 0, cells)
    o = ora_table(C, r, seed, "plain", 0, cells)
    res, sg = t.peel_signed(cap_keys=70000, cap=65536, allow_trunc=True)
    ref, rsg = o.peel_signed(cap_keys=70000, cap=65536, allow_trunc=True)
    assert res.status == pk.PEEL_ETRUNC and ref.truncated
    assert res.rounds == ref.rounds == 65536
    assert res.per_round.tolist() == ref.per_round.tolist()
    # one key per round: the order within a round is unique, so the sequences must match
    assert res.keys.cpu().numpy().view(np.uint64).tolist() == ref.keys.tolist()
    assert sg.cpu().numpy().tolist() == rsg.tolist()


@pytest.mark.parametrize("P", [1, 2, 3])
@pytest.mark.parametrize("blog", [0, 8])
def test_foreign_cells_partitioned_virtual(P, blog):
    C, r, seed = 3 * 4096, 3, 51
    keys = synth.random_keys(8000, 21)
    mode = "blocked" if blog else "plain"
    cells = honest_cells(O, keys, C, r, seed, mode, blog)
    forge_foreign_cells(O, cells, C, r, seed, mode, 30, 17, blog)
    o = ora_table(C, r, seed, mode, blog, cells)
    ref = o.peel()
    dev = torch.from_numpy(cells_to_dev_layout(cells)).to(DEV)
    res = pk.iblt_dist_recover_cells(pk.Comm.virtual_shards(P), dev, r, seed, blog=blog)
    got = np.sort(res.keys.cpu().numpy().view(np.uint64))
    assert np.array_equal(got, np.sort(ref.keys))
    assert res.rounds == ref.rounds and res.per_round.tolist() == ref.per_round.tolist()
    assert res.complete == ref.complete is False
