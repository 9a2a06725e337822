"""GPU parity for the IBLT through the C-ABI against the oracle:
cell contents after insert/delete (bit-exact), sorted recovered key set,
rounds, per-round counts, completeness; the C2 config at full size."""
import hashlib

import numpy as np
import pytest
import torch

import paper_1302_7014_b200 as pk
import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")


def keys_dev(k: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(k, dtype=np.uint64).view(np.int64)).to(DEV)


def dev_cells(t: pk.Iblt):
    c = t.cells().cpu().numpy()
    count = c[:, 0].astype(np.int64)
    hashsum = c[:, 1].view(np.uint32)
    keysum = c[:, 2:4].copy().view(np.uint64).ravel()
    return count, keysum, hashsum


def compare(C, r, seed, keys, deletes=None):
    t = pk.Iblt(C, r, seed, device=DEV)
    o = O.Iblt(C, r, seed)
    t.insert(keys_dev(keys))
    o.insert(keys)
    if deletes is not None:
        t.delete(keys_dev(deletes))
        o.delete(deletes)
    cnt, ks, hs = dev_cells(t)
    ocnt, oks, ohs = o.cells()
    assert np.array_equal(cnt.astype(np.int32), ocnt.astype(np.int32))
    assert np.array_equal(ks, oks) and np.array_equal(hs, ohs)
    res = t.peel()
    ref = o.peel()
    got = np.sort(res.keys.cpu().numpy().view(np.uint64))
    assert res.nrecovered == ref.keys.size
    assert np.array_equal(got, np.sort(ref.keys))
    assert res.rounds == ref.rounds and res.per_round.tolist() == ref.per_round.tolist()
    assert res.complete == ref.complete
    # destructive: remaining cells equal the oracle's remainder
    cnt, ks, hs = dev_cells(t)
    ocnt, oks, ohs = o.cells()
    assert np.array_equal(cnt.astype(np.int32), ocnt.astype(np.int32)) and np.array_equal(ks, oks)
    return res, ref


def test_empty_and_single():
    compare(100, 3, 1, np.zeros(0, dtype=np.uint64))
    compare(100, 3, 1, np.array([0], dtype=np.uint64))            # the zero key is recoverable
    compare(100, 3, 1, np.array([12345], dtype=np.uint64))


@pytest.mark.parametrize("r", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("load", [0.3, 0.75, 0.83, 1.0, 1.3])
def test_random_tables(r, load):
    for C in (r, 37, 1000, 65537):
        N = int(load * C)
        keys = synth.random_keys(N, seed=C + r)
        compare(C, r, seed=C * 7 + r, keys=keys)


def test_insert_delete_sparse_recovery():
    # insert N items, delete all but n, recover the remaining set
    C, r = 40000, 3
    allk = synth.random_keys(200000, 4)
    keep = allk[:30000]
    res, ref = compare(C, r, 9, allk, deletes=allk[30000:])
    assert res.complete and np.array_equal(np.sort(res.keys.cpu().numpy().view(np.uint64)), np.sort(keep))


@pytest.mark.parametrize("r,load", [(3, 0.75), (3, 0.83), (4, 0.75), (4, 0.83)])
def test_paper_loads_2pow20(r, load):
    # Tables 3a/3b workload shape (2^24 cells; here 2^20 so the oracle stays fast)
    C = 1 << 20
    N = int(load * C)
    seed = 100 + r
    keys = pk.gen_keys(N, seed, device=DEV)
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), O.gen_keys(N, seed))
    compare(C, r, seed, O.gen_keys(N, seed))


def test_to_hypergraph_matches_oracle():
    C, r, seed = 5000, 4, 3
    keys = O.gen_keys(3000, 1)
    t = pk.Iblt(C, r, seed, device=DEV)
    o = O.Iblt(C, r, seed)
    got = t.to_hypergraph(keys_dev(keys)).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, o.to_hypergraph(keys))


def test_key_cap_truncation():
    C, r = 1000, 3
    keys = synth.random_keys(500, 1)
    t = pk.Iblt(C, r, 5, device=DEV)
    t.insert(keys_dev(keys))
    with pytest.raises(pk.PeelError) as ei:
        t.peel(cap_keys=100)
    assert ei.value.status == pk.PEEL_ETRUNC


def test_c2_full_config(oracle_goldens):
    """BASELINE.json configs[1]: 10^7 cells, 7.5e6 keys, r=3, seed=2."""
    g = oracle_goldens["C2"]
    keys = pk.gen_keys(g["nkeys"], g["seed"], device=DEV)
    t = pk.Iblt(g["cells"], g["r"], g["seed"], device=DEV)
    t.insert(keys)
    res = t.peel(cap_keys=g["nkeys"])
    assert res.rounds == g["rounds"] and res.per_round.tolist() == g["per_round"]
    assert res.complete
    got = np.sort(res.keys.cpu().numpy().view(np.uint64))
    assert hashlib.sha256(got.tobytes()).hexdigest() == g["sorted_keys_sha256"]


# ---- subtable IBLT: the paper's GPU schedule ------------------------------------
@pytest.mark.parametrize("r", [2, 3, 4, 5])
@pytest.mark.parametrize("load", [0.5, 0.75, 0.83, 1.1])
def test_subtable_recovery_vs_oracle(r, load):
    C = r * 30011
    N = int(load * C)
    keys = O.gen_keys(N, 60 + r)
    t = pk.Iblt(C, r, 9, device=DEV, subtables=True)
    o = O.Iblt(C, r, 9, subtables=True)
    t.insert(keys_dev(keys))
    o.insert(keys)
    cnt, ks, hs = dev_cells(t)
    ocnt, oks, ohs = o.cells()
    assert np.array_equal(cnt.astype(np.int32), ocnt.astype(np.int32)) and np.array_equal(ks, oks)
    res = t.peel()
    ref = o.peel_subtables()
    assert res.rounds == ref.rounds and res.per_round.tolist() == ref.per_round.tolist()
    assert np.array_equal(np.sort(res.keys.cpu().numpy().view(np.uint64)), np.sort(ref.keys))
    assert res.complete == ref.complete


def test_subtable_table3_shape():
    # Tables 3a/3b workload shape (2^24 cells in the paper; 2^21 here), r=3, load 0.75 and 0.83
    for load in (0.75, 0.83):
        C = 3 * (1 << 21)
        N = int(load * C)
        keys = pk.gen_keys(N, 3, device=DEV)
        t = pk.Iblt(C, 3, 3, device=DEV, subtables=True)
        t.insert(keys)
        res = t.peel(cap_keys=N)
        o = O.Iblt(C, 3, 3, subtables=True)
        o.insert(O.gen_keys(N, 3))
        ref = o.peel_subtables(cap_keys=N + 1)
        assert res.rounds == ref.rounds and res.nrecovered == ref.keys.size and res.complete == ref.complete


# ---- set difference -------------------------------------------------
@pytest.mark.parametrize("r", [3, 4])
@pytest.mark.parametrize("diff", [100, 9000, 16000])
def test_set_difference_vs_oracle(r, diff):
    C = 30011
    common = synth.random_keys(150000, 21)
    only_a = synth.random_keys(diff, 22)
    only_b = synth.random_keys(diff, 23)
    ka, kb = np.concatenate([common, only_a]), np.concatenate([only_b, common])
    ga, gb = pk.Iblt(C, r, 6, device=DEV), pk.Iblt(C, r, 6, device=DEV)
    oa, ob = O.Iblt(C, r, 6), O.Iblt(C, r, 6)
    ga.insert(keys_dev(ka)); gb.insert(keys_dev(kb))
    oa.insert(ka); ob.insert(kb)
    ga.subtract(gb)
    oa.subtract(ob)
    cnt, ks, hs = dev_cells(ga)
    ocnt, oks, ohs = oa.cells()
    assert np.array_equal(cnt.astype(np.int32), ocnt.astype(np.int32)) and np.array_equal(ks, oks)
    assert np.array_equal(hs, ohs)
    res, sg = ga.peel_signed()
    ref, osg = oa.peel_signed()
    assert res.rounds == ref.rounds and res.per_round.tolist() == ref.per_round.tolist()
    assert res.complete == ref.complete
    got = sorted(zip(res.keys.cpu().numpy().view(np.uint64).tolist(), sg.cpu().numpy().tolist()))
    exp = sorted(zip(ref.keys.tolist(), osg.tolist()))
    assert got == exp
    if res.complete:
        kk = res.keys.cpu().numpy().view(np.uint64)
        s_ = sg.cpu().numpy()
        assert np.array_equal(np.sort(kk[s_ == 1]), np.sort(only_a))
        assert np.array_equal(np.sort(kk[s_ == -1]), np.sort(only_b))


def test_signed_peel_on_insert_only_equals_plain():
    C, r = 100003, 3
    keys = O.gen_keys(75000, 7)
    a, b = pk.Iblt(C, r, 1, device=DEV), pk.Iblt(C, r, 1, device=DEV)
    a.insert(keys_dev(keys)); b.insert(keys_dev(keys))
    pa = a.peel()
    pb, sg = b.peel_signed()
    assert pa.rounds == pb.rounds and pa.per_round.tolist() == pb.per_round.tolist()
    assert bool((sg == 1).all())


# ---- blocked (locality-aware) hashing, R27 ---------------------------
@pytest.mark.parametrize("r", [2, 3, 4])
@pytest.mark.parametrize("blog,load", [(4, 0.5), (8, 0.75), (12, 0.8), (16, 0.83), (20, 0.75)])
def test_blocked_recovery_vs_oracle(r, blog, load):
    C = max(1 << 20, 1 << blog)
    N = int(load * C)
    keys = O.gen_keys(N, 70 + r + blog)
    t = pk.Iblt(C, r, 13, device=DEV, blog=blog)
    o = O.Iblt(C, r, 13, blog=blog)
    t.insert(keys_dev(keys))
    o.insert(keys)
    cnt, ks, hs = dev_cells(t)
    ocnt, oks, ohs = o.cells()
    assert np.array_equal(cnt.astype(np.int32), ocnt.astype(np.int32)) and np.array_equal(ks, oks)
    assert np.array_equal(hs, ohs)
    res = t.peel(cap_keys=N)
    ref = o.peel(cap_keys=N + 1)
    assert res.rounds == ref.rounds and res.per_round.tolist() == ref.per_round.tolist()
    assert res.complete == ref.complete
    assert np.array_equal(np.sort(res.keys.cpu().numpy().view(np.uint64)), np.sort(ref.keys))
    e = t.to_hypergraph(keys_dev(keys[:1000])).cpu().numpy().view(np.uint32)
    assert np.array_equal(e, o.to_hypergraph(keys[:1000]))


def test_blocked_rejects_bad_shapes():
    with pytest.raises(pk.PeelError):
        pk.Iblt(1000, 3, 1, device=DEV, blog=8)            # 2^8 does not divide 1000
    with pytest.raises(pk.PeelError):
        pk.Iblt(1 << 12, 3, 1, device=DEV, blog=8, subtables=True)


@pytest.mark.parametrize("mode", ["plain", "subtables", "blocked"])
def test_large_table_beyond_2pow31_cells(mode):
    """C = 9 * 2^28 (2.4e9 cells > 2^31, 38 GB of cells; iblt_mem_bytes ~ 125 GB): cell
    indices above the signed 32-bit range.  The oracle cannot hold this table, but the hash
    (cells_of*) is per key: every key's r predicted cells must carry exactly its multiplicity
    of counts, the whole table must hold r*N counts (so nothing landed elsewhere), and the
    recovery of N << C keys is complete and returns exactly the inserted set (a unique result)."""
    C, r, N, seed = 9 << 28, 3, 100_000, 77
    keys = synth.random_keys(N, seed=5)
    blog = 16 if mode == "blocked" else 0
    t = pk.Iblt(C, r, seed, device=DEV, subtables=(mode == "subtables"), blog=blog)
    t.insert(keys_dev(keys))
    if mode == "plain":
        pred = np.stack([O.cells_of(int(x), C, r, seed) for x in keys])
    elif mode == "subtables":
        pred = np.stack([O.cells_of_subtable(int(x), C, r, seed) for x in keys])
    else:
        pred = np.stack([O.cells_of_blocked(int(x), C, r, seed, blog) for x in keys])
    assert pred.max() >= (1 << 31)  # the test really reaches the upper half
    cells, mult = np.unique(pred.ravel(), return_counts=True)
    cnt = t.cells()[:, 0]
    got = cnt[torch.from_numpy(cells.astype(np.int64)).to(DEV)].cpu().numpy()
    assert np.array_equal(got, mult.astype(np.int32))
    assert int(cnt.sum(dtype=torch.int64).item()) == r * N
    res = t.peel(cap_keys=N + 1)
    assert res.complete and res.nrecovered == N
    assert np.array_equal(np.sort(res.keys.cpu().numpy().view(np.uint64)), np.sort(keys))
    del t, cnt
    torch.cuda.empty_cache()
