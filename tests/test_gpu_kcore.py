"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs -- bit-exact core mask, rounds, every survivors[t] and
killed[t] -- plus full-scale configs against goldens and the local schedule
certificate (properties that hold at any size)."""
import hashlib

import numpy as np
import pytest
import torch

import paper_1302_7014_b200 as pk
import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")


def to_dev(e: np.ndarray) -> torch.Tensor:
    e = np.ascontiguousarray(e, dtype=np.uint32)
    return torch.from_numpy(e.view(np.int32)).to(DEV)


def check_vs_oracle(e_np, n, k, flags=0, twice=True):
    m, r = e_np.shape if e_np.size else (0, e_np.shape[1])
    ref = O.sync_peel(e_np, n, k, want_peel_round=True)
    ed = to_dev(e_np) if m else torch.zeros((0, r), dtype=torch.int32, device=DEV)
    for _ in range(2 if twice else 1):  # twice: expose nondeterminism
        res = pk.peel_kcore(ed, n, k, flags=flags, want_peel_round=True)
        assert res.rounds == ref.rounds, (res.rounds, ref.rounds)
        assert res.survivors.tolist() == ref.survivors.tolist()
        assert res.killed.tolist() == ref.killed.tolist()
        assert np.array_equal(res.core_mask.cpu().numpy(), ref.core_mask)
        assert np.array_equal(res.peel_round.cpu().numpy().view(np.uint32), ref.peel_round)
    return ref


# ---- generator (a1) ---------------------------------------------------------------------
@pytest.mark.parametrize("n,m,r,seed", [(100000, 70000, 3, 1), (1000, 12345, 4, 9), (7, 1001, 7, 3),
                                        (5, 333, 5, 2), (2**32, 5000, 3, 11), (3, 10, 3, 4),
                                        (1000003, 99999, 8, 5), (50, 1, 2, 0)])
def test_generator_matches_oracle(n, m, r, seed):
    got = pk.gen_hypergraph(n, m, r, seed, device=DEV).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, O.gen_hypergraph(n, m, r, seed))


def test_generator_c1_digest(oracle_goldens):
    g = oracle_goldens["C1"]
    got = pk.gen_hypergraph(g["n"], g["m"], g["r"], g["seed"], device=DEV).cpu().numpy().view(np.uint32)
    assert hashlib.sha256(got.tobytes()).hexdigest() == g["sha256"]


def test_generator_sampled_at_full_scale(oracle_goldens):
    # C5 (n=10^9, m=7.5e8): the oracle computes any edge on its own; compare 2000 sampled edges
    g = oracle_goldens["C5"]
    e = pk.gen_hypergraph(g["n"], g["m"], g["r"], g["seed"], device=DEV)
    rng = np.random.default_rng(0)
    idx = np.concatenate([[0, 1, g["m"] - 1], rng.integers(0, g["m"], 2000)])
    got = e[torch.from_numpy(idx).to(DEV)].cpu().numpy().view(np.uint32)
    for row, i in zip(got, idx):
        assert row.tolist() == O.gen_edge(g["seed"], g["n"], g["r"], int(i)).tolist()
    del e


def test_keys_match_oracle():
    got = pk.gen_keys(100001, 77, device=DEV).cpu().numpy().view(np.uint64)
    assert np.array_equal(got, O.gen_keys(100001, 77))


# ---- k-core parity (a2-a7) ----------------------------------------------------------------
def test_spec_examples():
    check_vs_oracle(np.array([[0, 1, 2]], dtype=np.uint32), 3, 2)
    check_vs_oracle(np.array([[0, 1, 2], [0, 1, 3], [0, 1, 4], [2, 3, 4]], dtype=np.uint32), 6, 2)
    check_vs_oracle(np.array([[0, 1, 2], [2, 3, 4], [4, 5, 6]], dtype=np.uint32), 7, 2)


@pytest.mark.parametrize("flags", [0, pk.PEEL_FLAG_CSR])
def test_degenerate_cases(flags):
    check_vs_oracle(np.zeros((0, 3), dtype=np.uint32), 10, 2, flags)        # no edges
    check_vs_oracle(np.zeros((0, 3), dtype=np.uint32), 1, 1, flags)
    check_vs_oracle(np.array([[0, 1, 2]], dtype=np.uint32), 3, 0, flags)    # k = 0: nothing peels
    check_vs_oracle(np.array([[0, 1, 2], [0, 1, 2]], dtype=np.uint32), 3, 2, flags)  # duplicate edge = core
    e, n = synth.chain(301, 2)
    check_vs_oracle(e, n, 2, flags)                                          # 151 rounds
    check_vs_oracle(synth.star(1001, 3), 1001, 2, flags)
    check_vs_oracle(synth.complete_r_graph(9, 3), 9, 3, flags)              # non-empty 3-core


def test_empty_vertex_set():
    res = pk.peel_kcore(torch.zeros((0, 3), dtype=torch.int32, device=DEV), 0, 2)
    assert res.rounds == 0


@pytest.mark.parametrize("r", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_random_small_vs_oracle(r, k):
    rng = np.random.default_rng(10 * r + k)
    for trial in range(6):
        n = int(rng.integers(r, 3000))
        m = int(rng.integers(0, 2 * n))
        e = synth.random_hypergraph(n, m, r, seed=trial)
        if trial % 2 and m:
            e = np.concatenate([e, e[: max(1, m // 50)]])  # duplicated edges
        check_vs_oracle(e, n, k, twice=False)
        if k <= 2:
            check_vs_oracle(e, n, k, flags=pk.PEEL_FLAG_CSR, twice=False)


@pytest.mark.parametrize("r,k,c", [(3, 2, 0.70), (3, 2, 0.818), (3, 2, 0.85), (4, 2, 0.75), (4, 2, 0.8),
                                   (3, 3, 1.6), (3, 3, 1.5), (5, 2, 0.7), (4, 3, 1.3)])
def test_paper_shaped_vs_oracle(r, k, c):
    # several tiles and a ragged tail: n not a multiple of 32 / 256 / 2048
    n = 200003
    m = int(c * n)
    seed = int(1000 * c) + 10 * r + k
    e = pk.gen_hypergraph(n, m, r, seed, device=DEV)
    e_np = O.gen_hypergraph(n, m, r, seed)
    assert np.array_equal(e.cpu().numpy().view(np.uint32), e_np)
    check_vs_oracle(e_np, n, k)
    if k == 2:
        check_vs_oracle(e_np, n, k, flags=pk.PEEL_FLAG_CSR, twice=False)


@pytest.mark.parametrize("n,c,r,seed", [((1 << 23) + 12345, 0.75, 3, 21), ((1 << 23) + 1, 0.85, 3, 22),
                                        (3 * (1 << 22) - 7, 0.8, 4, 23)])
def test_binned_build_vs_oracle(n, c, r, seed):
    # n > 2^23: the build partitions increments into 2^22-vertex bins (several bins + ragged last)
    m = int(c * n)
    e = pk.gen_hypergraph(n, m, r, seed, device=DEV)
    e_np = e.cpu().numpy().view(np.uint32)
    ref = O.sync_peel(e_np, n, 2, want_peel_round=True)
    res = pk.peel_kcore(e, n, 2, want_peel_round=True)
    assert res.rounds == ref.rounds and res.survivors.tolist() == ref.survivors.tolist()
    assert res.killed.tolist() == ref.killed.tolist()
    assert np.array_equal(res.core_mask.cpu().numpy(), ref.core_mask)
    assert np.array_equal(res.peel_round.cpu().numpy().view(np.uint32), ref.peel_round)


def test_binned_build_overflow_fallback():
    # every edge contains vertex 0: bin 0 overflows its capacity -> direct-build fallback
    n, m = (1 << 23) + 999, 600000
    rng = np.random.default_rng(5)
    e_np = np.zeros((m, 3), dtype=np.uint32)
    e_np[:, 1] = rng.integers(1, n // 2, m)
    e_np[:, 2] = e_np[:, 1] + n // 2 - 1
    e_np[m // 2:, 0] = 5  # a second hub
    check_vs_oracle(e_np, n, 2, twice=False)


def test_csr_binned_high_degree():
    # k = 3 (CSR) with n > 2^23 (binned CSR build): random edges, then the same with hubs of
    # degree ~1023-1025 (a 10-bit rank field's edge) and ~3000 added
    n, m = (1 << 23) + 4321, 9000000
    e_np = pk.gen_hypergraph(n, m, 3, 31, device=DEV).cpu().numpy().view(np.uint32).copy()
    check_vs_oracle(e_np, n, 3, twice=False)
    row = 0
    for hub, extra in ((7, 3000), (5000003, 1025), (6000011, 1023)):
        e_np[row:row + extra, 0] = hub
        row += extra
    bad = (e_np[:, 1] == e_np[:, 0]) | (e_np[:, 2] == e_np[:, 0])
    e_np[bad, 0] = 1  # keep the r vertices distinct
    e_np[bad & ((e_np[:, 1] == 1) | (e_np[:, 2] == 1)), 0] = 2
    assert np.all((e_np[:, 0] != e_np[:, 1]) & (e_np[:, 0] != e_np[:, 2]) & (e_np[:, 1] != e_np[:, 2]))
    check_vs_oracle(e_np, n, 3, twice=False)


def test_c1_golden_and_oracle(oracle_goldens):
    g = oracle_goldens["C1"]
    e = pk.gen_hypergraph(g["n"], g["m"], g["r"], g["seed"], device=DEV)
    res = pk.peel_kcore(e, g["n"], g["k"])
    assert res.rounds == g["rounds"] and res.survivors.tolist() == g["survivors"]
    assert res.killed.tolist() == g["killed"]
    check_vs_oracle(e.cpu().numpy().view(np.uint32), g["n"], g["k"])


@pytest.mark.parametrize("name", ["C4a_small", "C4b_small"])
def test_reduced_c4_vs_oracle(oracle_goldens, name):
    g = oracle_goldens[name]
    e = pk.gen_hypergraph(g["n"], g["m"], g["r"], g["seed"], device=DEV)
    e_np = e.cpu().numpy().view(np.uint32)
    assert hashlib.sha256(e_np.tobytes()).hexdigest() == g["sha256"]
    ref = check_vs_oracle(e_np, g["n"], g["k"], twice=False)
    assert ref.rounds == g["rounds"] and int(ref.core_mask.sum()) == g["core"]


def test_invalid_vertex_rejected():
    e = to_dev(np.array([[0, 1, 2], [3, 4, 10]], dtype=np.uint32))
    with pytest.raises(pk.PeelError) as ei:
        pk.peel_kcore(e, 10, 2)
    assert ei.value.status == pk.PEEL_EINVAL
    e = to_dev(np.array([[0, 1, 1]], dtype=np.uint32))
    with pytest.raises(pk.PeelError):
        pk.peel_kcore(e, 10, 2, flags=pk.PEEL_FLAG_CSR)


def test_round_cap_truncation():
    e, n = synth.chain(101, 2)
    ref = O.sync_peel(e, n, 2)
    res = pk.peel_kcore(to_dev(e), n, 2, cap=10, allow_trunc=True)
    assert res.status == pk.PEEL_ETRUNC and res.rounds == ref.rounds
    assert res.survivors.tolist() == ref.survivors[:10].tolist()


@pytest.mark.parametrize("n,m,r,k,pin", [(50021, 40000, 3, 2, True), ((1 << 23) + 4099, 6300000, 3, 2, True),
                                         ((1 << 23) + 4099, 7560000, 3, 2, True),  # c = 0.9: a core to copy back
                                         ((1 << 23) + 4099, 6300000, 3, 2, False), ((1 << 23) + 17, 9000000, 3, 3, True),
                                         (3000, 17, 4, 2, True)])
def test_host_buffer_entry_point(n, m, r, k, pin):
    # peel_kcore_host copies the edges in 16 chunks on its own stream; n > 2^23 (binned build)
    # partitions each chunk as it lands, and the mask comes back by chunks holding a core vertex
    # (the rest zeroed on the host); k = 3 (CSR) and small n wait for the whole copy
    e_np = O.gen_hypergraph(n, m, r, 5)
    ref = O.sync_peel(e_np, n, k)
    host = torch.from_numpy(e_np.view(np.int32))
    host = host.pin_memory() if pin else host
    for _ in range(2):
        res = pk.peel_kcore_host(host, n, k)
        assert res.rounds == ref.rounds and np.array_equal(res.core_mask, ref.core_mask)
        assert res.survivors.tolist() == ref.survivors.tolist() and res.killed.tolist() == ref.killed.tolist()


# ---- full-scale configs (BASELINE.json), checked against goldens + certificate -----------
def schedule_certificate_torch(edges: torch.Tensor, n: int, k: int, peel_round: torch.Tensor):
    """The local certificate of tests/test_oracle_peel.py, in torch on the device: with
    p(v) the removal round (inf = core) and d(e) = min p over e, deg_t(v) = #{e ni v: d(e) >= t};
    removed v: deg_{p(v)}(v) < k and deg_{p(v)-1}(v) >= k (p >= 2); core v: deg_inf(v) >= k."""
    INF = 1 << 40
    p = peel_round.to(torch.int64)
    p = torch.where(p == 0, torch.full_like(p, INF), p)
    el = edges.to(torch.int64)
    d = p[el].min(dim=1).values
    removed = p != INF

    def deg_at(tv):
        ok = d[:, None] >= tv[el]
        return torch.bincount(el[ok], minlength=n)

    tr = torch.where(removed, p, torch.ones_like(p))
    assert bool((deg_at(tr)[removed] < k).all())
    tp = torch.where(removed, torch.clamp(p - 1, min=1), torch.ones_like(p))
    late = removed & (p >= 2)
    assert bool((deg_at(tp)[late] >= k).all())
    core = ~removed
    tc = torch.where(core, torch.full_like(p, INF), torch.ones_like(p))
    assert bool((deg_at(tc)[core] >= k).all())


@pytest.mark.parametrize("name", ["C3", "C4a", "C4b"])
def test_full_scale_1e8_goldens_and_certificate(oracle_goldens, name):
    g = oracle_goldens[name]
    e = pk.gen_hypergraph(g["n"], g["m"], g["r"], g["seed"], device=DEV)
    assert e[0].cpu().numpy().view(np.uint32).tolist() == g["edges_head"][0]
    res = pk.peel_kcore(e, g["n"], g["k"], want_peel_round=True)
    assert res.rounds == g["rounds"]
    assert int(res.core_mask.sum().item()) == g["core"]
    if "survivors" in g:
        assert res.survivors.tolist() == g["survivors"] and res.killed.tolist() == g["killed"]
    else:
        assert res.survivors[:len(g["survivors_head"])].tolist() == g["survivors_head"]
        assert res.killed[:len(g["killed_head"])].tolist() == g["killed_head"]
        if "killed_tail" in g:
            assert res.killed[-len(g["killed_tail"]):].tolist() == g["killed_tail"]
    # survivors[t] == n - #{v : peel_round(v) <= t}
    hist = torch.bincount(res.peel_round.to(torch.int64), minlength=res.rounds + 1).cpu().numpy()
    assert np.array_equal(g["n"] - np.cumsum(hist[1:]), res.survivors)
    schedule_certificate_torch(e, g["n"], g["k"], res.peel_round)
    # packed and CSR paths agree at full scale (k=2)
    if g["k"] == 2:
        res2 = pk.peel_kcore(e, g["n"], g["k"], flags=pk.PEEL_FLAG_CSR)
        assert res2.rounds == res.rounds and res2.survivors.tolist() == res.survivors.tolist()
        assert torch.equal(res2.core_mask, res.core_mask)
    del e, res
    pk._ws_cache.clear()
    torch.cuda.empty_cache()


def test_full_scale_c5_north_star(oracle_goldens):
    """n = 10^9, m = 7.5e8, r=3, k=2 (the bench workload): goldens + certificate pieces."""
    g = oracle_goldens["C5"]
    e = pk.gen_hypergraph(g["n"], g["m"], g["r"], g["seed"], device=DEV)
    res = pk.peel_kcore(e, g["n"], g["k"])
    assert res.rounds == g["rounds"]
    assert res.survivors.tolist() == g["survivors"]
    assert res.killed.tolist() == g["killed"]
    assert int(res.core_mask.sum().item()) == 0
    del e, res
    pk._ws_cache.clear()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("path", ["cluster", "cooperative"])
def test_small_instances_both_round_loops(path, monkeypatch):
    """Small packed instances run in one thread-block cluster's shared memory
    (peel_cluster_kernel) unless PEEL_CLUSTER=0 selects the cooperative grid kernel:
    both bit-exact against the oracle, including C1 and ragged / degenerate shapes."""
    if path == "cooperative":
        monkeypatch.setenv("PEEL_CLUSTER", "0")
    else:
        monkeypatch.delenv("PEEL_CLUSTER", raising=False)
    rng = np.random.default_rng(77)
    for trial in range(12):
        r = int(rng.integers(2, 6))
        n = int(rng.integers(r, 140000)) if trial % 3 == 0 else int(rng.integers(r, 5000))
        m = int(rng.integers(0, int(0.95 * n)))
        e = synth.random_hypergraph(n, m, r, seed=500 + trial)
        check_vs_oracle(e, n, 2, twice=False)
    check_vs_oracle(synth.star(4001, 3), 4001, 2, twice=False)
    check_vs_oracle(synth.star(4001, 3), 4001, 1, twice=False)
    e, n = synth.chain(3001, 2)
    check_vs_oracle(e, n, 2, twice=False)
    e = pk.gen_hypergraph(100000, 70000, 3, 1, device=DEV)
    check_vs_oracle(e.cpu().numpy().view(np.uint32), 100000, 2, twice=False)


@pytest.mark.parametrize("r,c", [(2, 0.45), (5, 0.62), (8, 0.3), (4, 0.8)])
def test_binned_rounds_all_r_vs_oracle(r, c):
    # n > 2^23: binned build, frontier edge sort, binned kill/apply rounds, then the
    # persistent kernel -- for r other than 3 (row loads of 8 B and 16 B windows, R-wide rows)
    n = (1 << 23) + 4097
    m = int(c * n)
    e = pk.gen_hypergraph(n, m, r, 60 + r, device=DEV)
    e_np = e.cpu().numpy().view(np.uint32)
    ref = O.sync_peel(e_np, n, 2, want_peel_round=True)
    res = pk.peel_kcore(e, n, 2, want_peel_round=True)
    assert res.rounds == ref.rounds and res.survivors.tolist() == ref.survivors.tolist()
    assert res.killed.tolist() == ref.killed.tolist()
    assert np.array_equal(res.core_mask.cpu().numpy(), ref.core_mask)
    assert np.array_equal(res.peel_round.cpu().numpy().view(np.uint32), ref.peel_round)


def test_small_graph_replay_follows_buffer_contents(monkeypatch):
    """The small-instance path replays a captured CUDA graph keyed by buffers and shape: new
    contents in the same buffers must give the new results; PEEL_GRAPH=0 gives the same."""
    n, m, r = 30011, 21000, 3
    ws = torch.empty((pk.kcore_workspace_bytes(n, m, r, 2),), dtype=torch.uint8, device=DEV)
    mask = torch.empty((n,), dtype=torch.uint8, device=DEV)
    e = torch.empty((m, r), dtype=torch.int32, device=DEV)
    for seed in (1, 2, 3):
        e_np = O.gen_hypergraph(n, m, r, seed)
        e.copy_(torch.from_numpy(e_np.view(np.int32)))
        ref = O.sync_peel(e_np, n, 2)
        for graph in ("1", "0"):
            monkeypatch.setenv("PEEL_GRAPH", graph)
            res = pk.peel_kcore(e, n, 2, core_mask=mask, ws=ws)
            assert res.rounds == ref.rounds and res.survivors.tolist() == ref.survivors.tolist()
            assert res.killed.tolist() == ref.killed.tolist()
            assert np.array_equal(mask.cpu().numpy(), ref.core_mask)


@pytest.mark.parametrize("k,flags,c", [(2, 0, 0.7), (2, 0, 0.9), (2, "csr", 0.9), (3, 0, 1.6)])
def test_maximum_vertex_range(k, flags, c):
    """n = 2^32 (the largest vertex range peel.h allows): a compact random hypergraph on n0
    vertices, relabelled injectively into [0, 2^32) so that ids 0, 2^32-1 and ids either side
    of 2^22-vertex bin boundaries occur.  Peeling is label-invariant, so the oracle runs on
    the compact graph; the 2^32 - n0 isolated vertices all leave in round 1 on the GPU, so
    rounds, survivors[t] and killed[t] must agree exactly, and the core mask must be the
    oracle's at the mapped ids and empty elsewhere."""
    flags = pk.PEEL_FLAG_CSR if flags == "csr" else 0
    n0, r, N = 100_000, 3, 1 << 32
    rng = np.random.default_rng(7 + k)
    fixed = np.array([0, N - 1, N - 2, 1 << 22, (1 << 22) - 1, (1 << 31), (1 << 31) - 1, N - (1 << 22)],
                     dtype=np.uint64)
    rest = np.setdiff1d(np.unique(rng.integers(0, N, size=2 * n0, dtype=np.uint64)), fixed)
    ids = rng.permutation(np.concatenate([fixed, rng.permutation(rest)[: n0 - fixed.size]]))
    assert np.unique(ids).size == n0
    e0 = O.gen_hypergraph(n0, int(c * n0), r, 40 + k)
    ref = O.sync_peel(e0, n0, k)
    mask = torch.empty((N,), dtype=torch.uint8, device=DEV)
    res = pk.peel_kcore(to_dev(ids[e0.astype(np.int64)].astype(np.uint32)), N, k, flags=flags, core_mask=mask)
    assert res.rounds == ref.rounds
    assert res.survivors.tolist() == ref.survivors.tolist()
    assert res.killed.tolist() == ref.killed.tolist()
    got = mask[torch.from_numpy(ids.astype(np.int64)).to(DEV)].cpu().numpy()
    assert np.array_equal(got, ref.core_mask)
    assert int(mask.sum(dtype=torch.int64).item()) == int(ref.core_mask.sum())
    del mask, res
    pk._ws_cache.clear()
    torch.cuda.empty_cache()


# ---- slot-compacted rounds (kcompact.cuh; n > 2^23, k <= 2) --------------------------------
@pytest.mark.parametrize("tail,at,creg", [("0", None, None), ("2", None, None), (None, None, None),
                                          ("2", "1.0", None), ("2", "1.0", "0"), ("2", "0", None)])
@pytest.mark.parametrize("c,k,r", [(0.85, 2, 3), (0.75, 2, 3), (0.6, 1, 3), (0.77, 2, 4)])
def test_compact_rounds_modes(monkeypatch, tail, at, creg, c, k, r):
    """The binned rounds with edge-bin frontier regions and slot compaction: handing over to
    the persistent kernel at the first small frontier (tail 0), never (tail 2), or by the
    default rule; compacting whenever the live set shrank at all (at 1.0), never (at 0), or at
    the default halving -- and the uncompacted binned rounds (PEEL_COMPACT=0) on the same input,
    all bit-exact against the oracle."""
    n = (1 << 23) + 3 * 4097 + 5
    m = int(c * n)
    e = pk.gen_hypergraph(n, m, r, 70 + r, device=DEV)
    ref = O.sync_peel(e.cpu().numpy().view(np.uint32), n, k, want_peel_round=True)
    ratio = "0" if tail == "0" else None  # tail 0: hand over at the first small frontier
    for name, val in (("PEEL_COMPACT_TAIL", tail), ("PEEL_COMPACT_AT", at), ("PEEL_COMPACT_TAIL_RATIO", ratio),
                      ("PEEL_CREG", creg)):
        if val is None:
            monkeypatch.delenv(name, raising=False)
        else:
            monkeypatch.setenv(name, val)
    for compact in ("1", "0") if (tail, at, creg) == (None, None, None) else ("1",):
        monkeypatch.setenv("PEEL_COMPACT", compact)
        res = pk.peel_kcore(e, n, k, want_peel_round=True)
        assert res.rounds == ref.rounds and res.survivors.tolist() == ref.survivors.tolist(), compact
        assert res.killed.tolist() == ref.killed.tolist()
        assert np.array_equal(res.core_mask.cpu().numpy(), ref.core_mask)
        assert np.array_equal(res.peel_round.cpu().numpy().view(np.uint32), ref.peel_round)
