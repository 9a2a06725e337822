"""The C-ABI library loads and exports every entry point include/peel.h declares;
host-side argument validation and workspace queries (no GPU needed)."""
import ctypes
import os
import re

import pytest

import paper_1302_7014_b200 as pk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "peel.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"^typedef[^;]*;", "", src, flags=re.M | re.S)  # callback typedefs
    names = re.findall(r"^[A-Za-z_][\w \*]*?\b([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "while")))


def test_header_declares_the_north_star_entry_points():
    fns = header_functions()
    for f in ("peel_kcore", "iblt_build", "iblt_insert", "iblt_peel", "peel_gen_hypergraph"):
        assert f in fns


def test_library_exports_every_header_symbol():
    L = pk.lib()
    missing = [f for f in header_functions() if not hasattr(L, f)]
    assert not missing, missing


def test_abi_version_and_strerror():
    L = pk.lib()
    assert L.peel_abi_version() == 2
    for s in range(8):
        assert L.peel_strerror(s).decode().startswith("PEEL_")


def test_workspace_queries():
    L = pk.lib()
    n, m = 10**9, 750 * 10**6
    ws = L.peel_kcore_workspace_bytes(n, m, 3, 2, 0)
    # packed k=2 layout: 8n state + 2 x 8n (v, e) frontier entries (the compacted rounds' two
    # state buffers) + m/8 alive bits + stats, plus (n > 2^23) the binned build's 8-byte entry
    # buffer (r m entries + ~0.3% slack), the per-edge-bin frontier regions (r entries per edge,
    # whole edge bins of 2^22) and the 16-byte records of 64-vertex groups
    fe = 8 * 3 * (1 << 22) * ((m + (1 << 22) - 1) >> 22)
    assert 24 * n + 8 * 3 * m + fe + n // 4 < ws < 24 * n + 8 * 3 * m * 1.004 + fe + n // 4 + m // 8 + (16 << 20)
    small = L.peel_kcore_workspace_bytes(10**6, 750000, 3, 2, 0)   # no binning below 2^23
    assert 24 * 10**6 < small < 24 * 10**6 + (8 << 20)
    # CSR: deg + end offsets + 2 frontiers (4n each) + adj 4rm, plus the binned entries (n > 2^23)
    csr = L.peel_kcore_workspace_bytes(n, m, 3, 3, 0)
    assert 16 * n + 12 * 3 * m < csr < 16 * n + 12 * 3 * m * 1.004 + m // 8 + (16 << 20)
    assert L.peel_kcore_workspace_bytes(10, 10, 1, 2, 0) == 0  # r < 2
    assert L.peel_kcore_workspace_bytes(10, 10, 9, 2, 0) == 0  # r > 8
    assert L.peel_kcore_workspace_bytes(2**32 + 1, 10, 3, 2, 0) == 0
    assert L.iblt_mem_bytes(10**7, 3) >= 16 * 10**7
    assert L.iblt_mem_bytes(2, 3) == 0
    # cell-partitioned IBLT: per shard 16 B cells + 2 x 16 B frontier + 4 B list + 2 x 8 P B of
    # message buffers per owned cell; virtual shards hold all P shards
    for P in (1, 4, 8):
        c = pk.Comm.virtual_shards(P)
        b = L.iblt_dist_mem_bytes(c._h, 10**7, 3)
        assert (52 + 16 * P) * 10**7 <= b < (52 + 16 * P) * 10**7 * 1.01 + (8 << 20)
        assert L.iblt_dist_mem_bytes(c._h, 2, 3) == 0 and L.iblt_dist_mem_bytes(c._h, 10**7, 9) == 0


def test_invalid_arguments_rejected_before_any_launch():
    L = pk.lib()
    r = ctypes.c_uint32(0)
    # r = 1
    assert L.peel_kcore(None, 10, 0, 1, 2, 0, None, ctypes.addressof(r), None, None, 0, None, None, 0,
                        None) == pk.PEEL_EINVAL
    # null workspace
    assert L.peel_kcore(None, 10, 0, 3, 2, 0, 1, ctypes.addressof(r), None, None, 0, None, None, 0,
                        None) == pk.PEEL_EINVAL
    # workspace too small
    assert L.peel_kcore(None, 10, 0, 3, 2, 0, 1, ctypes.addressof(r), None, None, 0, None, 1, 16,
                        None) == pk.PEEL_ENOMEM
    assert L.peel_gen_hypergraph(2, 10, 3, 1, None, None) == pk.PEEL_EINVAL  # n < r
    h = ctypes.c_void_p(0)
    assert L.iblt_build(10, 1, 0, 16, 1 << 20, None, ctypes.byref(h)) == pk.PEEL_EINVAL
    assert L.iblt_build(100, 3, 0, 8, 1 << 20, None, ctypes.byref(h)) == pk.PEEL_EINVAL  # misaligned


def test_library_does_not_link_the_oracle():
    # the product library and the oracle share no code: no oracle symbol is exported
    L = pk.lib()
    for sym in ("ora_sync_peel", "ora_gen_edge", "ora_iblt_peel"):
        assert not hasattr(L, sym)
    import subprocess
    out = subprocess.run(["nm", "-D", pk.LIB_PATH], capture_output=True, text=True).stdout
    assert "ora_" not in out


def test_host_comm_validation():
    L = pk.lib()
    h = ctypes.c_void_p(0)
    null = pk._AR_FN()  # NULL function pointers
    assert L.peel_comm_init_host(2, 0, null, pk._AG_FN(), pk._A2A_FN(), None, ctypes.byref(h)) == pk.PEEL_EINVAL
    ok = pk._AR_FN(lambda c, v, n: 0), pk._AG_FN(lambda c, s, r, b: 0), pk._A2A_FN(lambda c, s, sb, r, rb: 0)
    assert L.peel_comm_init_host(2, 2, *ok, None, ctypes.byref(h)) == pk.PEEL_EINVAL  # rank >= nranks
    assert L.peel_comm_init_host(9, 0, *ok, None, ctypes.byref(h)) == pk.PEEL_EINVAL  # P > 8
    assert L.peel_comm_init_host(2, 1, *ok, None, ctypes.byref(h)) == pk.PEEL_OK
    assert L.iblt_dist_mem_bytes(h, 3 * 4096, 3) > 0
    L.peel_comm_destroy(h)
