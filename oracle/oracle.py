"""CPU oracle binding (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module.  The product package
``paper_1302_7014_b200`` never imports it, and this module imports nothing from
the product package.

Thin ctypes marshalling over ``peel_oracle.c`` (plain single-threaded C, built
with gcc); every function cites the paper passage it follows in that file.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "peel_oracle.c")
_LIB = os.path.join(_HERE, "_build", "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no vectorisation pragmas)."""
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            u32, u64, i32, p = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
            L.ora_philox4x32_10.argtypes = [p, p, p]
            L.ora_gen_edge.argtypes = [u64, u64, u32, u64, p]
            L.ora_gen_edge.restype = i32
            L.ora_gen_hypergraph.argtypes = [u64, u64, u64, u32, p]
            L.ora_gen_hypergraph.restype = i32
            L.ora_mix64.argtypes = [u64]
            L.ora_mix64.restype = u64
            L.ora_gen_keys.argtypes = [u64, u64, p]
            L.ora_seed_h.argtypes = [u64]
            L.ora_seed_h.restype = u64
            L.ora_seed_c.argtypes = [u64]
            L.ora_seed_c.restype = u64
            L.ora_checksum.argtypes = [u64, u64]
            L.ora_checksum.restype = u32
            L.ora_cells_of.argtypes = [u64, u64, u32, u64, p]
            L.ora_cells_of.restype = i32
            L.ora_sync_peel.argtypes = [p, u64, u64, u32, u32, p, p, p, p, u32, p]
            L.ora_sync_peel.restype = i32
            L.ora_queue_peel.argtypes = [p, u64, u64, u32, u32, p]
            L.ora_gen_partitioned.argtypes = [u64, u64, u64, u32, p]
            L.ora_gen_partitioned.restype = i32
            L.ora_subround_peel.argtypes = [p, u64, u64, u32, u32, p, p, p, p, p, u32]
            L.ora_subround_peel.restype = i32
            L.ora_queue_peel.restype = i32
            L.ora_iblt_new.argtypes = [u64, u32, u64]
            L.ora_iblt_new.restype = p
            L.ora_iblt_new_ex.argtypes = [u64, u32, u64, i32]
            L.ora_iblt_new_ex.restype = p
            L.ora_iblt_new_blocked.argtypes = [u64, u32, u64, u32]
            L.ora_iblt_new_blocked.restype = p
            L.ora_cells_of_blocked.argtypes = [u64, u64, u32, u64, u32, p]
            L.ora_cells_of_blocked.restype = i32
            L.ora_iblt_peel_subtables.argtypes = [p, p, u64, p, p, p, u32, p]
            L.ora_iblt_peel_subtables.restype = i32
            L.ora_cells_of_subtable.argtypes = [u64, u64, u32, u64, p]
            L.ora_iblt_subtract.argtypes = [p, p]
            L.ora_iblt_subtract.restype = i32
            L.ora_iblt_peel_signed.argtypes = [p, p, p, u64, p, p, p, u32, p]
            L.ora_iblt_peel_signed.restype = i32
            L.ora_iblt_free.argtypes = [p]
            L.ora_iblt_seed_h.argtypes = [p]
            L.ora_iblt_seed_h.restype = u64
            L.ora_iblt_seed_c.argtypes = [p]
            L.ora_iblt_seed_c.restype = u64
            L.ora_iblt_insert.argtypes = [p, p, u64]
            L.ora_iblt_insert.restype = i32
            L.ora_iblt_delete.argtypes = [p, p, u64]
            L.ora_iblt_delete.restype = i32
            L.ora_iblt_dump.argtypes = [p, p, p, p]
            L.ora_iblt_load.argtypes = [p, p, p, p]
            L.ora_iblt_peel.argtypes = [p, p, u64, p, p, p, u32, p]
            L.ora_iblt_peel.restype = i32
            L.ora_iblt_serial_recover.argtypes = [p, p, u64, p, p]
            L.ora_iblt_serial_recover.restype = i32
            L.ora_iblt_to_hypergraph.argtypes = [p, p, u64, p]
            _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ---------------------------------------------------------------------------
# generator (restated in DESIGN.md §3)
# ---------------------------------------------------------------------------
def philox4x32_10(ctr, key) -> tuple:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().ora_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return tuple(int(x) for x in out)


def gen_edge(seed: int, n: int, r: int, e: int) -> np.ndarray:
    out = np.zeros(r, dtype=np.uint32)
    if lib().ora_gen_edge(seed, n, r, e, _ptr(out)):
        raise ValueError("bad generator arguments")
    return out


def gen_hypergraph(n: int, m: int, r: int, seed: int) -> np.ndarray:
    """edges[m][r] u32, G^r_{n,cn} with m = cn edges."""
    edges = np.zeros((m, r), dtype=np.uint32)
    if lib().ora_gen_hypergraph(seed, n, m, r, _ptr(edges)):
        raise ValueError("bad generator arguments (need r>=2, n>=r)")
    return edges


def gen_partitioned(n: int, m: int, r: int, seed: int) -> np.ndarray:
    """edges[m][r]: the subtable model, one uniform vertex per class j in [j n/r, (j+1) n/r)."""
    edges = np.zeros((m, r), dtype=np.uint32)
    if lib().ora_gen_partitioned(seed, n, m, r, _ptr(edges)):
        raise ValueError("bad arguments (need r>=2, n>=r, r | n)")
    return edges


def mix64(z: int) -> int:
    return int(lib().ora_mix64(z & 0xFFFFFFFFFFFFFFFF))


def gen_keys(nkeys: int, seed: int) -> np.ndarray:
    keys = np.zeros(nkeys, dtype=np.uint64)
    lib().ora_gen_keys(seed, nkeys, _ptr(keys))
    return keys


def seed_h(seed: int) -> int:
    return int(lib().ora_seed_h(seed))


def seed_c(seed: int) -> int:
    return int(lib().ora_seed_c(seed))


def checksum(x: int, seed: int) -> int:
    return int(lib().ora_checksum(x, seed_c(seed)))


def cells_of_subtable(x: int, C: int, r: int, seed: int) -> np.ndarray:
    out = np.zeros(r, dtype=np.uint64)
    lib().ora_cells_of_subtable(x, C, r, seed_h(seed), _ptr(out))
    return out


def cells_of_blocked(x: int, C: int, r: int, seed: int, blog: int) -> np.ndarray:
    """The r cells of key x under blocked hashing (one block of 2^blog cells; R27)."""
    out = np.zeros(r, dtype=np.uint64)
    if lib().ora_cells_of_blocked(x, C, r, seed_h(seed), blog, _ptr(out)):
        raise RuntimeError("cells_of_blocked: no r distinct cells")
    return out


def cells_of(x: int, C: int, r: int, seed: int) -> np.ndarray:
    out = np.zeros(r, dtype=np.uint64)
    if lib().ora_cells_of(x, C, r, seed_h(seed), _ptr(out)):
        raise ValueError("bad cell-hash arguments")
    return out


# ---------------------------------------------------------------------------
# k-core peels
# ---------------------------------------------------------------------------
class PeelResult:
    def __init__(self, core_mask, rounds, survivors, killed, peel_round):
        self.core_mask = core_mask
        self.rounds = rounds
        self.survivors = survivors
        self.killed = killed
        self.peel_round = peel_round

    def __repr__(self):
        return (f"PeelResult(rounds={self.rounds}, core={int(self.core_mask.sum())}, "
                f"survivors={self.survivors.tolist()[:6]}...)")


def sync_peel(edges: np.ndarray, n: int, k: int, cap: int = 1 << 16,
              want_peel_round: bool = False) -> PeelResult:
    """Literal round-synchronous peel."""
    edges = np.ascontiguousarray(edges, dtype=np.uint32)
    m = edges.shape[0]
    r = edges.shape[1] if edges.ndim == 2 and m > 0 else (edges.shape[1] if edges.ndim == 2 else 0)
    core = np.zeros(max(n, 1), dtype=np.uint8)
    rounds = ctypes.c_uint32(0)
    surv = np.zeros(cap, dtype=np.uint64)
    killed = np.zeros(cap, dtype=np.uint64)
    pr = np.zeros(max(n, 1), dtype=np.uint32) if want_peel_round else None
    st = lib().ora_sync_peel(_ptr(edges) if m else None, n, m, r, k, _ptr(core),
                             ctypes.addressof(rounds), _ptr(surv), _ptr(killed), cap,
                             _ptr(pr) if pr is not None else None)
    if st < 0:
        raise ValueError("oracle sync_peel: bad input or out of memory")
    if st == 1:
        raise OverflowError("more rounds than cap")
    t = rounds.value
    return PeelResult(core[:n].copy(), t, surv[:t].copy(), killed[:t].copy(),
                      pr[:n].copy() if pr is not None else None)


class SubroundResult:
    def __init__(self, core_mask, rounds, subrounds, survivors, killed):
        self.core_mask, self.rounds, self.subrounds = core_mask, rounds, subrounds
        self.survivors, self.killed = survivors, killed


def subround_peel(edges: np.ndarray, n: int, k: int, cap: int = 1 << 16) -> SubroundResult:
    """Subround peel, classes [j n/r, (j+1) n/r).  survivors[s-1] after flattened subround s."""
    edges = np.ascontiguousarray(edges, dtype=np.uint32)
    m, r = edges.shape
    core = np.zeros(max(n, 1), dtype=np.uint8)
    rounds = ctypes.c_uint32(0)
    sub = ctypes.c_uint32(0)
    surv = np.zeros(cap, dtype=np.uint64)
    kil = np.zeros(cap, dtype=np.uint64)
    st = lib().ora_subround_peel(_ptr(edges) if m else None, n, m, r, k, _ptr(core), ctypes.addressof(rounds),
                                 ctypes.addressof(sub), _ptr(surv), _ptr(kil), cap)
    if st < 0:
        raise ValueError("oracle subround_peel: bad input (r | n required)")
    if st == 1:
        raise OverflowError("more subrounds than cap")
    return SubroundResult(core[:n].copy(), rounds.value, sub.value, surv[:sub.value].copy(),
                          kil[:sub.value].copy())


def queue_peel(edges: np.ndarray, n: int, k: int) -> np.ndarray:
    """Serial greedy peel; returns the k-core mask."""
    edges = np.ascontiguousarray(edges, dtype=np.uint32)
    m = edges.shape[0]
    r = edges.shape[1]
    core = np.zeros(max(n, 1), dtype=np.uint8)
    if lib().ora_queue_peel(_ptr(edges) if m else None, n, m, r, k, _ptr(core)):
        raise MemoryError("oracle queue_peel")
    return core[:n].copy()


# ---------------------------------------------------------------------------
# IBLT
# ---------------------------------------------------------------------------
class IbltResult:
    def __init__(self, keys, rounds, per_round, complete, truncated=False):
        self.keys = keys
        self.rounds = rounds
        self.per_round = per_round
        self.complete = complete
        self.truncated = truncated


class Iblt:
    """IBLT with C cells and r hashes."""

    def __init__(self, C: int, r: int, seed: int, subtables: bool = False, blog: int = 0):
        self.C, self.r, self.seed, self.subtables, self.blog = C, r, seed, subtables, blog
        if blog:
            self._t = lib().ora_iblt_new_blocked(C, r, seed, blog)
        else:
            self._t = lib().ora_iblt_new_ex(C, r, seed, 1 if subtables else 0)
        if not self._t:
            raise ValueError("bad IBLT arguments (need r>=2, C>=r, r | C for subtables, 2^blog | C for blocks)")

    def __del__(self):
        t = getattr(self, "_t", None)
        if t:
            lib().ora_iblt_free(t)
            self._t = None

    def insert(self, keys: np.ndarray):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        lib().ora_iblt_insert(self._t, _ptr(keys), keys.size)

    def delete(self, keys: np.ndarray):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        lib().ora_iblt_delete(self._t, _ptr(keys), keys.size)

    def cells(self):
        count = np.zeros(self.C, dtype=np.int64)
        keysum = np.zeros(self.C, dtype=np.uint64)
        hashsum = np.zeros(self.C, dtype=np.uint32)
        lib().ora_iblt_dump(self._t, _ptr(count), _ptr(keysum), _ptr(hashsum))
        return count, keysum, hashsum

    def load_cells(self, count, keysum, hashsum):
        """Overwrite every cell (a serialized table; tests forge cells with it)."""
        count = np.ascontiguousarray(count, dtype=np.int64)
        keysum = np.ascontiguousarray(keysum, dtype=np.uint64)
        hashsum = np.ascontiguousarray(hashsum, dtype=np.uint32)
        assert count.size == keysum.size == hashsum.size == self.C
        lib().ora_iblt_load(self._t, _ptr(count), _ptr(keysum), _ptr(hashsum))

    def peel(self, cap_keys: int | None = None, cap: int = 1 << 16, allow_trunc: bool = False) -> IbltResult:
        """Round-synchronous recovery, destructive.  allow_trunc: a truncated
        recovery (cap, cap_keys or the 65536-round limit) is returned with .truncated set."""
        cap_keys = self.C * 2 if cap_keys is None else cap_keys
        out = np.zeros(max(cap_keys, 1), dtype=np.uint64)
        nrec = ctypes.c_uint64(0)
        rounds = ctypes.c_uint32(0)
        per_round = np.zeros(cap, dtype=np.uint64)
        complete = ctypes.c_int(0)
        st = lib().ora_iblt_peel(self._t, _ptr(out), cap_keys, ctypes.addressof(nrec),
                                 ctypes.addressof(rounds), _ptr(per_round), cap,
                                 ctypes.addressof(complete))
        if st < 0:
            raise MemoryError("oracle iblt_peel")
        if st == 1 and not allow_trunc:
            raise OverflowError("cap exceeded")
        t = rounds.value
        k = min(nrec.value, cap_keys)
        return IbltResult(out[:k].copy(), t, per_round[:min(t, cap)].copy(), bool(complete.value), st == 1)

    def peel_subtables(self, cap_keys: int | None = None, cap: int = 1 << 16) -> IbltResult:
        """Subtable recovery, destructive; rounds = flattened index of the last
        subtable step that recovered a key, per_round = keys per flattened step."""
        cap_keys = self.C * 2 if cap_keys is None else cap_keys
        out = np.zeros(max(cap_keys, 1), dtype=np.uint64)
        nrec = ctypes.c_uint64(0)
        sub = ctypes.c_uint32(0)
        per = np.zeros(cap, dtype=np.uint64)
        complete = ctypes.c_int(0)
        st = lib().ora_iblt_peel_subtables(self._t, _ptr(out), cap_keys, ctypes.addressof(nrec),
                                           ctypes.addressof(sub), _ptr(per), cap, ctypes.addressof(complete))
        if st < 0:
            raise ValueError("not a subtable IBLT")
        if st == 1:
            raise OverflowError("cap exceeded")
        return IbltResult(out[:nrec.value].copy(), sub.value, per[:sub.value].copy(), bool(complete.value))

    def subtract(self, other: "Iblt"):
        """self <- self - other cell-wise: the IBLT of the signed multiset difference."""
        if lib().ora_iblt_subtract(self._t, other._t):
            raise ValueError("tables differ in C, r, seed or layout")

    def peel_signed(self, cap_keys: int | None = None, cap: int = 1 << 16, allow_trunc: bool = False):
        """Recovery of a signed table: pure = count +-1, a matching checksum, and the cell is
        one of the key's cells (R26, R28); a key found in several pure cells is recovered
        once, with the sign of the lowest such cell.  Returns (IbltResult, signs) with
        signs[i] = +1 (key of A only) or -1 (key of B only)."""
        cap_keys = self.C * 2 if cap_keys is None else cap_keys
        out = np.zeros(max(cap_keys, 1), dtype=np.uint64)
        sg = np.zeros(max(cap_keys, 1), dtype=np.int8)
        nrec = ctypes.c_uint64(0)
        rounds = ctypes.c_uint32(0)
        per = np.zeros(cap, dtype=np.uint64)
        complete = ctypes.c_int(0)
        st = lib().ora_iblt_peel_signed(self._t, _ptr(out), _ptr(sg), cap_keys, ctypes.addressof(nrec),
                                        ctypes.addressof(rounds), _ptr(per), cap, ctypes.addressof(complete))
        if st < 0:
            raise MemoryError("oracle iblt_peel_signed")
        if st == 1 and not allow_trunc:
            raise OverflowError("cap exceeded")
        t = rounds.value
        k = min(nrec.value, cap_keys)
        return (IbltResult(out[:k].copy(), t, per[:min(t, cap)].copy(), bool(complete.value), st == 1),
                sg[:k].copy())

    def serial_recover(self):
        """One-pure-cell-at-a-time recovery, destructive."""
        cap_keys = self.C * 2
        out = np.zeros(cap_keys, dtype=np.uint64)
        nrec = ctypes.c_uint64(0)
        complete = ctypes.c_int(0)
        st = lib().ora_iblt_serial_recover(self._t, _ptr(out), cap_keys, ctypes.addressof(nrec),
                                           ctypes.addressof(complete))
        if st != 0:
            raise MemoryError("oracle serial_recover")
        return out[:nrec.value].copy(), bool(complete.value)

    def to_hypergraph(self, keys: np.ndarray) -> np.ndarray:
        """edge i = the r cells of key i."""
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        edges = np.zeros((keys.size, self.r), dtype=np.uint32)
        lib().ora_iblt_to_hypergraph(self._t, _ptr(keys), keys.size, _ptr(edges))
        return edges
