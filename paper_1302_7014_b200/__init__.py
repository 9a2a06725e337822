"""paper_1302_7014_b200 -- parallel peeling (k-core / IBLT recovery) on B200.

Thin Python binding over the C-ABI of ``libpeel.so`` (``include/peel.h``):
argument marshalling only; every step of the method runs in the library's
sm_100a kernels.  torch supplies device memory and streams.  There is no CPU
fallback: if the library is missing, every call raises.

Tensors: edges are int32 tensors holding u32 vertex ids, shape [m, r];
keys are int64 tensors holding u64 bit patterns.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PEEL_LIB") or os.path.join(_PKG, "libpeel.so")  # PEEL_LIB: A/B builds

PEEL_OK, PEEL_EINVAL, PEEL_ENOMEM, PEEL_ECUDA, PEEL_ETRUNC, PEEL_ENCCL, PEEL_EOVERFLOW, PEEL_EPEER = range(8)
PEEL_FLAG_CSR = 1
PEEL_FLAG_SUBROUNDS = 2
IBLT_FLAG_SUBTABLES = 1
IBLT_FLAG_BLOCKED = 2
IBLT_BLOCK_LOG_SHIFT = 8

_lib = None

# host-transport callbacks (peel.h peel_comm_init_host)
_AR_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64)
_AG_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64)
_A2A_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p)


class PeelError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        msg = _L().peel_strerror(status).decode()
        if status == PEEL_ECUDA:
            msg += " -- " + _L().peel_last_cuda_error().decode()
        super().__init__(f"{what}: {msg}")


def _L() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        u32, u64, i32, p, sz = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t
        L.peel_strerror.argtypes = [i32]
        L.peel_strerror.restype = ctypes.c_char_p
        L.peel_last_cuda_error.restype = ctypes.c_char_p
        L.peel_abi_version.restype = i32
        L.peel_gen_hypergraph.argtypes = [u64, u64, u32, u64, p, p]
        L.peel_gen_keys.argtypes = [u64, u64, p, p]
        L.peel_gen_partitioned.argtypes = [u64, u64, u32, u64, p, p]
        L.peel_kcore_workspace_bytes.argtypes = [u64, u64, u32, u32, u32]
        L.peel_kcore_workspace_bytes.restype = sz
        L.peel_kcore.argtypes = [p, u64, u64, u32, u32, u32, p, p, p, p, u32, p, p, sz, p]
        L.peel_kcore_host_workspace_bytes.argtypes = [u64, u64, u32, u32, u32]
        L.peel_kcore_host_workspace_bytes.restype = sz
        L.peel_kcore_host.argtypes = [p, u64, u64, u32, u32, u32, p, p, p, p, u32, p, sz, p]
        L.peel_sweep_workspace_bytes.argtypes = [u64, u64, u32, u32, u32]
        L.peel_sweep_workspace_bytes.restype = sz
        L.peel_sweep.argtypes = [u64, u32, u32, p, p, u64, u32, p, p, p, sz, p]
        L.peel_comm_unique_id.argtypes = [p]
        L.peel_comm_init.argtypes = [p, i32, i32, ctypes.POINTER(p)]
        L.peel_comm_init_virtual.argtypes = [i32, ctypes.POINTER(p)]
        L.peel_comm_init_host.argtypes = [i32, i32, _AR_FN, _AG_FN, _A2A_FN, p, ctypes.POINTER(p)]
        L.peel_comm_destroy.argtypes = [p]
        L.peel_kcore_dist_workspace_bytes.argtypes = [p, u64, u64, u32, u32]
        L.peel_kcore_dist_workspace_bytes.restype = sz
        L.peel_kcore_dist.argtypes = [p, p, u64, u64, u32, u32, p, p, p, p, u32, p, sz, p]
        L.iblt_dist_mem_bytes.argtypes = [p, u64, u32]
        L.iblt_dist_mem_bytes.restype = sz
        L.iblt_dist_recover.argtypes = [p, u64, u32, u64, u32, p, u64, p, u64, p, p, p, u32, p, p, sz, p]
        L.iblt_dist_recover_cells.argtypes = [p, p, u64, u32, u64, u32, p, u64, p, p, p, u32, p, p, sz, p]
        L.iblt_mem_bytes.argtypes = [u64, u32]
        L.iblt_mem_bytes.restype = sz
        L.iblt_build.argtypes = [u64, u32, u64, p, sz, p, ctypes.POINTER(p)]
        L.iblt_build_ex.argtypes = [u64, u32, u64, u32, p, sz, p, ctypes.POINTER(p)]
        L.iblt_insert.argtypes = [p, p, u64, p]
        L.iblt_delete.argtypes = [p, p, u64, p]
        L.iblt_peel.argtypes = [p, p, u64, p, p, p, u32, p, p]
        L.iblt_subtract.argtypes = [p, p, p]
        L.iblt_peel_signed.argtypes = [p, p, p, u64, p, p, p, u32, p, p]
        L.iblt_cells.argtypes = [p]
        L.iblt_cells.restype = p
        L.iblt_to_hypergraph.argtypes = [p, p, u64, p, p]
        L.iblt_destroy.argtypes = [p]
        L.peel_profile_enable.argtypes = [i32]
        L.peel_profile_read.argtypes = [p, p, p, i32]
        L.peel_profile_read.restype = i32
        L.peel_last_launches.restype = u32
        L.peel_profile_rounds.argtypes = [p, u32]
        L.peel_profile_rounds.restype = i32
        for f in ("peel_gen_hypergraph", "peel_gen_keys", "peel_gen_partitioned", "peel_kcore", "peel_kcore_host", "peel_sweep",
                  "peel_comm_unique_id", "peel_comm_init", "peel_comm_init_virtual", "peel_kcore_dist", "iblt_build", "iblt_build_ex",
                  "iblt_dist_recover", "iblt_dist_recover_cells", "peel_comm_init_host",
                  "iblt_insert", "iblt_delete", "iblt_peel", "iblt_subtract", "iblt_peel_signed", "iblt_to_hypergraph"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def lib() -> ctypes.CDLL:
    """The loaded libpeel.so (raises if not built)."""
    return _L()


def _check(st: int, what: str, ok=(PEEL_OK,)):
    if st not in ok:
        raise PeelError(st, what)
    return st


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def _dev(device):
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


# ---------------------------------------------------------------------------
# a1 generator
# ---------------------------------------------------------------------------
def gen_hypergraph(n: int, m: int, r: int, seed: int, out: torch.Tensor | None = None,
                   device=None, stream=None) -> torch.Tensor:
    """edges [m, r] (int32 storage of u32 ids) of G^r_{n,cn} (peel.h peel_gen_hypergraph)."""
    if out is None:
        out = torch.empty((m, r), dtype=torch.int32, device=_dev(device))
    _check(_L().peel_gen_hypergraph(n, m, r, seed & (2**64 - 1), _ptr(out), _stream(stream)),
           "peel_gen_hypergraph")
    return out


def gen_partitioned(n: int, m: int, r: int, seed: int, out: torch.Tensor | None = None,
                    device=None, stream=None) -> torch.Tensor:
    """edges [m, r] of the subtable model: one vertex per class [c n/r, (c+1) n/r) (peel.h)."""
    if out is None:
        out = torch.empty((m, r), dtype=torch.int32, device=_dev(device))
    _check(_L().peel_gen_partitioned(n, m, r, seed & (2**64 - 1), _ptr(out), _stream(stream)),
           "peel_gen_partitioned")
    return out


def gen_keys(nkeys: int, seed: int, out: torch.Tensor | None = None, device=None, stream=None) -> torch.Tensor:
    """nkeys distinct u64 keys (int64 storage), SplitMix64 stream (peel.h peel_gen_keys)."""
    if out is None:
        out = torch.empty((nkeys,), dtype=torch.int64, device=_dev(device))
    _check(_L().peel_gen_keys(nkeys, seed & (2**64 - 1), _ptr(out), _stream(stream)), "peel_gen_keys")
    return out


# ---------------------------------------------------------------------------
# k-core
# ---------------------------------------------------------------------------
class KcoreResult:
    def __init__(self, core_mask, rounds, survivors, killed, peel_round, status):
        self.core_mask = core_mask
        self.rounds = rounds
        self.survivors = survivors
        self.killed = killed
        self.peel_round = peel_round
        self.status = status

    def __repr__(self):
        return f"KcoreResult(rounds={self.rounds}, survivors[-1]={self.survivors[-1] if len(self.survivors) else None})"


_ws_cache: dict = {}


def workspace(nbytes: int, device) -> torch.Tensor:
    """A cached uint8 device workspace of at least nbytes."""
    key = str(device)
    t = _ws_cache.get(key)
    if t is None or t.numel() < nbytes:
        _ws_cache.pop(key, None)
        t = torch.empty((max(nbytes, 256),), dtype=torch.uint8, device=device)
        _ws_cache[key] = t
    return t


def kcore_workspace_bytes(n: int, m: int, r: int, k: int, flags: int = 0) -> int:
    return int(_L().peel_kcore_workspace_bytes(n, m, r, k, flags))


def peel_kcore(edges: torch.Tensor, n: int, k: int, flags: int = 0, cap: int = 65536,
               core_mask: torch.Tensor | None = None, want_peel_round: bool = False,
               ws: torch.Tensor | None = None, stream=None, allow_trunc: bool = False) -> KcoreResult:
    """Round-synchronous peel of the hypergraph `edges` [m, r] to its k-core (peel.h peel_kcore)."""
    assert edges.dim() == 2 and edges.dtype == torch.int32 and edges.is_cuda and edges.is_contiguous()
    m, r = edges.shape
    dev = edges.device
    need = kcore_workspace_bytes(n, m, r, k, flags)
    if need == 0:
        raise PeelError(PEEL_EINVAL, "peel_kcore_workspace_bytes")
    if ws is None:
        ws = workspace(need, dev)
    if core_mask is None:
        core_mask = torch.empty((n,), dtype=torch.uint8, device=dev)
    pr = torch.empty((n,), dtype=torch.int32, device=dev) if want_peel_round else None
    rounds = ctypes.c_uint32(0)
    surv = np.zeros(cap, dtype=np.uint64)
    killed = np.zeros(cap, dtype=np.uint64)
    st = _L().peel_kcore(_ptr(edges), n, m, r, k, flags, _ptr(core_mask), ctypes.addressof(rounds),
                         surv.ctypes.data, killed.ctypes.data, cap, _ptr(pr), _ptr(ws), ws.numel(),
                         _stream(stream))
    _check(st, "peel_kcore", ok=(PEEL_OK, PEEL_ETRUNC) if allow_trunc else (PEEL_OK,))
    t = rounds.value
    nst = min(t, cap)
    return KcoreResult(core_mask, t, surv[:nst].copy(), killed[:nst].copy(), pr, st)


def peel_kcore_host(edges_host: np.ndarray, n: int, k: int, flags: int = 0, cap: int = 65536,
                    core_mask_host: np.ndarray | None = None, ws: torch.Tensor | None = None,
                    device=None, stream=None):
    """peel_kcore with host (preferably pinned) input edges and output mask (peel.h peel_kcore_host).
    edges_host: uint32/int32 numpy array or pinned CPU tensor [m, r]."""
    if isinstance(edges_host, torch.Tensor):
        m, r = edges_host.shape
        eptr = edges_host.data_ptr()
    else:
        m, r = edges_host.shape
        eptr = edges_host.ctypes.data
    dev = _dev(device)
    need = int(_L().peel_kcore_host_workspace_bytes(n, m, r, k, flags))
    if need == 0:
        raise PeelError(PEEL_EINVAL, "peel_kcore_host_workspace_bytes")
    if ws is None:
        ws = workspace(need, dev)
    if core_mask_host is None:
        core_mask_host = np.empty((n,), dtype=np.uint8)
    mptr = core_mask_host.data_ptr() if isinstance(core_mask_host, torch.Tensor) else core_mask_host.ctypes.data
    rounds = ctypes.c_uint32(0)
    surv = np.zeros(cap, dtype=np.uint64)
    killed = np.zeros(cap, dtype=np.uint64)
    st = _L().peel_kcore_host(eptr, n, m, r, k, flags, mptr, ctypes.addressof(rounds), surv.ctypes.data,
                              killed.ctypes.data, cap, _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "peel_kcore_host")
    t = rounds.value
    return KcoreResult(core_mask_host, t, surv[:min(t, cap)].copy(), killed[:min(t, cap)].copy(), None, st)


# ---------------------------------------------------------------------------
# trial sweeps (e1)
# ---------------------------------------------------------------------------
def sweep(n: int, r: int, k: int, m, seeds, batch: int = 128, device=None, ws: torch.Tensor | None = None,
          stream=None):
    """Per-trial (rounds, core vertices) for trials (m[t], seeds[t]) of G^r_{n,m[t]} (peel.h peel_sweep)."""
    m = np.ascontiguousarray(m, dtype=np.uint64)
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    assert m.shape == seeds.shape
    T = m.size
    rounds = np.zeros(T, dtype=np.uint32)
    core = np.zeros(T, dtype=np.uint64)
    if T == 0:
        return rounds, core
    batch = max(1, min(batch, T))
    need = int(_L().peel_sweep_workspace_bytes(n, int(m.max()), r, k, batch))
    if need == 0:
        raise PeelError(PEEL_EINVAL, "peel_sweep_workspace_bytes")
    if ws is None:
        ws = workspace(need, _dev(device))
    _check(_L().peel_sweep(n, r, k, m.ctypes.data, seeds.ctypes.data, T, batch, rounds.ctypes.data,
                           core.ctypes.data, _ptr(ws), ws.numel(), _stream(stream)), "peel_sweep")
    return rounds, core


# ---------------------------------------------------------------------------
# vertex-partitioned single instance over P GPUs (e2)
# ---------------------------------------------------------------------------
class Comm:
    """peel_comm: NCCL (one process per GPU) or P virtual shards on one GPU (peel.h e2)."""

    def __init__(self, handle, nshards: int, rank: int, virtual: bool):
        self._h, self.P, self.rank, self.virtual = handle, nshards, rank, virtual

    @classmethod
    def virtual_shards(cls, nshards: int):
        h = ctypes.c_void_p(0)
        _check(_L().peel_comm_init_virtual(nshards, ctypes.byref(h)), "peel_comm_init_virtual")
        return cls(h, nshards, -1, True)

    @classmethod
    def from_process_group(cls, group=None, device=None):
        """NCCL communicator over the ranks of a torch.distributed group (rank 0 makes the
        unique id, broadcast as a byte tensor); call after torch.cuda.set_device."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        idb = np.zeros(128, dtype=np.uint8)
        if rank == 0:
            _check(_L().peel_comm_unique_id(idb.ctypes.data), "peel_comm_unique_id")
        t = torch.from_numpy(idb).to(_dev(device))
        dist.broadcast(t, src=0, group=group)
        idb = t.cpu().numpy()
        h = ctypes.c_void_p(0)
        _check(_L().peel_comm_init(idb.ctypes.data, world, rank, ctypes.byref(h)), "peel_comm_init")
        return cls(h, world, rank, False)

    @classmethod
    def host_transport(cls, group=None):
        """Rank communicator whose collectives run through torch.distributed on the HOST
        (e.g. a gloo group; peel.h peel_comm_init_host): the per-rank protocol of the NCCL
        path with device<->host staging, so several ranks may share one GPU.  The callbacks
        only move bytes between the library's pinned buffers and the process group."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)

        def u8(ptr, nbytes):
            return np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(ptr)) if nbytes else \
                np.zeros(0, dtype=np.uint8)

        def allreduce(_ctx, vals, count):
            try:
                a = u8(vals, 8 * count).view(np.int64)
                t = torch.from_numpy(a.copy())
                dist.all_reduce(t, group=group)
                a[:] = t.numpy()
                return 0
            except Exception:  # noqa: BLE001 -- reported to the library as a transport failure
                return 1

        def allgather(_ctx, send, recv, nbytes):
            try:
                t = torch.from_numpy(u8(send, nbytes).copy())
                out = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(out, t, group=group)
                u8(recv, nbytes * world)[:] = torch.cat(out).numpy()
                return 0
            except Exception:  # noqa: BLE001
                return 1

        def alltoallv(_ctx, send, sbytes, recv, rbytes):
            try:
                sb = np.ctypeslib.as_array((ctypes.c_uint64 * world).from_address(sbytes)).astype(np.int64)
                rb = np.ctypeslib.as_array((ctypes.c_uint64 * world).from_address(rbytes)).astype(np.int64)
                so = np.concatenate([[0], np.cumsum(sb)])
                ro = np.concatenate([[0], np.cumsum(rb)])
                sall = u8(send, int(so[-1]))
                reqs, bufs = [], []
                for q in range(world):
                    if q != rank and rb[q]:
                        b = torch.empty(int(rb[q]), dtype=torch.uint8)
                        bufs.append((q, b))
                        reqs.append(dist.irecv(b, src=q, group=group))
                for q in range(world):
                    if q != rank and sb[q]:
                        reqs.append(dist.isend(torch.from_numpy(sall[so[q]:so[q + 1]].copy()), dst=q, group=group))
                for rq in reqs:
                    rq.wait()
                rall = u8(recv, int(ro[-1]))
                for q, b in bufs:
                    rall[ro[q]:ro[q + 1]] = b.numpy()
                return 0
            except Exception:  # noqa: BLE001
                return 1

        fns = (_AR_FN(allreduce), _AG_FN(allgather), _A2A_FN(alltoallv))
        h = ctypes.c_void_p(0)
        _check(_L().peel_comm_init_host(world, rank, *fns, None, ctypes.byref(h)), "peel_comm_init_host")
        c = cls(h, world, rank, False)
        c._fns = fns  # the library keeps the function pointers: keep them alive
        return c

    def shard(self, n: int, q: int | None = None) -> tuple[int, int]:
        q = self.rank if q is None else q
        return q * n // self.P, (q + 1) * n // self.P

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.peel_comm_destroy(h)
            self._h = None


def peel_kcore_dist(comm: Comm, edges: torch.Tensor, n: int, k: int, cap: int = 65536,
                    core_mask: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None):
    """Vertex-partitioned peel (peel.h peel_kcore_dist).  core_mask: this rank's slice
    (NCCL) or all n vertices (virtual shards).  rounds/survivors/killed are global."""
    assert edges.dim() == 2 and edges.dtype == torch.int32 and edges.is_cuda and edges.is_contiguous()
    m, r = edges.shape
    need = int(_L().peel_kcore_dist_workspace_bytes(comm._h, n, m, r, k))
    if need == 0:
        raise PeelError(PEEL_EINVAL, "peel_kcore_dist_workspace_bytes")
    if ws is None:
        ws = workspace(need, edges.device)
    if core_mask is None:
        lo, hi = (0, n) if comm.virtual else comm.shard(n)
        core_mask = torch.empty((hi - lo,), dtype=torch.uint8, device=edges.device)
    rounds = ctypes.c_uint32(0)
    surv = np.zeros(cap, dtype=np.uint64)
    killed = np.zeros(cap, dtype=np.uint64)
    st = _L().peel_kcore_dist(comm._h, _ptr(edges), n, m, r, k, _ptr(core_mask), ctypes.addressof(rounds),
                              surv.ctypes.data, killed.ctypes.data, cap, _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "peel_kcore_dist")
    t = rounds.value
    return KcoreResult(core_mask, t, surv[:min(t, cap)].copy(), killed[:min(t, cap)].copy(), None, st)


# ---------------------------------------------------------------------------
# IBLT
# ---------------------------------------------------------------------------
class IbltResult:
    def __init__(self, keys, nrecovered, rounds, per_round, complete, status):
        self.keys = keys
        self.nrecovered = nrecovered
        self.rounds = rounds
        self.per_round = per_round
        self.complete = complete
        self.status = status


class Iblt:
    """IBLT of `cells` 16-byte cells and r hashes in a torch-owned device buffer (peel.h iblt_*)."""

    def __init__(self, cells: int, r: int, seed: int, device=None, stream=None, mem: torch.Tensor | None = None,
                 subtables: bool = False, blog: int = 0):
        """blog > 0: blocked (locality-aware) hashing, all r cells of a key in one block of
        2^blog cells (peel.h IBLT_FLAG_BLOCKED)."""
        self.C, self.r, self.seed, self.subtables, self.blog = cells, r, seed, subtables, blog
        self.device = _dev(device) if mem is None else mem.device
        nb = int(_L().iblt_mem_bytes(cells, r))
        if nb == 0:
            raise PeelError(PEEL_EINVAL, "iblt_mem_bytes")
        self.mem = torch.empty((nb,), dtype=torch.uint8, device=self.device) if mem is None else mem
        self._h = None
        self.reset(stream)

    def reset(self, stream=None):
        """(Re)build: zero the cells in place (peel.h iblt_build)."""
        if self._h is not None and self._h.value:
            _L().iblt_destroy(self._h)
        h = ctypes.c_void_p(0)
        flags = IBLT_FLAG_SUBTABLES if self.subtables else 0
        if self.blog:
            flags |= IBLT_FLAG_BLOCKED | (self.blog << IBLT_BLOCK_LOG_SHIFT)
        _check(_L().iblt_build_ex(self.C, self.r, self.seed & (2**64 - 1), flags,
                                  _ptr(self.mem), self.mem.numel(), _stream(stream), ctypes.byref(h)), "iblt_build_ex")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.iblt_destroy(h)
            self._h = None

    def insert(self, keys: torch.Tensor, stream=None):
        assert keys.dtype == torch.int64 and keys.is_cuda and keys.is_contiguous()
        _check(_L().iblt_insert(self._h, _ptr(keys), keys.numel(), _stream(stream)), "iblt_insert")

    def delete(self, keys: torch.Tensor, stream=None):
        assert keys.dtype == torch.int64 and keys.is_cuda and keys.is_contiguous()
        _check(_L().iblt_delete(self._h, _ptr(keys), keys.numel(), _stream(stream)), "iblt_delete")

    def cells(self) -> torch.Tensor:
        """[C, 4] int32 COPY (count, hashSum, keySum_lo, keySum_hi) of the device cells."""
        return self.mem[: 16 * self.C].view(torch.int32).view(self.C, 4).clone()

    def load_cells(self, cells: torch.Tensor):
        """Overwrite every cell with `cells` ([C, 4] int32, the layout of cells()): a
        serialized or received table.  Goes through iblt_cells(), so recovery no longer
        assumes an insert-only table (peel.h)."""
        ptr = _L().iblt_cells(self._h)
        assert ptr == self.mem.data_ptr()
        self.mem[: 16 * self.C].view(torch.int32).view(self.C, 4).copy_(cells)

    def peel(self, cap_keys: int | None = None, cap: int = 65536, out: torch.Tensor | None = None,
             stream=None, allow_trunc: bool = False) -> IbltResult:
        cap_keys = self.C if cap_keys is None else cap_keys
        if out is None:
            out = torch.empty((max(cap_keys, 1),), dtype=torch.int64, device=self.device)
        nrec = ctypes.c_uint64(0)
        rounds = ctypes.c_uint32(0)
        per_round = np.zeros(cap, dtype=np.uint64)
        complete = ctypes.c_int(0)
        st = _L().iblt_peel(self._h, _ptr(out), cap_keys, ctypes.addressof(nrec), ctypes.addressof(rounds),
                            per_round.ctypes.data, cap, ctypes.addressof(complete), _stream(stream))
        _check(st, "iblt_peel", ok=(PEEL_OK, PEEL_ETRUNC) if allow_trunc else (PEEL_OK,))
        t = rounds.value
        return IbltResult(out[: min(nrec.value, cap_keys)], nrec.value, t, per_round[:min(t, cap)].copy(),
                          bool(complete.value), st)

    def subtract(self, other: "Iblt", stream=None):
        """self <- self - other cell-wise: the IBLT of the signed difference (peel.h iblt_subtract)."""
        _check(_L().iblt_subtract(self._h, other._h, _stream(stream)), "iblt_subtract")

    def peel_signed(self, cap_keys: int | None = None, cap: int = 65536, stream=None, allow_trunc: bool = False):
        """Recovery of a signed table (peel.h iblt_peel_signed): returns (IbltResult, signs)."""
        cap_keys = self.C if cap_keys is None else cap_keys
        out = torch.empty((max(cap_keys, 1),), dtype=torch.int64, device=self.device)
        sg = torch.empty((max(cap_keys, 1),), dtype=torch.int8, device=self.device)
        nrec = ctypes.c_uint64(0)
        rounds = ctypes.c_uint32(0)
        per_round = np.zeros(cap, dtype=np.uint64)
        complete = ctypes.c_int(0)
        st = _L().iblt_peel_signed(self._h, _ptr(out), _ptr(sg), cap_keys, ctypes.addressof(nrec),
                                   ctypes.addressof(rounds), per_round.ctypes.data, cap, ctypes.addressof(complete),
                                   _stream(stream))
        _check(st, "iblt_peel_signed", ok=(PEEL_OK, PEEL_ETRUNC) if allow_trunc else (PEEL_OK,))
        t = rounds.value
        k = min(nrec.value, cap_keys)
        return IbltResult(out[:k], nrec.value, t, per_round[:min(t, cap)].copy(), bool(complete.value), st), sg[:k]

    def to_hypergraph(self, keys: torch.Tensor, stream=None) -> torch.Tensor:
        edges = torch.empty((keys.numel(), self.r), dtype=torch.int32, device=self.device)
        _check(_L().iblt_to_hypergraph(self._h, _ptr(keys), keys.numel(), _ptr(edges), _stream(stream)),
               "iblt_to_hypergraph")
        return edges


def iblt_dist_recover(comm: Comm, cells: int, r: int, seed: int, keys: torch.Tensor, blog: int = 0,
                      cap_keys: int | None = None, cap: int = 65536, mem: torch.Tensor | None = None,
                      stream=None) -> IbltResult:
    """Cell-partitioned IBLT over the communicator's shards (peel.h iblt_dist_recover): insert
    `keys` (the same device array on every rank) and recover.  keys of the result: those found
    by this rank (virtual shards: all); rounds, per_round and complete are global."""
    assert keys.dtype == torch.int64 and keys.is_cuda and keys.is_contiguous()
    need = int(_L().iblt_dist_mem_bytes(comm._h, cells, r))
    if need == 0:
        raise PeelError(PEEL_EINVAL, "iblt_dist_mem_bytes")
    if mem is None:
        mem = workspace(need, keys.device)
    cap_keys = keys.numel() if cap_keys is None else cap_keys
    out = torch.empty((max(cap_keys, 1),), dtype=torch.int64, device=keys.device)
    flags = (IBLT_FLAG_BLOCKED | (blog << IBLT_BLOCK_LOG_SHIFT)) if blog else 0
    nrec = ctypes.c_uint64(0)
    rounds = ctypes.c_uint32(0)
    per_round = np.zeros(cap, dtype=np.uint64)
    complete = ctypes.c_int(0)
    st = _L().iblt_dist_recover(comm._h, cells, r, seed & (2**64 - 1), flags, _ptr(keys), keys.numel(), _ptr(out),
                                cap_keys, ctypes.addressof(nrec), ctypes.addressof(rounds), per_round.ctypes.data, cap,
                                ctypes.addressof(complete), _ptr(mem), mem.numel(), _stream(stream))
    _check(st, "iblt_dist_recover")
    t = rounds.value
    return IbltResult(out[: min(nrec.value, cap_keys)], nrec.value, t, per_round[:min(t, cap)].copy(),
                      bool(complete.value), st)


def iblt_dist_recover_cells(comm: Comm, cells: torch.Tensor, r: int, seed: int, blog: int = 0,
                            cap_keys: int | None = None, cap: int = 65536, mem: torch.Tensor | None = None,
                            stream=None) -> IbltResult:
    """Cell-partitioned recovery of an existing table (peel.h iblt_dist_recover_cells): cells
    is the [C, 4] int32 device table (Iblt.cells() layout), the same on every rank."""
    assert cells.is_cuda and cells.is_contiguous() and cells.dim() == 2 and cells.shape[1] == 4
    C = cells.shape[0]
    need = int(_L().iblt_dist_mem_bytes(comm._h, C, r))
    if need == 0:
        raise PeelError(PEEL_EINVAL, "iblt_dist_mem_bytes")
    if mem is None:
        mem = workspace(need, cells.device)
    cap_keys = C if cap_keys is None else cap_keys
    out = torch.empty((max(cap_keys, 1),), dtype=torch.int64, device=cells.device)
    flags = (IBLT_FLAG_BLOCKED | (blog << IBLT_BLOCK_LOG_SHIFT)) if blog else 0
    nrec = ctypes.c_uint64(0)
    rounds = ctypes.c_uint32(0)
    per_round = np.zeros(cap, dtype=np.uint64)
    complete = ctypes.c_int(0)
    st = _L().iblt_dist_recover_cells(comm._h, _ptr(cells), C, r, seed & (2**64 - 1), flags, _ptr(out), cap_keys,
                                      ctypes.addressof(nrec), ctypes.addressof(rounds), per_round.ctypes.data, cap,
                                      ctypes.addressof(complete), _ptr(mem), mem.numel(), _stream(stream))
    _check(st, "iblt_dist_recover_cells")
    t = rounds.value
    return IbltResult(out[: min(nrec.value, cap_keys)], nrec.value, t, per_round[:min(t, cap)].copy(),
                      bool(complete.value), st)


# ---------------------------------------------------------------------------
# measurement support
# ---------------------------------------------------------------------------
def profile_enable(on: bool = True):
    _L().peel_profile_enable(1 if on else 0)


def profile_read() -> list[tuple[str, float, int]]:
    names = (ctypes.c_char_p * 64)()
    ms = (ctypes.c_double * 64)()
    nl = (ctypes.c_uint32 * 64)()
    n = _L().peel_profile_read(ctypes.addressof(names), ctypes.addressof(ms), ctypes.addressof(nl), 64)
    return [(names[i].decode(), ms[i], nl[i]) for i in range(min(n, 64))]


def profile_rounds() -> list[float]:
    """Per-round device time (ms) of the last peel_kcore call (profiling enabled)."""
    buf = (ctypes.c_double * 65536)()
    n = _L().peel_profile_rounds(ctypes.addressof(buf), 65536)
    return [buf[i] for i in range(min(n, 65536))]


def last_launches() -> int:
    return int(_L().peel_last_launches())
