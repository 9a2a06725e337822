#!/usr/bin/env python
"""bench.py -- round-synchronous k-core peeling on B200 (BASELINE.json metric).

One "step" = one full peel_kcore call (a2-a7: degree/state build, every
round, core-mask output) over one synthetic G^r_{n,cn} instance already
resident in HBM; the generator (a1) produces the input outside the timed
region.  Default workload = BASELINE.json configs[4] at N=1: n=10^9, r=3,
k=2, c=0.75 (m=7.5e8), seed 6 -- the north-star instance.

  python bench.py [--gpus N --steps K --warmup W] [--config C5|C1|C3|C4a|C4b|C2]
  python bench.py --impl reference ...   (the CPU oracle on the host cores)

Multi-GPU (torchrun): every rank peels its own independent instance (seed +
rank; weak scaling, no data-path collective); time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_FLUSH_BELOW = 252 << 20  # 2x the B200 L2 (126 MB)


def timed_loop(steps, stream, dev, footprint, body):
    """Run body(i) for i < steps and return (device ms over the steps, l2 note).  A working set
    below 2x L2 gets a 256 MB L2 flush before every step, outside the timed intervals (each step
    is then timed alone with CUDA events on `stream`); a larger one is timed as one interval."""
    import torch
    flush = torch.empty((256 << 20,), dtype=torch.uint8, device=dev) if footprint < L2_FLUSH_BELOW else None
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps if flush is not None else 1)]
    if flush is None:
        evs[0][0].record(stream)
    for i in range(steps):
        if flush is not None:
            flush.fill_(i & 0xff)
            evs[i][0].record(stream)
        body(i)
        if flush is not None:
            evs[i][1].record(stream)
    if flush is None:
        evs[0][1].record(stream)
    torch.cuda.synchronize()
    note = (f"working set {footprint / 1e6:.0f} MB < 2x L2: 256 MB L2 flush before each step, outside the timed intervals"
            if flush is not None else f"working set {footprint / 1e9:.2f} GB > 2x L2; no flush needed")
    return sum(a.elapsed_time(b) for a, b in evs), note


CONFIGS = {
    # name: (kind, n_or_cells, m_or_keys, r, k, seed, BASELINE.json config text)
    "C1": ("kcore", 100_000, 70_000, 3, 2, 1, "k-core peel r=3 k=2 n=100,000 c=0.7"),
    "C2": ("iblt", 10_000_000, 7_500_000, 3, 2, 2, "IBLT recovery r=3, 10^7 cells, 7.5e6 keys"),
    "C3": ("kcore", 100_000_000, 75_000_000, 4, 2, 3, "k-core peel r=4 k=2 n=10^8 c=0.75"),
    "C4a": ("kcore", 100_000_000, 85_000_000, 3, 2, 4, "above-threshold k-core r=3 k=2 c=0.85 n=10^8"),
    "C4b": ("kcore", 100_000_000, 160_000_000, 3, 3, 5, "above-threshold k-core r=3 k=3 c=1.6 n=10^8"),
    "C5": ("kcore", 1_000_000_000, 750_000_000, 3, 2, 6, "r=3 k=2 c=0.75 n=10^9 (north star)"),
    "C5s": ("sweep", 1_000_000, 10_000, 3, 2, 1000, "sweep of 10^4 trials, n=10^6, r=3, k=2, c=0.700..0.898"),
}
METRIC = "hyperedges peeled/sec"
IBLT_METRIC = "IBLT keys recovered/sec (insert + recovery)"
SWEEP_METRIC = "sweep trials/sec"


def algorithmic_bytes(r, n, m, n_core, m_core, k):
    """SURVEY §8 d0 compulsory traffic of a work-efficient synchronous peel, split by kernel.
    k<=2 packed state: build = read edges 4rm + write state 8n; rounds = read state of removed
    vertices 8(n-n_core) + per killed edge re-read its ids 4r and RMW r-1 endpoints 16(r-1),
    plus the n-byte mask."""
    if k <= 2:
        build = 4 * r * m + 8 * n
        rounds = 8 * (n - n_core) + (m - m_core) * (4 * r + 16 * (r - 1)) + n
    else:  # CSR (u32 deg + offsets + adj): SURVEY §8 d0 general-k formula
        build = (4 * r * m + 4 * n) + 8 * n + 8 * r * m
        rounds = 12 * (n - n_core) + 4 * r * (m - m_core) + (m - m_core) * (4 * r + 8 * (r - 1)) + n
    return build, rounds


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# bench.py's per-call profiling names -> the kernel (tools/ncu_traffic.py short name) doing the work
NCU_KERNEL = {"peel_rounds_packed": ("peel_packed",), "peel_rounds_csr": ("peel_csr",), "iblt_peel_rounds": ("iblt_peel",),
              "peel_small_graph": ("build_packed", "peel_cluster"), "peel_rounds_cluster": ("peel_cluster",),
              "iblt_insert": ("iblt_update",), "frontier_edge_sort": ("esort_hist", "esort_scatter"),
              # slot-compacted binned rounds (kcompact.cuh) for n > 2^23, k <= 2
              "bin_accumulate": ("cbuild", "bin_accumulate"), "round_kill_partition": ("ckill", "round_kill_partition"),
              "round_apply": ("capply", "round_apply"), "compact_slots": ("ccompact", "ccompact_reg"),
              "compact_core_mask": ("ctail", "cmask"), "compact_writeback": ("cdecompact",),
              "compact_gather": ("cgather",)}
PROFILE_ROUNDS = ("r02", "r01")  # newest first: profiles/<round>_traffic_<config>.json


def profile_file(kind, config, kernel=None):
    """The newest committed profile of this kind for the config (None if there is none)."""
    for rnd in PROFILE_ROUNDS:
        name = f"{rnd}_{kind}_{kernel}_{config}.json" if kernel else f"{rnd}_{kind}_{config}.json"
        path = os.path.join(ROOT, "profiles", name)
        if os.path.exists(path):
            return path
    return None


def ncu_traffic(config, kernel, rounds=None):
    """DRAM bytes (read + write) per launch of `kernel`: from the committed `ncu --set full`
    capture of this config's kernel (profiles/r01_ncu_full_<kernel>_<config>.json) when there
    is one, else from the committed launch list (profiles/r01_traffic_<config>.json,
    tools/ncu_traffic.py), else None."""
    full = profile_file("ncu_full", config, kernel)
    if full:
        d = json.load(open(full))
        return int(d["dram_gb_per_launch"] * 1e9), \
            f"profiles/{os.path.basename(full)} (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum)"
    tf = profile_file("traffic", config)
    try:
        d = json.load(open(tf))
    except Exception:
        return None, None
    ks = [k for k in (d.get("kernels", {}).get(x) for x in NCU_KERNEL.get(kernel, (kernel,))) if k]
    if not ks:
        return None, None
    per_step = sum(k["dram_read_bytes_per_step"] + k["dram_write_bytes_per_step"] for k in ks)
    nlaunch = ks[-1]["launches_per_step"]
    if rounds and kernel in ("round_kill_partition", "round_apply"):
        nlaunch = min(nlaunch, rounds)  # launches after the device-side loop stopped move nothing
    return int(per_step / nlaunch), \
        f"profiles/{os.path.basename(tf)} (ncu, dram__bytes_read.sum + dram__bytes_write.sum)"


def dram_step(config, per_kernel, steps, ms_step, hbm):
    """Whole-step real DRAM traffic: the committed ncu bytes of every kernel this step launched
    (profiles/r01_traffic_<config>.json, per step) over this run's step time, or None."""
    tf = profile_file("traffic", config)
    try:
        d = json.load(open(tf))["kernels"]
    except Exception:
        return None
    tot, missing = 0.0, []
    for name in per_kernel:
        keys = NCU_KERNEL.get(name, (name,))
        found = [d[k] for k in keys if k in d]
        if not found:
            missing.append(name)
        tot += sum(f["dram_read_bytes_per_step"] + f["dram_write_bytes_per_step"] for f in found)
    return {"bytes": int(tot), "frac_of_peak": round(tot / (ms_step / 1e3) / 1e9 / hbm, 4),
            "kernels_without_traffic": missing,
            "source": f"profiles/{os.path.basename(tf)} (ncu dram__bytes_read.sum + dram__bytes_write.sum)"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def host_cpu():
    """CPU model and core count of this host (for the cpu_baseline record)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


class OneCore:
    """Pin this process to one core for the duration (the oracle is single-threaded by
    definition; SURVEY §8 d0 `taskset -c 0`)."""

    def __enter__(self):
        self.old = os.sched_getaffinity(0)
        self.core = min(self.old)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.old)


def cpu_baseline_kcore(r, k, c, target_s=12.0, config=None):
    """The oracle as it stands (single-threaded literal synchronous peel) on a bounded
    sample: instances of the same model (r, k, c) scaled down so they run ~10-30 s, pinned to
    one core.  Also timed on the same instances: the serial queue peel (ora_queue_peel, the
    work-efficient comparator of P:516's serial recovery).  The full-scale oracle run of the
    workload, when tests/golden/oracle_goldens.json recorded one, is quoted beside them."""
    from oracle import oracle as O
    n = 2_000_000
    t_total = t_queue = 0.0
    peeled = 0
    runs = 0
    with OneCore() as pin:
        while True:
            m = int(round(c * n))
            e = O.gen_hypergraph(n, m, r, 1000 + runs)
            t0 = time.perf_counter()
            res = O.sync_peel(e, n, k)
            dt = time.perf_counter() - t0
            t0 = time.perf_counter()
            O.queue_peel(e, n, k)
            t_queue += time.perf_counter() - t0
            inside = res.core_mask[e].all(axis=1)
            peeled += int(m - inside.sum())
            t_total += dt
            runs += 1
            if t_total > target_s or runs >= 4:
                break
            if dt < target_s / 4:
                n *= 2
    out = {"value": peeled / t_total, "unit": "edges/s", "cores": 1, "kind": "oracle",
           "sample": f"{runs} instance(s) of G^{r}_(n,cn), c={c}, k={k}, largest n={n} "
                     f"(literal synchronous oracle, single thread pinned to core {pin.core}, {t_total:.1f} s of peel)",
           "queue_peel": {"value": peeled / t_queue, "unit": "edges/s", "cores": 1,
                          "kind": "serial queue peel (oracle/peel_oracle.c ora_queue_peel, CSR build included)",
                          "seconds": round(t_queue, 2)}}
    out.update(host_cpu())
    try:
        g = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_goldens.json")))[config]
        if g.get("oracle_seconds"):
            out["full_scale_oracle"] = {
                "value": (g["m"] - g.get("core_edges", 0)) / g["oracle_seconds"] if g.get("core", 0) == 0 else None,
                "unit": "edges/s", "seconds": g["oracle_seconds"],
                "note": "tools/make_oracle_goldens.py on the build host (not this box), whole workload, one core"}
    except Exception:
        pass
    return out


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    kind, n_full, m_full, r, k, seed, text = CONFIGS[args.config]
    c = m_full / n_full
    # each step: one bounded sample instance of the workload (same r, k, c)
    n = 1_000_000 if kind == "kcore" else 1 << 20
    m = int(round(c * n))
    times, units = [], 0
    if kind == "sweep":  # C5s: each step = 2 oracle trials (generation + literal peel) of the grid
        from paper_1302_7014_b200 import trials as S
        n = n_full
        m_all, seeds_all = S.paper_trials(m_full, n=n)
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            for q in range(2):
                j = (2 * i + q) * 97 % m_full
                O.sync_peel(O.gen_hypergraph(n, int(m_all[j]), r, int(seeds_all[j])), n, k)
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
        T = sum(times)
        val = 2 * len(times) / T
        line = {"impl": "reference", "metric": SWEEP_METRIC, "value": val, "unit": "trials/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32/u64 integer",
                "data": "synthetic G^r_{n,cn} trials (oracle generator)",
                "config": {"workload": f"{args.config}: {text}", "trials": m_full},
                "cpu_baseline": {"value": val, "unit": "trials/s", "cores": 1, "kind": "oracle",
                                 "sample": "each step = 2 trials of the C5s grid (n=10^6)"},
                "e2e": {"value": val, "unit": "trials/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        emit(line)
        return 0
    pin = OneCore()
    pin.__enter__()  # single-threaded oracle on one core (released at exit)
    if kind == "kcore":
        e = O.gen_hypergraph(n, m, r, seed)
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = O.sync_peel(e, n, k)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
        inside = res.core_mask[e].all(axis=1)
        per_step = int(m - inside.sum())
        unit = "edges/s"
    else:
        keys = O.gen_keys(m, seed)
        for i in range(args.warmup + args.steps):
            t = O.Iblt(n, r, seed)
            t0 = time.perf_counter()
            t.insert(keys)
            res = t.peel(cap_keys=m + 1)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
        per_step = int(res.keys.size)
        unit = "keys/s"
    T = sum(times)
    val = per_step * len(times) / T
    metric = METRIC if kind == "kcore" else IBLT_METRIC
    line = {
        "impl": "reference", "metric": metric, "value": val, "unit": unit, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32/u64 integer",
        "data": "synthetic (counter-based G^r_{n,cn} generator, oracle implementation)",
        "config": {"workload": f"{args.config}: {text}", "sample_n": n, "sample_m": m, "r": r, "k": k},
        "cpu_baseline": dict({"value": val, "unit": unit, "cores": 1, "kind": "oracle",
                              "sample": f"each step = oracle peel of one n={n} instance of the same model, "
                                        f"pinned to core {pin.core}"}, **host_cpu()),
        "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


def iblt_bytes(C, N, r, nrec):
    """insert 8N + 16C (read keys, RMW cells once); peel 16C (round-1 scan) +
    per recovered key 16 (frontier entry) + 32r (RMW r cells) + 8 (output key)."""
    return 8 * N + 16 * C, 16 * C + nrec * (16 + 32 * r + 8)


def run_iblt_dist(args, pk, dev, ws, rank, local, C, N, r, seed, text, barrier, stream):
    """C2 as ONE table partitioned by cell range over the ranks (iblt_dist_recover; SURVEY
    §8 f3): NCCL under torchrun (--mode dist), or --virtual-shards P on one GPU.  Strong
    scaling: the table and the key set are fixed."""
    import torch
    import torch.distributed as dist
    if args.virtual_shards > 0:
        comm = pk.Comm.virtual_shards(args.virtual_shards)
        P = args.virtual_shards
    else:
        comm = pk.Comm.from_process_group(device=dev)
        P = ws
    keys = pk.gen_keys(N, seed, device=dev)  # the same keys on every rank
    mem = torch.empty((int(pk.lib().iblt_dist_mem_bytes(comm._h, C, r)),), dtype=torch.uint8, device=dev)
    for _ in range(max(args.warmup, 3)):
        res = pk.iblt_dist_recover(comm, C, r, seed, keys, mem=mem)
    clk = ClockSampler(local)
    barrier()
    clk.start()
    pk.profile_enable(True)
    per_kernel, launches = {}, 0
    res = None

    def body(i):
        nonlocal res, launches
        res = pk.iblt_dist_recover(comm, C, r, seed, keys, mem=mem)
        launches += pk.last_launches()
        for name, ms_, nl in pk.profile_read():
            a_ = per_kernel.setdefault(name, [0.0, 0])
            a_[0] += ms_
            a_[1] += nl
    ms_total, l2_note = timed_loop(args.steps, stream, dev, 16 * C // P + 8 * N, body)
    barrier()
    pk.profile_enable(False)
    clocks = clk.stop()
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    tot = torch.tensor([float(res.nrecovered)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot)
    value = tot.item() * args.steps / (t.item() / 1e3)
    # roofline: the whole step per rank against this rank's 1/P share of SURVEY §8 d0's bytes
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs") or 6650.0
    b_ins, b_peel = iblt_bytes(C, N, r, N)
    alg = (b_ins + b_peel) / (1 if args.virtual_shards else P)
    k_ms = sum(v[0] for v in per_kernel.values()) / args.steps
    roof = None
    if k_ms > 0:
        roof = {"bound": "hbm", "kernel": "whole step per rank (all shard kernels)",
                "achieved": round(alg / (k_ms / 1e3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(alg / (k_ms / 1e3) / 1e9 / hbm, 4), "traffic": None,
                "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks.get("hbm_gbs") else
                "fallback (B200_PROFILING.md 6.65 TB/s)", "alg_bytes_per_launch": int(alg),
                "avg_launch_ms": round(k_ms, 4)}
    # e2e through the public call: pinned host keys -> every rank, each rank's recovered keys -> host
    e2e = None
    if not args.no_e2e:
        k_host = torch.empty((N,), dtype=torch.int64, pin_memory=True)
        k_host.copy_(keys)
        o_host = torch.empty((N,), dtype=torch.int64, pin_memory=True)

        def e2e_step():
            keys.copy_(k_host, non_blocking=True)
            rr = pk.iblt_dist_recover(comm, C, r, seed, keys, mem=mem)
            o_host[:rr.keys.numel()].copy_(rr.keys, non_blocking=True)
            return rr
        e2e_step()
        barrier()
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(args.e2e_steps):
            rr = e2e_step()
        h1.record(stream)
        barrier()
        te = torch.tensor([h0.elapsed_time(h1)], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        assert rr.complete
        e2e = {"value": tot.item() * args.e2e_steps / (te.item() / 1e3), "unit": "keys/s",
               "h2d_bytes_per_step": 8 * N * ws, "d2h_bytes_per_step": 8 * N, "steps": args.e2e_steps,
               "api": "iblt_dist_recover (C-ABI); pinned host keys -> every rank, recovered keys -> host"}
    if rank == 0:
        line = {"metric": IBLT_METRIC, "value": value, "unit": "keys/s", "n_gpus": ws, "steps": args.steps,
                "warmup": max(args.warmup, 3), "ms_per_step": round(t.item() / args.steps, 4),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32/u64 integer",
                "data": "synthetic distinct 64-bit keys (SplitMix64 stream on device), replicated on every rank",
                "config": {"workload": f"{args.config}: {text}", "cells": C, "keys": N, "r": r, "seed": seed,
                           "rounds": res.rounds, "complete": res.complete,
                           "parallelism": (f"virtual{P} (1 GPU)" if args.virtual_shards else f"cell-partitioned{P}"),
                           "l2": l2_note},
                "kernels": {nm: {"ms_per_step": round(v[0] / args.steps, 4)} for nm, v in per_kernel.items()},
                "gpu_launches": launches, "clocks": clocks, "roofline": roof, "cpu_baseline": None, "e2e": e2e}
        emit(line)
    del comm
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


def run_iblt(args, pk, dev, ws, rank, local, C, N, r, seed, text, barrier, stream):
    """C2: one step = zero the table + insert N resident keys + round-synchronous recovery."""
    import torch
    import torch.distributed as dist
    keys = pk.gen_keys(N, seed, device=dev)
    mem = torch.empty((int(pk.lib().iblt_mem_bytes(C, r)),), dtype=torch.uint8, device=dev)
    out = torch.empty((N,), dtype=torch.int64, device=dev)
    tb = pk.Iblt(C, r, seed, mem=mem)

    def step():
        tb.reset()
        tb.insert(keys)
        return tb.peel(cap_keys=N, out=out), []

    for _ in range(max(args.warmup, 3)):
        res, _ = step()
    assert res.complete and res.nrecovered == N
    pk.profile_enable(True)
    clk = ClockSampler(local)
    barrier()
    clk.start()
    per_kernel, launches = {}, 0
    res = None

    def body(i):
        nonlocal res, launches
        res, ins = step()
        launches += pk.last_launches()  # insert + peel launches
        for name, ms_, nl in ins + pk.profile_read():
            a = per_kernel.setdefault(name, [0.0, 0])
            a[0] += ms_
            a[1] += nl
    ms_total, l2_note = timed_loop(args.steps, stream, dev, 16 * C + 8 * N, body)
    barrier()
    clocks = clk.stop()
    round_ms = [round(x, 4) for x in pk.profile_rounds()]
    pk.profile_enable(False)
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_keys = float(res.nrecovered) * ws
    value = total_keys * args.steps / (t.item() / 1e3)
    b_ins, b_peel = iblt_bytes(C, N, r, res.nrecovered)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs") or 6650.0
    name, (ms_sum, nl) = max(per_kernel.items(), key=lambda kv: kv[1][0])
    alg = b_peel if "peel" in name else b_ins
    ach = alg / (ms_sum / nl / 1e3) / 1e9
    traffic, tsrc = ncu_traffic(args.config, name)
    roof = {"bound": "hbm", "kernel": name, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(ach / hbm, 4), "traffic": traffic, "traffic_source": tsrc,
            "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks.get("hbm_gbs") else
            "fallback (B200_PROFILING.md 6.65 TB/s)",
            "dram_frac_of_peak": (round(traffic / (ms_sum / nl / 1e3) / 1e9 / hbm, 4) if traffic else None),
            "alg_bytes_per_launch": alg, "avg_launch_ms": round(ms_sum / nl, 4),
            "note": "160 MB table ~ L2-sized: L2-atomic/latency bound, HBM roofline is a loose bound"}
    # e2e through the public API: pinned host keys -> device, insert, recover, recovered keys -> host
    e2e = None
    if not args.no_e2e:
        k_host = torch.empty((N,), dtype=torch.int64, pin_memory=True)
        k_host.copy_(keys)
        o_host = torch.empty((N,), dtype=torch.int64, pin_memory=True)
        k_dev = torch.empty_like(keys)

        def e2e_step():
            k_dev.copy_(k_host, non_blocking=True)
            tb.reset()
            tb.insert(k_dev)
            rr = tb.peel(cap_keys=N, out=out)
            o_host[:rr.nrecovered].copy_(out[:rr.nrecovered], non_blocking=True)
            return rr
        e2e_step()
        barrier()
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(args.e2e_steps):
            rr = e2e_step()
        h1.record(stream)
        barrier()
        te = torch.tensor([h0.elapsed_time(h1)], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        assert rr.complete and rr.nrecovered == N
        e2e = {"value": float(rr.nrecovered) * ws * args.e2e_steps / (te.item() / 1e3), "unit": "keys/s",
               "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * int(rr.nrecovered), "steps": args.e2e_steps,
               "api": "Iblt.reset/insert/peel (C-ABI iblt_insert / iblt_peel), pinned host keys in, recovered keys out"}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        Cs = 1 << 21
        Ns = int(0.75 * Cs)
        ks = O.gen_keys(Ns, seed)
        tt = O.Iblt(Cs, r, seed)
        t0 = time.perf_counter()
        tt.insert(ks)
        rr = tt.peel(cap_keys=Ns + 1)
        dt = time.perf_counter() - t0
        cpu = {"value": rr.keys.size / dt, "unit": "keys/s", "cores": 1, "kind": "oracle",
               "sample": f"oracle insert+recover of 2^21 cells at load 0.75 ({dt:.1f} s)"}
    if rank == 0:
        line = {
            "metric": IBLT_METRIC, "value": value, "unit": "keys/s",
            "n_gpus": ws, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(t.item() / args.steps, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32/u64 integer",
            "data": "synthetic distinct 64-bit keys (SplitMix64 stream on device)",
            "config": {"workload": f"C2: {text}", "cells": C, "keys": N, "r": r, "seed": seed,
                       "rounds": res.rounds, "complete": res.complete,
                       "l2": l2_note + "; each step zeroes the table, re-inserts the keys and recovers them"},
            "paper_context": "Tesla C2070, 2^24 cells, r=3, load 0.75: recovery 0.33 s + insert 0.31 s (P:539)",
            "roofline": roof,
            "kernels": {k: {"ms_per_step": round(v[0] / args.steps, 4)} for k, v in per_kernel.items()},
            "round_ms": round_ms, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        emit(line)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_sweep_bench(args, pk, dev, ws, rank, local, n, T, r, k, text, barrier, stream):
    """C5s: the 10^4-trial sweep over c, sharded by contiguous trial ranges across ranks
    (paper_1302_7014_b200/trials.py).  One step = this rank's whole shard, batch 64."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1302_7014_b200 import trials as S
    m_all, seeds_all = S.paper_trials(T, n=n)
    lo, hi = S.shard(T, ws, rank)
    m, seeds = m_all[lo:hi], seeds_all[lo:hi]
    batch = int(os.environ.get("PEEL_SWEEP_BATCH", "128"))  # r01: 32 / 64 / 128 / 256 / 512 -> 2177 / 1756 / 1547 / 1970 / 2346 ms
    wsb = int(pk.lib().peel_sweep_workspace_bytes(n, int(m_all.max()), r, k, batch))
    wsp = torch.empty((wsb,), dtype=torch.uint8, device=dev)
    for _ in range(max(args.warmup, 3)):
        rounds, core = pk.sweep(n, r, k, m, seeds, batch=batch, ws=wsp)
    clk = ClockSampler(local)
    barrier()
    clk.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    pk.profile_enable(True)
    per_kernel, launches = {}, 0
    e0.record(stream)
    for _ in range(args.steps):
        rounds, core = pk.sweep(n, r, k, m, seeds, batch=batch, ws=wsp)
        launches += pk.last_launches()
        for name, ms_, nl in pk.profile_read():
            a_ = per_kernel.setdefault(name, [0.0, 0])
            a_[0] += ms_
            a_[1] += nl
    e1.record(stream)
    barrier()
    pk.profile_enable(False)
    clocks = clk.stop()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        R, C = S.run_sweep(lambda mm, ss: (rounds, core), m_all, seeds_all, device=dev)
    else:
        R, C = rounds, core
    value = T * args.steps / (t.item() / 1e3)
    if rank == 0:
        j = np.arange(T) // 100
        fail = np.array([(C[j == q] > 0).mean() for q in range(j.max() + 1)])
        cs = 0.700 + 0.002 * np.arange(fail.size)
        cross = float(cs[np.argmax(fail >= 0.5)]) if (fail >= 0.5).any() else None
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            from oracle import oracle as O
            t0 = time.perf_counter()
            for q in range(8):
                O.sync_peel(O.gen_hypergraph(n, int(m_all[q * 1250]), r, int(seeds_all[q * 1250])), n, k)
            dt = time.perf_counter() - t0
            cpu = {"value": 8 / dt, "unit": "trials/s", "cores": 1, "kind": "oracle",
                   "sample": f"8 trials (gen + literal peel) spread over the c grid, {dt:.1f} s"}
        line = {"metric": SWEEP_METRIC, "value": value, "unit": "trials/s", "n_gpus": ws,
                "steps": args.steps, "warmup": max(args.warmup, 3),
                "ms_per_step": round(t.item() / args.steps, 3), "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u32/u64 integer",
                "data": "synthetic G^r_{n,cn} trials (generation on device inside the timed region)",
                "config": {"workload": f"C5s: {text}", "trials": T, "batch": batch,
                           "path": ("per-trial groups (one trial per group of CTAs, 32-bit states in L2, rows "
                                    "regenerated from the seed; sweep.cu)"
                                    if os.environ.get("PEEL_SWEEP_GROUPS", "") != "0" and k == 2 and r <= 4
                                    and n <= (1 << 22) else f"disjoint union of {batch} trials per peel_kcore call"),
                           "parallelism": f"trials sharded over {ws} rank(s)"},
                "result": {"failure_fraction_crosses_half_at_c": cross, "c_star_2_3": 0.818469,
                           "mean_rounds_c0.70": float(R[:100].mean()), "mean_rounds_c0.898": float(R[-100:].mean()),
                           "max_mean_rounds": float(max(R[j == q].mean() for q in range(j.max() + 1)))},
                "kernels": {nm: {"ms_per_step": round(v[0] / args.steps, 3),
                                 "launches_per_step": v[1] / args.steps} for nm, v in per_kernel.items()},
                "gpu_launches": launches,
                # pk.sweep is the public call: it takes the (m_t, seed_t) arrays from the host and
                # returns each trial's rounds and core size to the host, inside the timed region
                "e2e": {"value": value, "unit": "trials/s", "h2d_bytes_per_step": 16 * (hi - lo),
                        "d2h_bytes_per_step": 12 * (hi - lo),
                        "api": "peel_sweep (host trial parameters in, host per-trial results out)"},
                "cpu_baseline": cpu, "clocks": clocks}
        emit(line)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_dist_bench(args, pk, dev, ws, rank, local, n, m, r, k, seed, text, barrier, stream):
    """One instance partitioned by vertex range over the ranks: NCCL under
    torchrun, or --virtual-shards P on one GPU.  Strong scaling: the instance is fixed."""
    import torch
    import torch.distributed as dist
    if args.virtual_shards > 0:
        comm = pk.Comm.virtual_shards(args.virtual_shards)
        P = args.virtual_shards
    else:
        comm = pk.Comm.from_process_group(device=dev)
        P = ws
    edges = pk.gen_hypergraph(n, m, r, seed, device=dev)  # replicated (same seed on every rank)
    need = int(pk.lib().peel_kcore_dist_workspace_bytes(comm._h, n, m, r, k))
    wsp = torch.empty((need,), dtype=torch.uint8, device=dev)
    for _ in range(max(args.warmup, 3)):
        res = pk.peel_kcore_dist(comm, edges, n, k, ws=wsp, cap=4096)
    n_core_local = int(res.core_mask.sum().item())
    clk = ClockSampler(local)
    barrier()
    clk.start()
    pk.profile_enable(True)
    per_kernel, launches = {}, 0

    def body(i):
        nonlocal res, launches
        res = pk.peel_kcore_dist(comm, edges, n, k, ws=wsp, cap=4096)
        launches += pk.last_launches()
        for name, ms_, nl in pk.profile_read():
            a = per_kernel.setdefault(name, [0.0, 0])
            a[0] += ms_
            a[1] += nl
    ms_total, l2_note = timed_loop(args.steps, stream, dev, 4 * r * m + (8 * n + n // 8) // P, body)
    barrier()
    pk.profile_enable(False)
    clocks = clk.stop()
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    cores = torch.tensor([float(n_core_local)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(cores)
    peeled = int(sum(res.killed))
    value = peeled * args.steps / (t.item() / 1e3)
    # roofline: the whole step per rank (the shard kernels have no per-kernel byte formula): this
    # rank's 1/P share of the instance's algorithmic bytes over its kernel time
    roof = None
    n_core_all = int(cores.item())
    if per_kernel and n_core_all == 0:  # m_core = 0 for an empty core; otherwise it needs every slice
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        hbm = peaks.get("hbm_gbs") or 6650.0
        bb, br = algorithmic_bytes(r, n, m, 0, 0, k)
        alg = (bb + br) / (1 if args.virtual_shards else P)  # virtual shards: all P shards on this GPU
        k_ms = sum(v[0] for v in per_kernel.values()) / args.steps
        ach = alg / (k_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": "whole step per rank (all shard kernels)", "achieved": round(ach, 1),
                "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4), "traffic": None,
                "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks.get("hbm_gbs") else
                "fallback (B200_PROFILING.md 6.65 TB/s)",
                "alg_bytes_per_launch": int(alg), "avg_launch_ms": round(k_ms, 4)}
    # e2e through the public call: every rank copies the (replicated) edge list from pinned host
    # memory into its device buffer, peels, and reads its core-mask slice back, per step
    e2e = None
    if not args.no_e2e:
        try:
            e_host = torch.empty((m, r), dtype=torch.int32, pin_memory=True)
            e_host.copy_(edges)
            m_host = torch.empty((res.core_mask.numel(),), dtype=torch.uint8, pin_memory=True)

            def e2e_step():
                edges.copy_(e_host, non_blocking=True)
                rr = pk.peel_kcore_dist(comm, edges, n, k, ws=wsp, cap=4096)
                m_host.copy_(rr.core_mask, non_blocking=True)
                return rr
            e2e_step()
            barrier()
            h0 = torch.cuda.Event(enable_timing=True)
            h1 = torch.cuda.Event(enable_timing=True)
            h0.record(stream)
            for _ in range(args.e2e_steps):
                rr = e2e_step()
            h1.record(stream)
            barrier()
            te = torch.tensor([h0.elapsed_time(h1)], dtype=torch.float64, device=dev)
            if ws > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            assert int(sum(rr.killed)) == peeled
            e2e = {"value": peeled * args.e2e_steps / (te.item() / 1e3), "unit": "edges/s",
                   "h2d_bytes_per_step": 4 * r * m * ws, "d2h_bytes_per_step": n,
                   "steps": args.e2e_steps,
                   "api": "peel_kcore_dist (C-ABI); pinned host edges -> every rank, core-mask slices -> host"}
            del e_host, m_host
        except Exception as ex:  # pragma: no cover
            e2e = {"value": None, "unit": "edges/s", "error": repr(ex)[:200],
                   "h2d_bytes_per_step": 4 * r * m * ws, "d2h_bytes_per_step": n}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": ws, "steps": args.steps,
                "warmup": max(args.warmup, 3), "ms_per_step": round(t.item() / args.steps, 4),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32/u64 integer",
                "data": "synthetic G^r_{n,cn}, edge list replicated on every rank",
                "config": {"workload": f"{args.config}: {text}", "n": n, "m": m, "r": r, "k": k, "seed": seed,
                           "rounds": res.rounds, "core_vertices": int(cores.item()), "peeled_edges": peeled,
                           "parallelism": (f"virtual{P} (1 GPU)" if args.virtual_shards else f"vertex-partitioned{P}"),
                           "l2": l2_note},
                "kernels": {nm: {"ms_per_step": round(v[0] / args.steps, 4)} for nm, v in per_kernel.items()},
                "gpu_launches": launches, "clocks": clocks, "roofline": roof, "cpu_baseline": None, "e2e": e2e}
        emit(line)
    del comm
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


_JSON_OUT = None


def emit(line):
    """The one JSON line, on the real stdout (everything else -- library banners such as NCCL's
    version line -- was redirected to stderr by main())."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # keep fd 1 for the JSON line only: native libraries (NCCL, CUDA) print to fd 1 directly
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="auto", choices=["auto", "replicas", "dist"],
                    help="N>1: 'dist' = one instance vertex-partitioned over the ranks (peel_kcore_dist, "
                         "strong scaling; default for k<=2 configs), 'replicas' = one instance per rank (weak)")
    ap.add_argument("--virtual-shards", type=int, default=0,
                    help="N=1 only: run the partitioned path with P virtual shards on one GPU")
    ap.add_argument("--profile-steps", action="store_true",
                    help="record per-kernel CUDA events inside the timed steps (default on)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1302_7014_b200 as pk

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1 or (args.mode == "dist" and not args.virtual_shards):
        # --mode dist at N=1 runs the NCCL transport with world size 1 (plain or torchrun)
        os.environ.setdefault("NCCL_DEBUG", "WARN")  # no version banner on stdout: one JSON line
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(ws))
        dist.init_process_group("nccl", device_id=dev)
    kind, n, m, r, k, seed, text = CONFIGS[args.config]
    seed = seed + rank  # independent instance per rank (weak scaling)
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    if kind == "iblt":
        if args.virtual_shards > 0 or args.mode == "dist":
            return run_iblt_dist(args, pk, dev, ws, rank, local, n, m, r, seed - rank, text, barrier, stream)
        return run_iblt(args, pk, dev, ws, rank, local, n, m, r, seed, text, barrier, stream)
    if kind == "sweep":
        return run_sweep_bench(args, pk, dev, ws, rank, local, n, m, r, k, text, barrier, stream)
    use_dist = args.virtual_shards > 0 or (k <= 2 and (args.mode == "dist" or (ws > 1 and args.mode == "auto")))
    if use_dist:
        return run_dist_bench(args, pk, dev, ws, rank, local, n, m, r, k, seed - rank, text, barrier, stream)

    edges = pk.gen_hypergraph(n, m, r, seed, device=dev)
    wsb = pk.kcore_workspace_bytes(n, m, r, k)
    wsp = torch.empty((wsb,), dtype=torch.uint8, device=dev)
    mask = torch.empty((n,), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    def step():
        return pk.peel_kcore(edges, n, k, core_mask=mask, ws=wsp, cap=4096)

    for _ in range(max(args.warmup, 3)):
        res = step()
    # results of this instance (deterministic): peeled edges = edges not wholly in the core
    n_core = int(mask.sum().item())
    if n_core:
        inside = mask[edges.long()].all(dim=1)
        m_core = int(inside.sum().item())
        del inside
    else:
        m_core = 0
    peeled = m - m_core
    b_build, b_rounds = algorithmic_bytes(r, n, m, n_core, m_core, k)

    pk.profile_enable(True)
    clk = ClockSampler(local)
    barrier()
    clk.start()
    per_kernel = {}
    launches = 0
    res = None

    def body(i):
        nonlocal res, launches
        res = step()
        launches += pk.last_launches()
        for name, ms, nl in pk.profile_read():
            a = per_kernel.setdefault(name, [0.0, 0])
            a[0] += ms
            a[1] += nl
    ms_total, l2_note = timed_loop(args.steps, stream, dev, 4 * r * m + 8 * n + n // 8, body)
    barrier()
    clocks = clk.stop()
    round_ms = [round(x, 3) for x in pk.profile_rounds()]
    pk.profile_enable(False)
    ms_step = ms_total / args.steps
    t_max = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        tot = torch.tensor([float(peeled)], dtype=torch.float64, device=dev)
        dist.all_reduce(tot)
        total_peeled = tot.item()
    else:
        total_peeled = float(peeled)
    t_max_s = t_max.item() / 1e3
    value = total_peeled * args.steps / t_max_s

    # roofline for the dominant kernel: algorithmic bytes apportioned to the
    # kernels that did the work.  Per round t: 8 |F_t| (state of removed vertices) +
    # killed_t (4r re-read of the edge + 16(r-1) RMW of its other endpoints); the first
    # `nb` rounds run as round_kill_partition (8|F_t| + 4r killed_t) + round_apply
    # (16(r-1) killed_t), the rest in the persistent kernel (+ n for the mask).
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if hbm else "fallback (B200_PROFILING.md 6.65 TB/s)"
    hbm = hbm or 6650.0
    surv = [n] + [int(x) for x in res.survivors]
    F = [surv[i] - surv[i + 1] for i in range(len(surv) - 1)]
    kl = [int(x) for x in res.killed]
    nb = int(round(per_kernel.get("round_kill_partition", [0.0, 0])[1] / args.steps))
    kb = {}
    if k <= 2:
        kb["bin_partition"] = 4 * r * m
        kb["bin_accumulate"] = 8 * n
        kb["build_packed"] = 4 * r * m + 8 * n
        kb["round_kill_partition"] = sum(8 * F[t] + 4 * r * kl[t] for t in range(min(nb, len(F))))
        kb["round_apply"] = sum(16 * (r - 1) * kl[t] for t in range(min(nb, len(F))))
        kb["peel_rounds_packed"] = sum(8 * F[t] + (4 * r + 16 * (r - 1)) * kl[t] for t in range(nb, len(F))) + n
        kb["peel_rounds_cluster"] = kb["peel_rounds_packed"]
        kb["compact_core_mask"] = n  # the mask of the compacted path (no persistent tail)
        kb["compact_slots"] = 0      # compaction moves no compulsory bytes
    dom = max(per_kernel.items(), key=lambda kv: kv[1][0]) if per_kernel else None
    roof = None
    if dom:
        name, (ms_sum, nl) = dom
        if name in ("round_kill_partition", "round_apply") and res.rounds:
            # the compacted rounds' device-side loop launches 4 rounds per host sync; the launches
            # after the loop stopped exit at once: per-launch figures count the rounds that ran
            nl = min(nl, args.steps * int(res.rounds))
        avg_ms = ms_sum / max(nl, 1)
        alg = kb.get(name)  # bytes per STEP of this kernel (all its launches)
        if alg is None:  # CSR path / graph replay: whole-step formula over the whole-step time of its kernels
            alg = b_build + b_rounds
            avg_ms = sum(v[0] for v in per_kernel.values()) / args.steps
            ds = dram_step(args.config, per_kernel, args.steps, avg_ms, hbm)
            traffic, tsrc = ((ds["bytes"], ds["source"] + ", whole step") if ds and not ds["kernels_without_traffic"]
                             else (None, None))
        else:
            alg = alg / max(nl / args.steps, 1.0)  # per launch, like avg_ms
            traffic, tsrc = ncu_traffic(args.config, name, int(res.rounds))
        ach = alg / (avg_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": name, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 4), "traffic": traffic, "traffic_source": tsrc, "peak_source": peak_src,
                # the same kernel's real DRAM bytes (ncu) over its time here: random 8-12 B accesses move
                # 64 B DRAM granules, so traffic >> algorithmic bytes by construction
                "dram_frac_of_peak": (round(traffic / (avg_ms / 1e3) / 1e9 / hbm, 4) if traffic else None),
                "alg_bytes_per_launch": int(alg), "avg_launch_ms": round(avg_ms, 4)}
    step_alg = b_build + b_rounds
    kernels = {nm: {"ms_per_step": round(v[0] / args.steps, 4), "launches_per_step": v[1] / args.steps}
               for nm, v in per_kernel.items()}

    # e2e: through the C-ABI with HOST buffers (H2D of the edges + D2H of the mask inside)
    e2e = None
    if not args.no_e2e:
        try:
            e_host = torch.empty((m, r), dtype=torch.int32, pin_memory=True)
            e_host.copy_(edges)
            m_host = torch.empty((n,), dtype=torch.uint8, pin_memory=True)
            hws = torch.empty((int(pk.lib().peel_kcore_host_workspace_bytes(n, m, r, k, 0)),),
                              dtype=torch.uint8, device=dev)
            del wsp
            torch.cuda.empty_cache()
            pk.peel_kcore_host(e_host, n, k, core_mask_host=m_host, ws=hws, cap=4096)  # warm-up
            barrier()
            h0 = torch.cuda.Event(enable_timing=True)
            h1 = torch.cuda.Event(enable_timing=True)
            h0.record(stream)
            for _ in range(args.e2e_steps):
                pk.peel_kcore_host(e_host, n, k, core_mask_host=m_host, ws=hws, cap=4096)
            h1.record(stream)
            barrier()
            te = torch.tensor([h0.elapsed_time(h1)], dtype=torch.float64, device=dev)
            if ws > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            assert int(m_host.sum().item()) == n_core
            # the mask comes back by 64 chunks, only those holding a core vertex (the host buffer
            # is zeroed by host threads while the GPU peels), plus the 64 chunk flags
            d2h = 256
            if n > (1 << 23):
                chunk = (((n + 63) // 64) + 15) & ~15
                for c in range(64):
                    lo = c * chunk
                    if lo < n and bool(m_host[lo:min(n, lo + chunk)].any()):
                        d2h += min(chunk, n - lo)
            else:
                d2h = n
            e2e = {"value": total_peeled * args.e2e_steps / (te.item() / 1e3), "unit": "edges/s",
                   "h2d_bytes_per_step": 4 * r * m, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
                   "api": "peel_kcore_host (C-ABI, pinned host edges in, host core mask out: the mask "
                          "chunks that hold a core vertex are copied, the rest zeroed on the host)"}
            del hws, e_host, m_host
        except Exception as ex:  # pragma: no cover
            e2e = {"value": None, "unit": "edges/s", "error": repr(ex)[:200],
                   "h2d_bytes_per_step": 4 * r * m, "d2h_bytes_per_step": n}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_kcore(r, k, m / n, config=args.config)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(t_max_s * 1e3 / args.steps, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32/u64 integer",
            "data": "synthetic G^r_{n,cn} (counter-based Philox generator on device, seed per rank)",
            "config": {"workload": f"{args.config}: {text}", "n": n, "m": m, "r": r, "k": k, "seed": seed - rank,
                       "rounds": res.rounds, "core_vertices": n_core, "peeled_edges": peeled,
                       "parallelism": f"replicas{ws}" if ws > 1 else "single",
                       "l2": l2_note},
            "rounds": res.rounds,
            "hbm_roofline_step": {"alg_bytes": step_alg, "frac_of_measured": round(step_alg / (ms_step / 1e3) / 1e9 / hbm, 4),
                                  "frac_of_8TBs": round(step_alg / (ms_step / 1e3) / 8e12, 4)},
            "dram_step": dram_step(args.config, per_kernel, args.steps, ms_step, hbm),
            "roofline": roof, "kernels": kernels, "round_ms": round_ms,
            "kernel_alg_bytes": kb, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks,
        }
        emit(line)
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
