"""Blocked (locality-aware) IBLT hashing vs the plain hash (the paper's open question,
P:706-708; R27): (1) recovery success near the threshold c*_{2,3} = 0.818 as a
function of the block size, (2) insert + recovery time at the C2 shape.

  python tools/blocked_iblt.py [--trials 40] > profiles/r01_blocked_iblt.md
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1302_7014_b200 as pk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--trials", type=int, default=40)
a = ap.parse_args()
dev = torch.device("cuda:0")
r = 3
print("# Blocked IBLT hashing (P:706-708), B200\n")
print("## Recovery success near the threshold (r = 3, C = 2^22 cells, %d trials per cell)\n" % a.trials)
C = 1 << 22
loads = [0.78, 0.80, 0.81, 0.815, 0.82, 0.83]
blogs = [0, 8, 10, 12, 14, 16, 18, 20]
print("| block (cells) | " + " | ".join("load %.3f" % l for l in loads) + " |")
print("|---|" + "---|" * len(loads))
mem = torch.empty((int(pk.lib().iblt_mem_bytes(C, r)),), dtype=torch.uint8, device=dev)
out = torch.empty((C,), dtype=torch.int64, device=dev)
for blog in blogs:
    row = []
    for load in loads:
        N = int(load * C)
        ok = 0
        for t in range(a.trials):
            keys = pk.gen_keys(N, 1000 * blog + t, device=dev)
            tb = pk.Iblt(C, r, 77 + t, mem=mem, blog=blog)
            tb.insert(keys)
            ok += tb.peel(cap_keys=C, out=out).complete
        row.append("%.3f" % (ok / a.trials))
    print("| %s | " % ("plain" if blog == 0 else "2^%d" % blog) + " | ".join(row) + " |", flush=True)

print("\n## Time at the C2 shape (r = 3, C = 10·2^20 cells, load 0.75; median of 20)\n")
print("| block (cells) | insert ms | recovery ms | rounds | recovered |")
print("|---|---|---|---|---|")
C = 10 << 20
N = int(0.75 * C)
keys = pk.gen_keys(N, 2, device=dev)
mem = torch.empty((int(pk.lib().iblt_mem_bytes(C, r)),), dtype=torch.uint8, device=dev)
out = torch.empty((N,), dtype=torch.int64, device=dev)
for blog in [0, 12, 14, 16, 18, 20]:
    ti, tp = [], []
    for it in range(23):
        tb = pk.Iblt(C, r, 2, mem=mem, blog=blog)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        tb.insert(keys)
        e1.record()
        res = tb.peel(cap_keys=N, out=out)
        e2.record()
        torch.cuda.synchronize()
        if it >= 3:
            ti.append(e0.elapsed_time(e1))
            tp.append(e1.elapsed_time(e2))
    print("| %s | %.3f | %.3f | %d | %d |" % ("plain" if blog == 0 else "2^%d" % blog, np.median(ti), np.median(tp),
                                              res.rounds, res.nrecovered), flush=True)
