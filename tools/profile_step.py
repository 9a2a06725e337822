"""One peel_kcore call on a synthetic G^r_{n,cn} instance (for ncu / compute-sanitizer).

  python tools/profile_step.py --n 100000000 --c 0.75 --r 3 --k 2 --seed 6 [--warm 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1302_7014_b200 as pk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--c", type=float, default=0.75)
ap.add_argument("--r", type=int, default=3)
ap.add_argument("--k", type=int, default=2)
ap.add_argument("--seed", type=int, default=6)
ap.add_argument("--warm", type=int, default=1)
ap.add_argument("--iblt", action="store_true", help="IBLT insert+peel instead (n = cells, c = load)")
a = ap.parse_args()
dev = torch.device("cuda:0")
if a.iblt:
    nk = int(round(a.c * a.n))
    keys = pk.gen_keys(nk, a.seed, device=dev)
    for _ in range(a.warm + 1):
        t = pk.Iblt(a.n, a.r, a.seed, device=dev)
        t.insert(keys)
        res = t.peel(cap_keys=nk)
    print(f"iblt rounds={res.rounds} recovered={res.nrecovered} complete={res.complete}")
else:
    m = int(round(a.c * a.n))
    e = pk.gen_hypergraph(a.n, m, a.r, a.seed, device=dev)
    for _ in range(a.warm + 1):
        res = pk.peel_kcore(e, a.n, a.k)
    print(f"kcore rounds={res.rounds} survivors_last={res.survivors[-1] if len(res.survivors) else None}")
torch.cuda.synchronize()
