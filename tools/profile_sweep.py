"""One C5s sweep call (10^4 trials, n = 10^6, r = 3, k = 2, the paper's c grid) for ncu
captures: python tools/profile_sweep.py [--trials T]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--trials", type=int, default=10_000)
ap.add_argument("--n", type=int, default=1_000_000)
a = ap.parse_args()

import torch  # noqa: E402

import paper_1302_7014_b200 as pk  # noqa: E402
from paper_1302_7014_b200 import trials as S  # noqa: E402

dev = torch.device("cuda:0")
m, seeds = S.paper_trials(a.trials, n=a.n)
rounds, core = pk.sweep(a.n, 3, 2, m, seeds, batch=128, device=dev)
torch.cuda.synchronize()
print("trials", a.trials, "mean rounds", float(rounds.mean()), "failed", int((core > 0).sum()))
