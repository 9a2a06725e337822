"""Write tests/golden/oracle_goldens.json: the full-size results of every bench config as the
ORACLE computes them (oracle/ only -- nothing here touches the CUDA path).

The full-scale GPU tests compare against this file.  tests/test_oracle_goldens.py checks on
CPU that it agrees, field for field, with the independent implementation's goldens that
SURVEY.md §8 c3 quotes (tests/golden/survey_c3_goldens.json).  That comparison pins the oracle
at full scale.

    python tools/make_oracle_goldens.py [CONFIG ...]   # default: all; C5 takes minutes, ~25 GB RAM
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_goldens.json")

# (n, m, r, k, seed): BASELINE.json configs / SURVEY §8 (a); reduced C4 as in SURVEY §8 c3
KCORE = {
    "C1": (100_000, 70_000, 3, 2, 1),
    "C4a_small": (1_000_000, 850_000, 3, 2, 4),
    "C4b_small": (1_000_000, 1_600_000, 3, 3, 5),
    "C3": (100_000_000, 75_000_000, 4, 2, 3),
    "C4a": (100_000_000, 85_000_000, 3, 2, 4),
    "C4b": (100_000_000, 160_000_000, 3, 3, 5),
    "C5": (1_000_000_000, 750_000_000, 3, 2, 6),
}
IBLT = {"C2": (10_000_000, 7_500_000, 3, 2)}  # cells, keys, r, seed


def kcore(name):
    n, m, r, k, seed = KCORE[name]
    t0 = time.time()
    e = O.gen_hypergraph(n, m, r, seed)
    sha = hashlib.sha256(e.tobytes()).hexdigest()
    head = e[:2].tolist()
    res = O.sync_peel(e, n, k)
    out = {"n": n, "m": m, "r": r, "k": k, "seed": seed, "edges_head": head, "sha256": sha,
           "rounds": int(res.rounds), "core": int(res.core_mask.sum()),
           "survivors": [int(x) for x in res.survivors], "killed": [int(x) for x in res.killed],
           "oracle_seconds": round(time.time() - t0, 1)}
    del e, res
    return out


def iblt(name):
    C, N, r, seed = IBLT[name]
    t0 = time.time()
    keys = O.gen_keys(N, seed)
    t = O.Iblt(C, r, seed)
    t.insert(keys)
    res = t.peel(cap_keys=N + 1)
    return {"cells": C, "nkeys": N, "r": r, "seed": seed,
            "sorted_keys_sha256": hashlib.sha256(np.sort(res.keys).tobytes()).hexdigest(),
            "rounds": int(res.rounds), "complete": bool(res.complete),
            "per_round": [int(x) for x in res.per_round], "oracle_seconds": round(time.time() - t0, 1)}


def main(argv):
    names = argv or list(KCORE) + list(IBLT)
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data["_source"] = ("tools/make_oracle_goldens.py: oracle/ only (ora_gen_hypergraph + ora_sync_peel; "
                       "ora_gen_keys + ora_iblt insert/peel). survivors[t-1] = alive vertices after round t; "
                       "killed[t-1] = edges killed in round t.")
    for nm in names:
        data[nm] = iblt(nm) if nm in IBLT else kcore(nm)
        print(nm, data[nm].get("rounds"), data[nm].get("oracle_seconds"), "s", flush=True)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
            f.write("\n")


if __name__ == "__main__":
    main(sys.argv[1:])
