"""One rank of a multi-process run of the partitioned calls over the HOST transport
(peel.h peel_comm_init_host, torch.distributed gloo): several ranks share one GPU, which
is safe because no kernel waits on another rank.  Launched by tests/test_gpu_multirank.py;
writes its results to --out (npz).  Not a test module itself."""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1302_7014_b200 as pk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--port", type=int, required=True)
    ap.add_argument("--case", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--r", type=int, default=3)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--blog", type=int, default=0)
    ap.add_argument("--cells", default="")
    ap.add_argument("--shrink_ws_rank", type=int, default=-1)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{a.port}", rank=a.rank, world_size=a.world)
    comm = pk.Comm.host_transport()
    out = {"rank": a.rank}
    try:
        if a.case == "kcore":
            e = pk.gen_hypergraph(a.n, a.m, a.r, a.seed, device=dev)
            ws = None
            if a.shrink_ws_rank == a.rank:
                need = int(pk.lib().peel_kcore_dist_workspace_bytes(comm._h, a.n, a.m, a.r, 2))
                ws = torch.empty((need - 1,), dtype=torch.uint8, device=dev)
            try:
                res = pk.peel_kcore_dist(comm, e, a.n, 2, ws=ws)
                out.update(status=res.status, rounds=res.rounds, survivors=res.survivors, killed=res.killed,
                           mask=res.core_mask.cpu().numpy())
            except pk.PeelError as err:
                out.update(status=err.status)
        elif a.case == "iblt":
            keys = pk.gen_keys(a.m, a.seed, device=dev)
            try:
                res = pk.iblt_dist_recover(comm, a.n, a.r, a.seed, keys, blog=a.blog)
                out.update(status=res.status, rounds=res.rounds, per_round=res.per_round,
                           complete=res.complete, keys=res.keys.cpu().numpy().view(np.uint64))
            except pk.PeelError as err:
                out.update(status=err.status)
        elif a.case == "iblt_cells":
            cells = torch.from_numpy(np.load(a.cells)).to(dev)
            try:
                res = pk.iblt_dist_recover_cells(comm, cells, a.r, a.seed, blog=a.blog)
                out.update(status=res.status, rounds=res.rounds, per_round=res.per_round,
                           complete=res.complete, keys=res.keys.cpu().numpy().view(np.uint64))
            except pk.PeelError as err:
                out.update(status=err.status)
        else:
            raise SystemExit(f"unknown case {a.case}")
    finally:
        np.savez(a.out, **{k: np.asarray(v) for k, v in out.items()})
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
