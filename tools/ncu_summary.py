"""Summarise an `ncu --set full` report: per profiled launch, duration, DRAM traffic, L2
atomic/reduction sectors, sectors per request, occupancy and the top stall reasons.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "ms",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sectors_op_atom.sum": "l2_atom_sectors",
    "lts__t_sectors_op_red.sum": "l2_red_sectors",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "ld_sectors",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum": "ld_requests",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_atom.sum": "atom_sectors",
    "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum": "atom_requests",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum": "red_sectors",
    "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum": "red_requests",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
        "ns": 1e-6, "us": 1e-3, "ms": 1.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--json")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[head.index("Kernel Name")].split("(")[0].replace("void ", "")}
        stalls = {}
        for i, name in enumerate(head):
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            if name in KEYS:
                d[KEYS[name]] = v * UNIT.get(units[i], 1.0)
            elif name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued"):
                stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v
        tot = sum(stalls.values()) or 1.0
        d["stall_top"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        for s_, q in (("ld_sectors", "ld_requests"), ("atom_sectors", "atom_requests"), ("red_sectors", "red_requests")):
            if d.get(q):
                d[s_.split("_")[0] + "_sectors_per_request"] = round(d[s_] / d[q], 2)
        out.append(d)
    for d in out:
        print(json.dumps(d))
    if a.json:
        json.dump(out, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
