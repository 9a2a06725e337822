"""Summarise an ncu launch list taken with
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv
into per-kernel DRAM traffic per launch (the `traffic` field of bench.py's roofline).
Only the launches of the LAST step are kept: bench.py --steps 1 --warmup W runs W+1
identical peels, so the last len/(W+1) launches of each kernel are one step.

  python tools/ncu_traffic.py gpurun_out/traffic_C5.csv --steps 4 > profiles/r01_traffic_C5.json
"""
import argparse
import csv
import json
import re
import collections


def short(name: str) -> str:
    m = re.search(r"(?:peel::)?([A-Za-z_0-9]+)(?:<[^>]*>)?\(", name)
    base = m.group(1) if m else name
    return base.replace("_kernel", "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--steps", type=int, default=4, help="identical peels in the run (warm-ups + timed)")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
    h = rows[0]
    iid, iname, imet, ival = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    iunit = h.index("Metric Unit")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = per.setdefault(int(r[iid]), {"kernel": short(r[iname])})
        d[r[imet]] = float(r[ival].replace(",", "")) * scale[r[iunit]]  # bytes; durations in ms
    by = collections.defaultdict(list)
    for d in per.values():
        by[d["kernel"]].append(d)
    out = {}
    for k, L in by.items():
        n = max(1, len(L) // a.steps) if len(L) >= a.steps else len(L)
        last = L[-n:]
        rd = sum(x.get("dram__bytes_read.sum", 0) for x in last)
        wr = sum(x.get("dram__bytes_write.sum", 0) for x in last)
        ms = sum(x.get("gpu__time_duration.sum", 0) for x in last)
        out[k] = {"launches_per_step": n, "dram_read_bytes_per_step": rd, "dram_write_bytes_per_step": wr,
                  "traffic_per_launch": (rd + wr) / n, "ncu_ms_per_step": ms}
    print(json.dumps({"source": a.csv, "method": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                      "gpu__time_duration.sum --clock-control none (single pass, no replay)", "kernels": out},
                     indent=1))


if __name__ == "__main__":
    main()
