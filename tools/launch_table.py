"""Print an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) as one line per launch and per-kernel totals.

  python tools/launch_table.py gpurun_out/launches_c5.csv [--totals]
"""
import argparse
import collections
import csv
import re

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--totals", action="store_true")
a = ap.parse_args()
rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
h = rows[0]
iid, iname, imet, ival, iu = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
         "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
per = collections.OrderedDict()
for r in rows[1:]:
    d = per.setdefault(int(r[iid]), {"k": re.sub(r"\(.*", "", r[iname]).replace("void ", "")[:44]})
    d[r[imet]] = float(r[ival].replace(",", "")) * scale.get(r[iu], 1.0)
tot = collections.OrderedDict()
for i, d in per.items():
    ms, rd, wr = d.get("gpu__time_duration.sum", 0), d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
    t = tot.setdefault(re.sub(r"<.*", "", d["k"]), [0, 0.0, 0.0, 0.0])
    t[0] += 1; t[1] += ms; t[2] += rd; t[3] += wr
    if not a.totals:
        print(f"{i:4d} {d['k']:44s} {ms:8.3f} ms  R {rd / 1e9:7.2f} GB  W {wr / 1e9:7.2f} GB")
print("--- totals")
S = [0, 0.0, 0.0, 0.0]
for k, t in tot.items():
    print(f"{k:40s} n={t[0]:3d} {t[1]:8.3f} ms  R {t[2] / 1e9:7.2f} GB  W {t[3] / 1e9:7.2f} GB")
    S = [x + y for x, y in zip(S, t)]
print(f"{'ALL':40s} n={S[0]:3d} {S[1]:8.3f} ms  R {S[2] / 1e9:7.2f} GB  W {S[3] / 1e9:7.2f} GB")
