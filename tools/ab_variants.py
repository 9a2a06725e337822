"""A/B: build libpeel variants with extra -D defines and time one bench config with each
(PEEL_LIB selects the library), printing ms/step and the per-kernel split.

  python tools/ab_variants.py --config C5 --steps 3 base: spec0:PEEL_KILL_SPEC=0 ...
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--build-only", action="store_true")
ap.add_argument("--prebuilt", action="store_true", help="use variants/libpeel_<name>.so as built")
ap.add_argument("--env", default="", help="extra NAME=VALUE,... for every run")
ap.add_argument("--extra", default="", help="extra bench.py arguments, e.g. '--virtual-shards 8'")
ap.add_argument("variants", nargs="+", help="name:DEF=V,DEF=V (name: alone = the default build)")
a = ap.parse_args()
from paper_1302_7014_b200 import build as B  # noqa: E402

os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
libs = {}
for v in a.variants:
    name, _, defs = v.partition(":")
    out = os.path.join(ROOT, "variants", f"libpeel_{name}.so")
    if not a.prebuilt:
        B.build(force=True, out=out, defines=[d for d in defs.split(",") if d])
    libs[name] = out
if a.build_only:
    sys.exit(0)
for name, lib in libs.items():
    env = dict(os.environ, PEEL_LIB=lib)
    for kv in filter(None, a.env.split(",")):
        k, _, val = kv.partition("=")
        env[k] = val
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", a.config, "--steps", str(a.steps),
                        "--warmup", str(a.warmup), "--no-e2e", "--no-cpu-baseline", *a.extra.split()], env=env,
                       capture_output=True,
                       text=True, timeout=900)
    line = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    if not line:
        print(name, "FAILED", p.stdout[-500:], p.stderr[-1500:])
        continue
    d = json.loads(line[-1])
    ks = {k: round(v["ms_per_step"], 2) for k, v in d.get("kernels", {}).items()}
    print(json.dumps({"variant": name, "ms_per_step": d["ms_per_step"], "kernels": ks}))
