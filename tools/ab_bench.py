#!/usr/bin/env python
"""A/B of library builds in ONE GPU session (box-to-box spread is ~3 %, so
variants are only compared within a call): runs the bench step with each
libamsim build (AMSIM_LIB), interleaved over several rounds, and prints the
per-kind and total ms per step of each.

    python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so base=build/variants/libamsim_base.so [--rounds 2]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+", help="name=path")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--args", default="--steps 5 --warmup 3")
    a = ap.parse_args()
    res = {}
    for r in range(a.rounds):
        for spec in a.libs:
            name, path = spec.split("=", 1)
            env = dict(os.environ, AMSIM_LIB=os.path.join(ROOT, path))
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), *a.args.split(), "--no-full-step", "--no-cpu-baseline",
                   "--no-e2e", "--no-exact-step"]
            out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT)
            line = [l for l in out.stdout.splitlines() if l.startswith("{")]
            if not line:
                print(name, "failed", out.stderr[-500:], flush=True)
                continue
            d = json.loads(line[0])
            k = d["roofline"]["per_kind_ms_per_step"]
            res.setdefault(name, []).append((d["ms_per_step"], k))
            print(json.dumps({"round": r, "lib": name, "ms": d["ms_per_step"], "kinds": k}), flush=True)
    for name, v in res.items():
        print(json.dumps({"lib": name, "median_ms": statistics.median(x[0] for x in v),
                          "kinds": {kk: statistics.median(x[1][kk] for x in v) for kk in v[0][1]}}), flush=True)


if __name__ == "__main__":
    main()
