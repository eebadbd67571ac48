#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel (amsim_mm_kernel split by operand loader), launches, total device
time and share.  Usage: python tools/summarize_launches.py gpurun_out/launches.csv
"""
import collections
import csv
import io
import sys

LOADERS = [("FwdX", "conv fwd"), ("WgX", "conv wgrad"), ("DgDY", "conv dgrad"), ("GemmOp, amsim::dev::GemmOp", "gemm")]


def main(path):
    text = open(path).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r["Kernel Name"]
        key = name.split("(")[0].replace("void ", "").split("<")[0]
        if "amsim_mm_kernel" in name:
            for tag, label in LOADERS:
                if tag in name:
                    key = f"amsim_mm_kernel [{label}]"
                    break
        agg[key][0] += 1
        agg[key][1] += float(r["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k:40s} {v[0]:8d} {v[1] / 1e6:10.2f} {v[1] / tot:7.1%}")
    out.append(f"{'total':40s} {len(rows):8d} {tot / 1e6:10.2f}")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
