#!/usr/bin/env python
"""Summarise an ncu launch list of `bench.py --steps 1 --warmup 1`
(`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv`):
the launches of the timed step (the second of the two identical steps), per
kernel kind -- launches, device time, share, DRAM bytes per launch -- and,
with --traffic-json, the per-kind DRAM traffic per layer pass next to the
algorithmic bytes 4(|X| + |W| + |Y|) of the ResNet-50 b256 passes, for
bench.py's roofline "traffic" field.

    python tools/summarize_launches.py gpurun_out/launches.csv [--traffic-json profiles/r01_traffic.json]
"""
import argparse
import collections
import csv
import io
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

LOADERS = [("FwdX", "conv_fwd"), ("WgX", "conv_wgrad"), ("DgDY", "conv_dgrad"), ("GemmOp, amsim::dev::GemmOp", "dense")]


def kind_of(name):
    if "amsim_mm_kernel" in name or "splitk_reduce_kernel" in name:
        for tag, label in LOADERS:
            if tag in name:
                return label + (" (split-K reduce)" if "splitk" in name else "")
        return "amsim other"
    return name.split("(")[0].replace("void ", "").split("<")[0]


def load(path):
    text = open(path).read()
    text = text[text.index('"ID"'):]
    launches = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO(text)):
        d = launches.setdefault(int(r["ID"]), {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["ns"] = v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        elif r["Metric Name"].startswith("dram__bytes"):
            d["dram"] = d.get("dram", 0.0) + v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return list(launches.values())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--traffic-json")
    args = ap.parse_args()
    rows = load(args.csv)
    am_idx = [i for i, r in enumerate(rows) if "amsim_mm_kernel" in r["name"] or "splitk_reduce" in r["name"]]
    half = len(am_idx) // 2
    step = rows[am_idx[half]:am_idx[-1] + 1] if half else rows
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in step:
        k = kind_of(r["name"])
        agg[k][0] += 1
        agg[k][1] += r.get("ns", 0.0)
        agg[k][2] += r.get("dram", 0.0)
    tot = sum(v[1] for v in agg.values())
    out = [f"timed step = launches {am_idx[half] if half else 0}..{am_idx[-1]} of {len(rows)} in the list "
           f"(second of two identical steps); ncu times are cold-cache and serialised: compare shares",
           f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'DRAM MB/launch':>15s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k:40s} {v[0]:8d} {v[1] / 1e6:10.2f} {v[1] / tot:7.1%} {v[2] / max(v[0], 1) / 1e6:15.1f}")
    out.append(f"{'total':40s} {len(step):8d} {tot / 1e6:10.2f}")
    print("\n".join(out))

    if args.traffic_json:
        import amsim_inputs as inp
        layers = inp.resnet50_layers(256)
        alg = collections.defaultdict(list)
        for l in layers:
            if hasattr(l, "H"):
                xb, wb, yb = l.N * l.H * l.W * l.C, l.R * l.S * l.C * l.K, l.N * l.OH * l.OW * l.K
                alg["conv_fwd"].append(4 * (xb + wb + yb))
                alg["conv_wgrad"].append(4 * (xb + yb + wb))
                if not l.first:
                    alg["conv_dgrad"].append(4 * (yb + wb + xb))
        res = {}
        for kind in ("conv_fwd", "conv_wgrad", "conv_dgrad"):
            n = agg[kind][0]
            dram = agg[kind][2] + agg[kind + " (split-K reduce)"][2]
            passes = len(alg[kind])
            res[kind] = {"layer_passes": passes, "mm_launches": n,
                         "dram_bytes_per_pass": dram / passes, "algorithmic_bytes_per_pass": sum(alg[kind]) / passes,
                         "ratio": dram / sum(alg[kind])}
        res["source"] = os.path.basename(args.csv) + " (ncu dram__bytes_read.sum + dram__bytes_write.sum, timed step)"
        json.dump(res, open(args.traffic_json, "w"), indent=1)
        print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
