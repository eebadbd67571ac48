#!/usr/bin/env python
"""Per-layer-pass throughput of the bench's training step (one B200).

Runs the bench's TrainStep (ResNet-50 b256 by default), times every C-ABI
launch with CUDA events on the launching stream, and prints one JSON line per
layer pass (name, pass, GEMM shape, ms, T approx-MAC/s, share of the step),
sorted by the time lost against the step's best rate -- where the next
optimisation pays.  With AMSIM_DEBUG_PLAN=1 the library also logs each plan.

    python tools/layer_table.py [--workload resnet50] [--model mbm] [--m 7] [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50", choices=["resnet50", "resnet18", "lenet5"])
    ap.add_argument("--model", default="mbm")
    ap.add_argument("--m", type=int, default=7)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (default: the workload's global batch)")
    args = ap.parse_args()

    import torch

    import amsim_inputs as inp
    import paper_2209_04161_b200 as am
    from paper_2209_04161_b200.train_step import TrainStep

    batch = args.batch or {"resnet50": 256, "resnet18": 128, "lenet5": 64}[args.workload]
    layers = {"resnet50": inp.resnet50_layers, "resnet18": inp.resnet18_cifar_layers,
              "lenet5": inp.lenet5_layers}[args.workload](batch)
    lut = am.Lut.build(args.model, args.m)
    step = TrainStep(layers, lut, seed=1000)
    step.step()
    torch.cuda.synchronize()
    # launch order of TrainStep: forward of every layer, then in reverse wgrad (+ dgrad unless first)
    names = [(l.name, "fwd", l) for l in layers]
    for l in layers[::-1]:
        names.append((l.name, "wgrad", l))
        if not l.first:
            names.append((l.name, "dgrad", l))
    acc = [0.0] * len(names)
    for _ in range(args.reps):
        step.timers = []
        step.step()
        torch.cuda.synchronize()
        assert len(step.timers) == len(names)
        for i, (_, _, a, b) in enumerate(step.timers):
            acc[i] += a.elapsed_time(b) / args.reps
    total = sum(acc)
    rows = []
    for (name, pss, l), ms in zip(names, acc):
        macs = l.macs()
        if hasattr(l, "H"):
            shape = {"fwd": (l.N * l.OH * l.OW, l.K, l.R * l.S * l.C), "wgrad": (l.R * l.S * l.C, l.K, l.N * l.OH * l.OW),
                     "dgrad": (l.N * l.H * l.W, l.C, l.R * l.S * l.K)}[pss]
        else:
            shape = {"fwd": (l.N, l.OUT, l.IN), "wgrad": (l.IN, l.OUT, l.N), "dgrad": (l.N, l.IN, l.OUT)}[pss]
        rows.append({"layer": name, "pass": pss, "MNK": shape, "ms": ms, "tmacs": macs / (ms * 1e-3) / 1e12,
                     "share": ms / total})
    best = max(r["tmacs"] for r in rows if r["ms"] > 1.0)
    for r in rows:
        r["lost_ms"] = r["ms"] - r["ms"] * r["tmacs"] / best
    rows.sort(key=lambda r: -r["lost_ms"])
    print(json.dumps({"batch": batch, "total_ms": total, "tmacs": sum(l.macs() for _, _, l in names) / (total * 1e-3) / 1e12, "best_tmacs": best, "lost_ms": sum(r["lost_ms"] for r in rows)}))
    for r in rows[:args.top]:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
