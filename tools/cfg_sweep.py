#!/usr/bin/env python
"""Tile-configuration sweep over the distinct layer passes of a training step.

For every distinct (shape, pass) of the workload, time the planner's own
choice and every forced configuration (AMSIM_FORCE_CFG: 0..5 normal
orientation, 10 + cfg transposed; part of the plan-cache key), median of
--reps CUDA-event timings after a warm-up.  One JSON line per pass with the
multiplicity in the step, then a summary: step time at the planner's choices
vs at the per-pass best -- what a better cost model could recover.

    python tools/cfg_sweep.py [--workload resnet50] [--model mbm] [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CFGS = ["auto", "0", "1", "2", "3", "4", "5", "6", "7", "12", "14", "15", "16", "18", "19", "20"]
NAMES = {"0": "Small", "1": "Mid", "2": "Big", "3": "Lean", "4": "Wide", "5": "Huge",
         "6": "Flat", "7": "Tall",
         "12": "Big^T", "14": "Wide^T", "15": "Huge^T", "16": "Flat^T", "18": "Flat3^T", "19": "TallT^T", "20": "Flat8^T", "auto": "auto"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50", choices=["resnet50", "resnet18", "lenet5"])
    ap.add_argument("--model", default="mbm")
    ap.add_argument("--m", type=int, default=7)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (default: the workload's global batch)")
    args = ap.parse_args()

    import torch

    import amsim_inputs as inp
    from amsim_inputs import device as gen
    import paper_2209_04161_b200 as am

    batch = args.batch or {"resnet50": 256, "resnet18": 128, "lenet5": 64}[args.workload]
    layers = {"resnet50": inp.resnet50_layers, "resnet18": inp.resnet18_cifar_layers,
              "lenet5": inp.lenet5_layers}[args.workload](batch)
    lut = am.Lut.build(args.model, args.m)
    groups = {}
    for l in layers:
        if not hasattr(l, "H"):
            continue
        key = (l.N, l.H, l.W, l.C, l.K, l.R, l.S, l.stride, l.pad)
        g = groups.setdefault(key, [l, 0])
        g[1] += 1
    tot_auto = tot_best = 0.0
    for key, (l, mult) in groups.items():
        d = am.conv_desc(*key)
        x = gen.relu_normal((l.N, l.H, l.W, l.C), 1)
        w = gen.he_normal((l.R, l.S, l.C, l.K), l.R * l.S * l.C, 2)
        dy = gen.normal((l.N, l.OH, l.OW, l.K), 3, 2 ** -10)
        y = torch.empty((l.N, l.OH, l.OW, l.K), device="cuda")
        dx = torch.empty((l.N, l.H, l.W, l.C), device="cuda")
        dw = torch.empty((l.R, l.S, l.C, l.K), device="cuda")
        passes = ["fwd", "wgrad"] + ([] if l.first else ["dgrad"])
        for pss in passes:
            res = {}
            for cfg in CFGS:
                if cfg == "auto":
                    os.environ.pop("AMSIM_FORCE_CFG", None)
                else:
                    os.environ["AMSIM_FORCE_CFG"] = cfg
                try:
                    if pss == "wgrad":
                        ws = torch.empty(max(am.amsim_conv2d_bwd_filter_workspace(lut, d) // 4, 1), device="cuda")
                except am.AmsimError as ex:
                    res[NAMES[cfg]] = f"error: {ex}"
                    continue
                fn = {"fwd": lambda: am.amsim_conv2d_fwd(lut, d, x, w, y),
                      "dgrad": lambda: am.amsim_conv2d_bwd_data(lut, d, dy, w, dx),
                      "wgrad": lambda: am.amsim_conv2d_bwd_filter(lut, d, x, dy, dw, ws)}[pss]
                try:
                    fn()
                except am.AmsimError as ex:
                    res[NAMES[cfg]] = f"error: {ex}"
                    continue
                torch.cuda.synchronize()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.reps)]
                for i in range(args.reps):
                    ev[2 * i].record()
                    fn()
                    ev[2 * i + 1].record()
                torch.cuda.synchronize()
                ts = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(args.reps))
                res[NAMES[cfg]] = round(ts[len(ts) // 2], 4)
            os.environ.pop("AMSIM_FORCE_CFG", None)
            timed = {k: v for k, v in res.items() if isinstance(v, float)}
            best = min(timed, key=timed.get)
            tot_auto += mult * timed["auto"]
            tot_best += mult * timed[best]
            print(json.dumps({"layer": l.name, "pass": pss, "mult": mult, "shape": key, "auto_ms": timed["auto"],
                              "best": best, "best_ms": timed[best], "gain": timed["auto"] / timed[best] - 1,
                              "all": res}), flush=True)
        del x, w, dy, y, dx, dw
        torch.cuda.empty_cache()
    print(json.dumps({"step_ms_auto": tot_auto, "step_ms_best": tot_best, "potential": tot_auto / tot_best - 1}))


if __name__ == "__main__":
    main()
