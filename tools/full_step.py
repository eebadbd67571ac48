#!/usr/bin/env python
"""Whole training and inference steps on one B200 (the
B200 analog of the paper's per-batch timing tables).

Per workload (LeNet-5 b64, ResNet-18 CIFAR b128, ResNet-50 b256), ms per step:
  ATxG train / infer : net.py with AMSim (MBM table, m = 7) -- CUDA-graph replay
  ATnG train / infer : the same graph with AMSIM_MUL_NATIVE (native FP32 multiply)
  TFnG train / infer : the same architecture in PyTorch FP32 (cuDNN / cuBLAS,
                       TF32 off, channels_last), eager, SGD-momentum
plus the share of the ATxG training step spent in the approximate passes
(bench.py's step).  One JSON line per workload.

    python tools/full_step.py [--workloads lenet5 resnet18 resnet50] [--steps 5] [--model mbm]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

BATCH = {"lenet5": 64, "resnet18": 128, "resnet50": 256}


def torch_model(name):
    import torch
    import torch.nn as nn
    if name == "lenet5":
        return nn.Sequential(nn.Conv2d(1, 6, 5, padding=2), nn.ReLU(), nn.MaxPool2d(2), nn.Conv2d(6, 16, 5), nn.ReLU(),
                             nn.MaxPool2d(2), nn.Flatten(), nn.Linear(400, 120), nn.ReLU(), nn.Linear(120, 84),
                             nn.ReLU(), nn.Linear(84, 10))
    import torchvision
    if name == "resnet50":
        return torchvision.models.resnet50(num_classes=1000)
    m = torchvision.models.resnet18(num_classes=10)
    m.conv1 = nn.Conv2d(3, 64, 3, 1, 1, bias=False)
    m.maxpool = nn.Identity()
    return m


def time_fn(fn, warmup, steps):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", nargs="+", default=["lenet5", "resnet18", "resnet50"])
    ap.add_argument("--model", default="mbm")
    ap.add_argument("--m", type=int, default=7)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()

    import torch

    import paper_2209_04161_b200 as am
    from paper_2209_04161_b200 import net as netmod
    from paper_2209_04161_b200.train_step import TrainStep
    import amsim_inputs as inp

    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    dev = torch.device("cuda", 0)
    lut = am.Lut.build(args.model, args.m)
    for w in args.workloads:
        B = BATCH[w]
        steps = args.steps if w == "resnet50" else 10 * args.steps
        res = {"workload": w, "batch": B, "model": args.model, "m": args.m}
        net = netmod.BUILDERS[w](lut, batch=B, seed=11)
        res["approx_macs_per_step"] = net.approx_macs
        for tag, mode in (("ATxG", am.AMSIM_MUL_LUT), ("ATnG", am.AMSIM_MUL_NATIVE)):
            with am.multiply_mode(mode):
                net.train_step()
                tr = net.capture(net.train_step)
                res[f"{tag}_train_ms"] = time_fn(tr, args.warmup, steps)
                net.infer_step()
                inf = net.capture(net.infer_step)
                res[f"{tag}_infer_ms"] = time_fn(inf, args.warmup, steps)
                res[f"{tag}_loss_after"] = float(net.loss_value.item())
        del net, tr, inf
        torch.cuda.empty_cache()
        # the approximate passes alone (bench.py's step), same table
        layers = {"lenet5": inp.lenet5_layers, "resnet18": inp.resnet18_cifar_layers,
                  "resnet50": inp.resnet50_layers}[w](B)
        ts = TrainStep(layers, lut, device=dev, seed=11, first_input="mnist" if w == "lenet5" else "relu")
        ts.step()
        res["approx_passes_ms"] = time_fn(ts.capture(), args.warmup, steps)
        del ts
        torch.cuda.empty_cache()
        # TFnG analog
        model = torch_model(w).to(dev).to(memory_format=torch.channels_last)
        opt = torch.optim.SGD(model.parameters(), lr=0.01, momentum=0.9, weight_decay=5e-5)
        shape = {"lenet5": (B, 1, 28, 28), "resnet18": (B, 3, 32, 32), "resnet50": (B, 3, 224, 224)}[w]
        x = torch.randn(shape, device=dev).to(memory_format=torch.channels_last)
        y = torch.randint(0, 10 if w != "resnet50" else 1000, (B,), device=dev)
        lossf = torch.nn.CrossEntropyLoss()

        def tf_train():
            opt.zero_grad(set_to_none=True)
            lossf(model(x), y).backward()
            opt.step()

        def tf_infer():
            with torch.no_grad():
                model(x)
        model.train()
        res["TFnG_train_ms"] = time_fn(tf_train, args.warmup, steps)
        model.eval()
        res["TFnG_infer_ms"] = time_fn(tf_infer, args.warmup, steps)
        del model, opt, x
        torch.cuda.empty_cache()
        res["ratios"] = {"train ATxG/TFnG": res["ATxG_train_ms"] / res["TFnG_train_ms"],
                         "train ATnG/TFnG": res["ATnG_train_ms"] / res["TFnG_train_ms"],
                         "infer ATxG/TFnG": res["ATxG_infer_ms"] / res["TFnG_infer_ms"],
                         "approx share of ATxG train": res["approx_passes_ms"] / res["ATxG_train_ms"]}
        res["paper_context"] = ("PAPER.md:888-942 per-batch training/inference times; ATxG/TFnG 7.32x geomean on "
                                "GTX1080/V100 (PAPER.md:35, 994)")
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
