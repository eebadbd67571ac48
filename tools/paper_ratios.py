#!/usr/bin/env python
"""The paper's runtime comparisons on one B200.

PAPER.md:956-1006 compares, per training step of LeNet-5 / ResNet models:
  TFnG  native TF on the GPU (cuDNN / cuBLAS)       -> here: PyTorch FP32 conv / matmul
                                                       (cuDNN / cuBLAS, TF32 off)
  ATnG  ApproxTrain's own GEMM kernels, native mult -> libamsim, AMSIM_MUL_NATIVE
  ATxG  ApproxTrain with AMSim (LUT)                 -> libamsim, AMSIM_MUL_LUT  (the product)
  ATxC  ApproxTrain on the CPU                       -> bench.py cpu_baseline (the oracle)
and AMSim against direct simulation of the multiplier:
  DIRECT  the functional model evaluated per product, no table -> AMSIM_MUL_DIRECT.
Every variant runs the same approximate-layer passes of one training step (fwd
for all Conv2D / Dense layers, wgrad for all, dgrad for all but the first),
timed with CUDA events after warm-up.  One JSON line per (workload, model).

    python tools/paper_ratios.py [--workloads lenet5 resnet18 resnet50] [--models mbm mitchell exact]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

BATCH = {"lenet5": 64, "resnet18": 128, "resnet50": 256}


def torch_native_step(layers, dev, seed=7):
    """The same passes through PyTorch FP32 (cuDNN convolution / cuBLAS matmul):
    activations NHWC (channels_last), weights OIHW."""
    import torch

    from amsim_inputs import device as gen
    from amsim_inputs import workloads as wl

    ops = []
    for i, l in enumerate(layers):
        s = seed + 16 * i
        if isinstance(l, wl.ConvLayer):
            x = gen.relu_normal((l.N, l.H, l.W, l.C), s, device=dev).permute(0, 3, 1, 2)  # NCHW view, NHWC memory
            w = gen.he_normal((l.K, l.C, l.R, l.S), l.R * l.S * l.C, s + 1, device=dev)
            dy = gen.normal((l.N, l.OH, l.OW, l.K), s + 2, 2 ** -10, device=dev).permute(0, 3, 1, 2)
            st, pd = [l.stride, l.stride], [l.pad, l.pad]

            def fwd(x=x, w=w, st=st, pd=pd):
                return torch.nn.functional.conv2d(x, w, None, st, pd)

            def bwd(x=x, w=w, dy=dy, st=st, pd=pd, first=l.first):
                return torch.ops.aten.convolution_backward(dy, x, w, None, st, pd, [1, 1], False, [0, 0], 1,
                                                           [not first, True, False])
            ops.append((fwd, bwd))
        else:
            x = gen.relu_normal((l.N, l.IN), s, device=dev)
            w = gen.he_normal((l.IN, l.OUT), l.IN, s + 1, device=dev)
            dy = gen.normal((l.N, l.OUT), s + 2, 2 ** -10, device=dev)

            def fwd(x=x, w=w):
                return x @ w

            def bwd(x=x, w=w, dy=dy, first=l.first):
                dw = x.t() @ dy
                return dw if first else (dw, dy @ w.t())
            ops.append((fwd, bwd))

    def step():
        for f, _ in ops:
            f()
        for _, b in reversed(ops):
            b()
    return step


def time_fn(fn, warmup, reps):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", nargs="+", default=["lenet5", "resnet18", "resnet50"])
    ap.add_argument("--models", nargs="+", default=["mbm", "mitchell", "exact"])
    ap.add_argument("--m", type=int, default=7)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()

    import torch

    import amsim_inputs as inp
    import paper_2209_04161_b200 as am
    from paper_2209_04161_b200.train_step import TrainStep

    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    dev = torch.device("cuda", 0)
    nets = {"lenet5": inp.lenet5_layers, "resnet18": inp.resnet18_cifar_layers, "resnet50": inp.resnet50_layers}
    for wname in args.workloads:
        layers = nets[wname](BATCH[wname])
        macs = sum(l.macs() * (2 if l.first else 3) for l in layers)
        reps = args.reps if wname == "resnet50" else 4 * args.reps
        tfng = time_fn(torch_native_step(layers, dev), args.warmup, reps)
        for model in args.models:
            lut = am.Lut.build(model, args.m)
            step = TrainStep(layers, lut, device=dev, seed=7, first_input="mnist" if wname == "lenet5" else "relu")
            t = {}
            for name, mode in (("ATxG", am.AMSIM_MUL_LUT), ("ATnG", am.AMSIM_MUL_NATIVE),
                               ("DIRECT", am.AMSIM_MUL_DIRECT)):
                with am.multiply_mode(mode):
                    t[name] = time_fn(step.step, args.warmup, reps)
            del step
            torch.cuda.empty_cache()
            line = {"workload": wname, "batch": BATCH[wname], "model": model, "m": args.m,
                    "entry_bits": lut.info()[1], "macs_per_step": macs,
                    "ms_per_step": {"TFnG": tfng, **t},
                    "gmacs": {k: macs / (v * 1e-3) / 1e9 for k, v in {"TFnG": tfng, **t}.items()},
                    "ratios": {"ATxG/TFnG": t["ATxG"] / tfng, "ATnG/TFnG": t["ATnG"] / tfng,
                               "ATxG/ATnG": t["ATxG"] / t["ATnG"], "DIRECT/ATxG": t["DIRECT"] / t["ATxG"]},
                    "paper_context": "PAPER.md:35,994: ATxG ~8x (7.32x geomean) slower than TFnG on V100/GTX1080; "
                                     "AMSim GEMM ~2x native, direct simulation 4.6-78.2x (PAPER.md:398)"}
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
