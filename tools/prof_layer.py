#!/usr/bin/env python
"""Run one ResNet/LeNet layer pass (or a GEMM) a few times -- a short target
for ncu captures and quick per-kernel timing.

    python tools/prof_layer.py --layer l1.0.conv2 --pass fwd [--batch 256] [--reps 3]
    python tools/prof_layer.py --gemm 4096 4096 4096
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="resnet50")
    ap.add_argument("--layer", default="l1.0.conv2")
    ap.add_argument("--pass", dest="which", default="fwd", choices=["fwd", "dgrad", "wgrad"])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--model", default="mbm")
    ap.add_argument("--m", type=int, default=7)
    ap.add_argument("--gemm", type=int, nargs=3, default=None)
    ap.add_argument("--policy", type=int, default=0)
    args = ap.parse_args()

    import torch

    import amsim_inputs as inp
    from amsim_inputs import device as gen
    import paper_2209_04161_b200 as am

    lut = am.Lut.build(args.model, args.m)
    am.amsim_set_path_policy(args.policy)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.reps)]
    if args.gemm:
        M, N, K = args.gemm
        A = gen.normal((M, K), 1)
        B = gen.normal((K, N), 2)
        C = torch.empty((M, N), device="cuda")
        fn = lambda: am.amsim_gemm(lut, A, B, C)  # noqa: E731
        macs = M * N * K
        label = f"gemm {M}x{N}x{K}"
    else:
        nets = {"resnet50": inp.resnet50_layers, "resnet18": inp.resnet18_cifar_layers, "lenet5": inp.lenet5_layers}
        L = {l.name: l for l in nets[args.net](args.batch)}[args.layer]
        if not hasattr(L, "H"):   # dense layer: fwd X W, wgrad X^T dY, dgrad dY W^T
            x = gen.relu_normal((L.N, L.IN), 1)
            w = gen.he_normal((L.IN, L.OUT), L.IN, 2)
            dy = gen.normal((L.N, L.OUT), 3, 2 ** -10)
            out = {"fwd": torch.empty((L.N, L.OUT), device="cuda"), "wgrad": torch.empty((L.IN, L.OUT), device="cuda"),
                   "dgrad": torch.empty((L.N, L.IN), device="cuda")}[args.which]
            fn = {"fwd": lambda: am.amsim_gemm(lut, x, w, out),
                  "wgrad": lambda: am.amsim_gemm(lut, x, dy, out, trans_a=True),
                  "dgrad": lambda: am.amsim_gemm(lut, dy, w, out, trans_b=True)}[args.which]
            macs = L.macs()
            label = f"{args.net} {args.layer} {args.which} b{args.batch}"
            return _time(fn, args, ev, macs, label)
        d = am.conv_desc(L.N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad)
        x = gen.relu_normal((L.N, L.H, L.W, L.C), 1)
        w = gen.he_normal((L.R, L.S, L.C, L.K), L.R * L.S * L.C, 2)
        dy = gen.normal((L.N, L.OH, L.OW, L.K), 3, 2 ** -10)
        macs = L.macs()
        if args.which == "fwd":
            y = torch.empty((L.N, L.OH, L.OW, L.K), device="cuda")
            fn = lambda: am.amsim_conv2d_fwd(lut, d, x, w, y)  # noqa: E731
        elif args.which == "dgrad":
            dx = torch.empty((L.N, L.H, L.W, L.C), device="cuda")
            fn = lambda: am.amsim_conv2d_bwd_data(lut, d, dy, w, dx)  # noqa: E731
        else:
            dw = torch.empty((L.R, L.S, L.C, L.K), device="cuda")
            ws = torch.empty(max(am.amsim_conv2d_bwd_filter_workspace(lut, d) // 4, 1), device="cuda")
            fn = lambda: am.amsim_conv2d_bwd_filter(lut, d, x, dy, dw, ws)  # noqa: E731
        label = f"{args.net} {args.layer} {args.which} b{args.batch}"
    _time(fn, args, ev, macs, label)


def _time(fn, args, ev, macs, label):
    import torch
    fn()
    torch.cuda.synchronize()
    for i in range(args.reps):
        ev[2 * i].record()
        fn()
        ev[2 * i + 1].record()
    torch.cuda.synchronize()
    ts = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(args.reps)]
    best = min(ts)
    print(f"{label}: {best:.3f} ms  {macs / best / 1e6:.1f} GMAC/s  (reps {[round(t, 3) for t in ts]})")


if __name__ == "__main__":
    main()
