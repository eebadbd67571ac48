#!/usr/bin/env python
"""BASELINE.json config 5: approx-GEMM throughput sweep on one B200.

Cubes M = N = K in {512, ..., 16384} and LUT widths m = 4..7, Mitchell (the
config's model) with the exact multiplier as the model-independence check,
each beside the measured LUT-lookup rate of the same m and device layout
(amsim_bench_lut_lookup).  One JSON line per point on stdout.

    python tools/sweep.py [--sizes 512 1024 ...] [--ms 4 5 6 7] [--models mitchell exact] [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[512, 1024, 2048, 4096, 8192, 16384])
    ap.add_argument("--ms", type=int, nargs="+", default=[4, 5, 6, 7])
    ap.add_argument("--models", nargs="+", default=["mitchell", "exact"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--policy", type=int, default=0)
    ap.add_argument("--modes", nargs="+", default=["lut"], choices=["lut", "native", "direct"],
                    help="multiply mode: the AMSim table (product) or the native / direct-model instruments")
    args = ap.parse_args()

    import numpy as np
    import torch

    from amsim_inputs import device as gen
    import paper_2209_04161_b200 as am

    am.amsim_set_path_policy(args.policy)
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    idx_cache = {}
    for model in args.models:
        for m in args.ms:
            lut = am.Lut.build(model, m)
            width = lut.info()[1]
            if (m, width) not in idx_cache:
                idx = np.random.default_rng(0).integers(0, 1 << m, 1 << 16).astype(np.uint32)
                try:
                    idx_cache[(m, width)] = am.amsim_bench_lut_lookup(m, width, idx, iters=2048) / 1e9
                except am.AmsimError:       # table beyond shared memory: no smem-lookup instrument
                    idx_cache[(m, width)] = None
            lookup = idx_cache[(m, width)]
            for n, mode in [(n, md) for n in args.sizes for md in args.modes]:
                am.amsim_set_multiply_mode({"lut": 0, "native": 1, "direct": 2}[mode])
                A = gen.normal((n, n), 1, device=dev)
                B = gen.normal((n, n), 2, device=dev)
                C = torch.empty((n, n), device=dev)
                # per-repetition CUDA events, median reported (single slow reps -- allocator,
                # clock transitions -- do not move it); more reps for the short problems
                reps = max(3, min(50, int(20 * 1024 ** 3 / n ** 3) + 3))
                for _ in range(2):
                    am.amsim_gemm(lut, A, B, C)      # warm-up (table upload, plan)
                torch.cuda.synchronize()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
                for i in range(reps):
                    ev[2 * i].record()
                    am.amsim_gemm(lut, A, B, C)
                    ev[2 * i + 1].record()
                torch.cuda.synchronize()
                ts = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(reps))
                ms = ts[len(ts) // 2]
                gmacs = n ** 3 / (ms * 1e-3) / 1e9
                peak = sms * 32 * 1965e6 / 1e9
                am.amsim_set_multiply_mode(0)
                print(json.dumps({"mode": mode, "model": model, "m": m, "entry_bits": width, "M": n, "N": n, "K": n,
                                  "ms": ms, "gmacs": gmacs, "frac_of_32_lookups_per_clk": gmacs / peak,
                                  "lookup_measured_gps": lookup,
                                  "frac_of_measured_lookup": gmacs / lookup if lookup else None,
                                  "reps": reps, "ms_min": ts[0], "ms_max": ts[-1]}), flush=True)
                del A, B, C
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
