#!/usr/bin/env python
"""Per-configuration cost per padded approx-MAC from a `tools/cfg_sweep.py`
run: for every timed (pass, tile configuration) the device time divided by
the MACs of the padded tiles it computes, then the median per configuration
over the dense-operand passes (dgrad) and the layer-input passes (fwd / wgrad)
-- the `measured_cost16` table of csrc/amsim_dispatch.cuh (ms per G padded
approx-MACs).  Strided dgrad (several stride-phase sub-problems) is left out.

    python tools/fit_costs.py profiles/r02_cfg_sweep_b256.jsonl
"""
import json
import statistics
import sys

# (BM, BN) of each configuration; ^T = transposed orientation (rows = the
# original N dimension, lanes = the original M dimension)
SHAPE = {"Small": (64, 32), "Mid": (128, 64), "Big": (128, 128), "Lean": (64, 64), "Wide": (64, 128),
         "Huge": (128, 256), "Flat": (64, 256), "Tall": (160, 64), "Flat3": (64, 192), "TallT": (64, 160),
         "Flat8": (64, 512)}


def ceil_to(x, m):
    return (x + m - 1) // m * m


def problem(shape, pss):
    N, H, W, C, K, R, S, st, pd = shape
    OH = (H + 2 * pd - R) // st + 1
    OW = (W + 2 * pd - S) // st + 1
    if pss == "fwd":
        return N * OH * OW, K, R * S * C
    if pss == "wgrad":
        return R * S * C, K, N * OH * OW
    if st != 1:
        return None
    return N * H * W, C, R * S * K


def main():
    rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith('{"layer"')]
    costs = {}
    for r in rows:
        pr = problem(r["shape"], r["pass"])
        if pr is None:
            continue
        M, N, K = pr
        kind = "dense" if r["pass"] == "dgrad" else "act"
        for name, ms in r["all"].items():
            if not isinstance(ms, float) or name == "auto":
                continue
            base = name.rstrip("^T")
            trn = name.endswith("^T")
            BM, BN = SHAPE[base]
            rows_, lanes = (N, M) if trn else (M, N)
            padded = ceil_to(rows_, BM) * ceil_to(lanes, BN) * ceil_to(K, 16)
            costs.setdefault((name, kind), []).append(ms / (padded / 1e9))
    print(f"{'config':10s} {'act':>8s} {'dense':>8s}  (ms per G padded approx-MACs, median; n passes)")
    for name in sorted({k[0] for k in costs}):
        a = costs.get((name, "act"), [])
        d = costs.get((name, "dense"), [])
        fa = f"{statistics.median(a):8.4f}" if a else "       -"
        fd = f"{statistics.median(d):8.4f}" if d else "       -"
        print(f"{name:10s} {fa} {fd}  ({len(a)}, {len(d)})")


if __name__ == "__main__":
    main()
