#!/usr/bin/env python
"""Split an ncu source page (--page source --csv --print-source sass) of
amsim_mm_kernel into regions and report where the warp-stall samples and the
executed instructions go: the fast-path inner loop (the basic blocks holding
the table lookups, LDS.U16 / LDS.U8), the per-k-tile decode + barrier, and
the rest (prologue, tile switch, epilogue, stream-K fix-up).

    python tools/sass_regions.py gpurun_out/src_<tag>.csv [--top 25]
"""
import argparse
import csv
import io
import re


def load(path):
    text = open(path).read()
    i = text.index('"Address"')
    rows = list(csv.DictReader(io.StringIO(text[i:])))
    out = []
    for r in rows:
        try:
            out.append((int(r["Address"], 16), r["Source"].strip(), int(r["Warp Stall Sampling (All Samples)"] or 0),
                        int(r["Instructions Executed"] or 0)))
        except (ValueError, KeyError):
            continue
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    ins = load(a.path)
    tot_s = sum(x[2] for x in ins)
    tot_i = sum(x[3] for x in ins)
    # hot loop: maximal runs of instructions executed at the top frequency band around lookups
    lut = [k for k, x in enumerate(ins) if re.match(r"@?!?P?\d*\s*LDS\.U(16|8)\b", x[1].split(" ", 1)[-1].strip()) or
           re.search(r"\bLDS\.U(16|8)\b", x[1])]
    lo, hi = (min(lut), max(lut)) if lut else (0, -1)
    # extend to the enclosing branch targets (whole loop body)
    hot = set(range(lo, hi + 1))
    dec = {k for k, x in enumerate(ins) if ("BAR.SYNC" in x[1] or "REDUX" in x[1] or "VIMNMX" in x[1]) and k not in hot}
    reg = {"hot loop": [0, 0], "barrier/redux": [0, 0], "other": [0, 0]}
    for k, x in enumerate(ins):
        key = "hot loop" if k in hot else ("barrier/redux" if k in dec else "other")
        reg[key][0] += x[2]
        reg[key][1] += x[3]
    print(f"{a.path}: {len(ins)} SASS instructions, {tot_s} stall samples, {tot_i} warp instructions executed")
    for k, (s, i) in reg.items():
        print(f"  {k:14s} samples {s:9d} ({100 * s / max(tot_s, 1):5.1f} %)  instr {i:12d} ({100 * i / max(tot_i, 1):5.1f} %)")
    hot_ins = [x for k, x in enumerate(ins) if k in hot]
    ops = {}
    for x in hot_ins:
        op = re.sub(r"^@!?U?P\w+\s+", "", x[1]).split(" ")[0]
        o = ops.setdefault(op, [0, 0])
        o[0] += x[3]
        o[1] += x[2]
    print("  hot-loop opcode mix (instr executed, samples):")
    for op, (i, s) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:14]:
        print(f"    {op:14s} {i:12d} {s:9d}")
    print(f"  top {a.top} instructions outside the hot loop by samples:")
    outside = sorted([(x[2], k, x) for k, x in enumerate(ins) if k not in hot], reverse=True)[:a.top]
    for s, k, x in outside:
        print(f"    {s:8d} #{k:5d} exec {x[3]:10d}  {x[1][:80]}")


if __name__ == "__main__":
    main()
