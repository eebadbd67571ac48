#!/usr/bin/env python
"""SASS evidence for the hot amsim_mm_kernel instantiations (no GPU needed):
opcode histogram of each kernel, the TMA / mbarrier opcodes present
(UTMALDG, SYNCS), and the static instruction count per table lookup in the
innermost loop (the basic block with the most LDS.U16 / LDS.U8 lookups).

    python tools/sass_histogram.py build/amsim_conv_dgrad.cu.o [--match Li16ELi8E] > profiles/r02_sass.md
"""
import argparse
import collections
import re
import subprocess


def functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs, cur, name = {}, None, None
    for ln in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            name = m.group(1)
            cur = funcs.setdefault(name, [])
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m and cur is not None:
            cur.append((int(m.group(1), 16), m.group(2).strip()))
    return funcs


def opcode(ins):
    ins = re.sub(r"^@!?U?P[T0-9]+\s+", "", ins)
    return ins.split(" ")[0]


def blocks(code):
    """Split at branch targets and after branches."""
    targets = set()
    for addr, ins in code:
        m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", ins)
        if m and m.group(1):
            targets.add(int(m.group(1), 16))
    bl, cur = [], []
    for addr, ins in code:
        if addr in targets and cur:
            bl.append(cur)
            cur = []
        cur.append((addr, ins))
        if opcode(ins) in ("BRA", "EXIT", "RET"):
            bl.append(cur)
            cur = []
    if cur:
        bl.append(cur)
    return bl


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("objs", nargs="+")
    ap.add_argument("--match", default="", help="regex on the mangled name")
    a = ap.parse_args()
    print("| kernel (demangled template args) | SASS instr | UTMALDG | SYNCS | LDS.U16/U8 | inner block: instr / lookups = per lookup |")
    print("|---|---|---|---|---|---|")
    for obj in a.objs:
        for name, code in functions(obj).items():
            if "amsim_mm_kernel" not in name or not re.search(a.match, name):
                continue
            ops = collections.Counter(opcode(i) for _, i in code)
            utma = sum(v for k, v in ops.items() if k.startswith("UTMALDG"))
            syncs = sum(v for k, v in ops.items() if k.startswith("SYNCS"))
            lk = sum(v for k, v in ops.items() if k in ("LDS.U16", "LDS.U8"))
            best = max(blocks(code), key=lambda b: sum(opcode(i) in ("LDS.U16", "LDS.U8") for _, i in b))
            nl = sum(opcode(i) in ("LDS.U16", "LDS.U8") for _, i in best)
            cfg = re.search(r"KCfgILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELb(\d)EEELi(\d+)E(.*?)ELb(\d)ELi(\d)ELb(\d)E", name)
            label = name[:60]
            if cfg:
                nt, tm, tn, wn, np_, eb, ops_, gl, mul, trn = cfg.groups()
                kinds = re.findall(r"(FwdX|WgX|DgDY|DgW|GemmOp)", ops_)
                label = f"{tm}x{tn} WN={wn}{' NP' if np_ == '1' else ''} EB={eb} {'/'.join(kinds)} GL={gl} MUL={mul} TRN={trn}"
            per = f"{len(best)} / {nl} = {len(best) / nl:.2f}" if nl else "-"
            print(f"| {label} | {len(code)} | {utma} | {syncs} | {lk} | {per} |")


if __name__ == "__main__":
    main()
