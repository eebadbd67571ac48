#!/usr/bin/env python
"""Summarise an ncu --set full report (.ncu-rep) into the numbers DESIGN.md and
bench.py's roofline refer to.  Usage: python tools/ncu_summary.py rep [rep ...]
"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("sm__cycles_active.max", "SM active cycles (max)"),
    ("sm__cycles_active.min", "SM active cycles (min)"),
    ("sm__cycles_elapsed.max", "SM elapsed cycles"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sass__inst_executed_shared_loads", "shared load instr"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "LSU data-pipe wavefronts % of peak"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe inst % of peak"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA-pipe inst %"),
    ("dram__bytes_read.sum", "DRAM read bytes"),
    ("dram__bytes_write.sum", "DRAM write bytes"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard /issue"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio_throttle /issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait /issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier /issue"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard /issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe /issue"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected /issue"),
]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    name = d.get("Kernel Name", ("", "?"))[1]
    out = [f"### {path}", f"kernel: {name[:160]}"]
    for key, label in WANT:
        if key in d:
            u, v = d[key]
            out.append(f"- {label}: {v} {u}".rstrip())
    return "\n".join(out)


if __name__ == "__main__":
    print("\n\n".join(summarise(p) for p in sys.argv[1:]))
