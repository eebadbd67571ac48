"""Latency of small approx GEMMs (BASELINE config 1 is 256^3): per-call device time, median of 200."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2209_04161_b200 as am
from amsim_inputs import device as gen
lut = am.Lut.build(sys.argv[1] if len(sys.argv) > 1 else "mitchell", 7)
for n in (256, 512):
    A, B = gen.normal((n, n), 1), gen.normal((n, n), 2)
    C = torch.empty(n, n, device="cuda")
    for _ in range(5):
        am.amsim_gemm(lut, A, B, C)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(400)]
    for i in range(200):
        ev[2 * i].record(); am.amsim_gemm(lut, A, B, C); ev[2 * i + 1].record()
    torch.cuda.synchronize()
    ts = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(200))
    print(json.dumps({"n": n, "cfg": os.environ.get("AMSIM_FORCE_CFG", "auto"), "us_median": ts[100] * 1e3, "us_min": ts[0] * 1e3}))
