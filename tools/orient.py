"""Does a skinny-N GEMM run faster transposed?  (M, 64, K) vs (64, M, K), MBM m=7."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2209_04161_b200 as am
from amsim_inputs import device as gen
lut = am.Lut.build("mbm", 7)
for (M, N, K) in [(802816, 64, 576), (64, 802816, 576), (802816, 64, 64), (64, 802816, 64), (200704, 128, 1152), (128, 200704, 1152)]:
    A, B = gen.normal((M, K), 1), gen.normal((K, N), 2)
    C = torch.empty(M, N, device="cuda")
    for _ in range(2):
        am.amsim_gemm(lut, A, B, C)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    for i in range(3):
        ev[2 * i].record(); am.amsim_gemm(lut, A, B, C); ev[2 * i + 1].record()
    torch.cuda.synchronize()
    ms = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(3))[1]
    print(json.dumps({"M": M, "N": N, "K": K, "ms": ms, "gmacs": M * N * K / ms / 1e6}))
    del A, B, C
    torch.cuda.empty_cache()
