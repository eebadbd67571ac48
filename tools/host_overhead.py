"""Host-side cost per C-ABI call (enqueue only) and device time of the same call
replayed from a CUDA graph -- separates launch overhead from kernel time."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2209_04161_b200 as am
from paper_2209_04161_b200 import _lib as L
from amsim_inputs import device as gen
lut = am.Lut.build("mitchell", 7)
n = 256
A, B = gen.normal((n, n), 1), gen.normal((n, n), 2)
C = torch.empty(n, n, device="cuda")
for _ in range(10):
    am.amsim_gemm(lut, A, B, C)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000):
    am.amsim_gemm(lut, A, B, C)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
# raw ctypes call, pointers precomputed
lib = L.lib()
h, pa, pb, pc = lut.handle, A.data_ptr(), B.data_ptr(), C.data_ptr()
st = torch.cuda.current_stream().cuda_stream
t3 = time.perf_counter()
for _ in range(2000):
    lib.amsim_gemm(h, 0, 0, n, n, n, pa, n, pb, n, pc, n, 0, st)
t4 = time.perf_counter()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    am.amsim_gemm(lut, A, B, C)
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(g):
    for _ in range(20):
        am.amsim_gemm(lut, A, B, C)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g.replay()
e1.record(); torch.cuda.synchronize()
print(json.dumps({"python_call_us": (t1 - t0) / 2000 * 1e6, "drain_us_total": (t2 - t1) * 1e6,
                  "raw_ctypes_call_us": (t4 - t3) / 2000 * 1e6,
                  "graph_device_us_per_gemm": e0.elapsed_time(e1) / 200 * 1e3}))
