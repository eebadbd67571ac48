import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2209_04161_b200 as am
from paper_2209_04161_b200 import _lib as L
from amsim_inputs import device as gen
lut = am.Lut.build("mitchell", 7)
lib = L.lib()
st = torch.cuda.current_stream().cuda_stream
def t(M, N, K, policy=0, reps=2000):
    am.amsim_set_path_policy(policy)
    A, B = gen.normal((M, K), 1), gen.normal((K, N), 2)
    C = torch.empty(M, N, device="cuda")
    h, pa, pb, pc = lut.handle, A.data_ptr(), B.data_ptr(), C.data_ptr()
    for _ in range(10):
        lib.amsim_gemm(h, 0, 0, M, N, K, pa, K, pb, N, pc, N, 0, st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        lib.amsim_gemm(h, 0, 0, M, N, K, pa, K, pb, N, pc, N, 0, st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    am.amsim_set_path_policy(0)
    return (t1 - t0) / reps * 1e6
x = torch.empty(1, device="cuda")
t0 = time.perf_counter()
for _ in range(2000):
    lib.amsim_abi_version()
t1 = time.perf_counter()
print(json.dumps({"noop_ctypes_us": (t1 - t0) / 2000 * 1e6,
                  "gemm_256_split": t(256, 256, 256), "gemm_256_nosplit(policy2)": t(256, 256, 256, 2),
                  "gemm_256_nosplit_noTMA(policy10)": t(256, 256, 256, 10),
                  "gemm_256_K16": t(256, 256, 16), "gemm_256_N5_noTMA": t(256, 5, 16)}))
