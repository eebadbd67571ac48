#!/usr/bin/env python
"""Benchmark of the AMSim hot path on B200 (one JSON line on rank 0).

Default workload (BASELINE.json configs[3], the metric's "ResNet-50 train
step"): ResNet-50 ImageNet-shaped training step, global batch 256 sharded over
the GPUs (strong scaling), every Conv2D / Dense pass through the C ABI with the
AFM16/MBM stand-in table at m = 7, plus the NCCL weight-gradient all-reduce
when N > 1.  value = approx-GMAC/s of the whole job.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl amsim|reference]
                    [--workload resnet50|resnet18|lenet5] [--model mbm|exact|mitchell] [--m 7]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AMSim approx-GEMM/conv GMAC/s at 1/2/4/8 B200; ResNet-50 train step ms"


def workload_layers(name: str, batch: int):
    import amsim_inputs as inp
    if name == "resnet50":
        return inp.resnet50_layers(batch), 256
    if name == "resnet18":
        return inp.resnet18_cifar_layers(batch), 128
    if name == "lenet5":
        return inp.lenet5_layers(batch), 64
    raise SystemExit(f"unknown workload {name}")


def global_batch(name):
    return {"resnet50": 256, "resnet18": 128, "lenet5": 64}[name]


def workload_label(name, model, m, size=16384):
    if name == "gemm":
        return f"approx GEMM M=N=K={size} (BASELINE.json config 5), {model} LUT m={m}, rows sharded over the GPUs"
    return {"resnet50": "ResNet-50 ImageNet-shaped (224x224x3) train step, global batch 256",
            "resnet18": "ResNet-18 CIFAR-shaped (32x32x3) train step, batch 128",
            "lenet5": "LeNet-5 MNIST-shaped (28x28x1) train step, batch 64"}[name] + f", {model} LUT m={m}"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md clocks line)

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle (as it stands) on a bounded sample of the workload

def oracle_gemm_sample(n: int, model: str, m: int, budget_s: float):
    """The oracle on whole output rows of the n^3 GEMM (config 5), blocks of
    max(16, threads) rows (A rows and B drawn from seeded N(0,1) generators, the GPU run's
    distribution) until `budget_s` is spent."""
    import amsim_inputs as inp
    import oracle
    B = inp.normal((n, n), 2)
    blk = max(16, oracle.num_threads())      # the oracle parallelises over output rows
    macs, done = 0, 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < budget_s and done < n:
        A = inp.normal((blk, n), 100 + done)
        oracle.gemm(A, B, model, m)
        macs += blk * n * n
        done += blk
    dt = time.perf_counter() - t0
    desc = f"{done} output rows of the {n}^3 GEMM ({macs / 1e9:.2f} G approx-MACs), plain-C oracle -O2 OpenMP"
    return macs, dt, oracle.num_threads(), desc


def cpu_info():
    """CPU model name and logical core count of this host (cpu_baseline context)."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def oracle_sample(workload: str, model: str, m: int, budget_s: float, size: int = 16384, keep=0):
    """Run the oracle over the workload's layer passes at batch 1 (in step
    order: all forwards, then wgrad/dgrad in reverse) until `budget_s` is
    spent.  Returns (macs, seconds, threads, description[, kept]) -- with keep > 0
    also the inputs and oracle results of the first `keep` passes, for the
    GPU-vs-oracle check of the same sample (sample_parity)."""
    import numpy as np

    import amsim_inputs as inp
    import oracle
    if workload == "gemm":
        return oracle_gemm_sample(size, model, m, budget_s)
    layers, _ = workload_layers(workload, 1)
    passes = [("fwd", l) for l in layers] + [(p, l) for l in layers[::-1] for p in
                                              (("wgrad",) if l.first else ("wgrad", "dgrad"))]
    macs = 0
    t0 = time.perf_counter()
    done = 0
    kept = []
    for i, (kind, l) in enumerate(passes):
        if isinstance(l, inp.ConvLayer):
            d = oracle.conv_desc(l.N, l.H, l.W, l.C, l.K, l.R, l.S, l.stride, l.pad)
            x = inp.relu_normal((l.N, l.H, l.W, l.C), 10 + i)
            w = inp.he_normal((l.R, l.S, l.C, l.K), l.R * l.S * l.C, 11 + i)
            dy = inp.normal((l.N, l.OH, l.OW, l.K), 12 + i, 2 ** -10)
            if kind == "fwd":
                res = oracle.conv_fwd(d, x, w, model, m)
            elif kind == "wgrad":
                res = oracle.conv_bwd_filter(d, x, dy, model, m)
            else:
                res = oracle.conv_bwd_data(d, dy, w, model, m)
        else:
            x = inp.relu_normal((l.N, l.IN), 10 + i)
            w = inp.he_normal((l.IN, l.OUT), l.IN, 11 + i)
            dy = inp.normal((l.N, l.OUT), 12 + i, 2 ** -10)
            if kind == "fwd":
                res = oracle.gemm(x, w, model, m)
            elif kind == "wgrad":
                res = oracle.gemm(np.ascontiguousarray(x.T), dy, model, m)
            else:
                res = oracle.gemm(dy, np.ascontiguousarray(w.T), model, m)
        if len(kept) < keep:
            kept.append((kind, l, x, w, dy, res))
        macs += l.macs()
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    desc = (f"{workload} at batch 1: first {done} of {len(passes)} layer passes in step order "
            f"({macs / 1e9:.2f} G approx-MACs), plain-C oracle -O2 OpenMP")
    if keep:
        return macs, dt, oracle.num_threads(), desc, kept
    return macs, dt, oracle.num_threads(), desc


def sample_parity(am, lut, kept):
    """The GPU path on the cpu_baseline sample's own inputs: every kept pass
    through the C ABI, compared with the oracle's result element by element
    (|gpu - c64| <= 1e-5 sum|p| + FLT_MIN, reading C12).  Returns a summary."""
    import numpy as np
    import torch
    worst, n_el = 0.0, 0
    for kind, l, x, w, dy, res in kept:
        X, Wt, DY = (torch.from_numpy(np.ascontiguousarray(t)).cuda() for t in (x, w, dy))
        if hasattr(l, "H"):
            d = am.conv_desc(l.N, l.H, l.W, l.C, l.K, l.R, l.S, l.stride, l.pad)
            if kind == "fwd":
                out = torch.empty((l.N, l.OH, l.OW, l.K), device="cuda")
                am.amsim_conv2d_fwd(lut, d, X, Wt, out)
            elif kind == "wgrad":
                out = torch.empty((l.R, l.S, l.C, l.K), device="cuda")
                ws = torch.empty(max(am.amsim_conv2d_bwd_filter_workspace(lut, d) // 4, 1), device="cuda")
                am.amsim_conv2d_bwd_filter(lut, d, X, DY, out, ws)
            else:
                out = torch.empty((l.N, l.H, l.W, l.C), device="cuda")
                am.amsim_conv2d_bwd_data(lut, d, DY, Wt, out)
        else:
            if kind == "fwd":
                out = am.amsim_gemm(lut, X, Wt, torch.empty((l.N, l.OUT), device="cuda"))
            elif kind == "wgrad":
                out = am.amsim_gemm(lut, X, DY, torch.empty((l.IN, l.OUT), device="cuda"), trans_a=True)
            else:
                out = am.amsim_gemm(lut, DY, Wt, torch.empty((l.N, l.IN), device="cuda"), trans_b=True)
        got = out.cpu().numpy().reshape(res.c64.shape).astype(np.float64)
        tol = 1e-5 * res.abs64 + np.finfo(np.float32).tiny
        worst = max(worst, float(np.max(np.abs(got - res.c64) / tol)))
        n_el += got.size
    return {"passes": len(kept), "elements": n_el, "max_err_over_tol": worst, "ok": worst <= 1.0}


def run_reference(args):
    """--impl reference: the oracle timed as it stands on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # torchrun sets OMP_NUM_THREADS=1 per rank; rank 0 alone runs the oracle, on all host cores
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    import oracle
    oracle.build()
    for _ in range(args.warmup):
        oracle_sample(args.workload, args.model, args.m, args.ref_budget, args.size)
    vals, secs = [], []
    macs = 0
    desc = ""
    threads = 0
    for _ in range(args.steps):
        macs, dt, threads, desc = oracle_sample(args.workload, args.model, args.m, args.ref_budget, args.size)
        secs.append(dt)
    tot = sum(secs)
    value = macs * args.steps / tot / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GMAC/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded, shapes and value distributions of the paper's workloads)",
        "config": {"workload": workload_label(args.workload, args.model, args.m, args.size) + " [oracle sample]",
                   "model": args.model, "m": args.m},
        "cpu_baseline": {"value": value, "unit": "GMAC/s", "cores": threads, "kind": "oracle", "sample": desc,
                         **cpu_info()},
        "e2e": {"value": value, "unit": "GMAC/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# BASELINE.json config 5 at N GPUs: one M = N = K approx GEMM, rows sharded

def run_gemm(args, world, rank, gpu, dev, comm=None):
    """rows of A / C partitioned over the ranks, B and the
    table replicated (B broadcast from rank 0 outside the timed region), no
    collective on the data path; the all-gather of C is timed separately.
    value = n^3 approx-MACs / (max over ranks of the device time per GEMM)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from amsim_inputs import device as gen
    import paper_2209_04161_b200 as am
    from paper_2209_04161_b200.dp import gather_rows, max_over_ranks, shard_batch, sharded_gemm

    n = args.size
    lut = am.Lut.build(args.model, args.m)
    am.amsim_set_path_policy(args.policy)
    r0, rows = shard_batch(n, world, rank)
    A = gen.normal((n, n), 1, device=dev)           # every rank reads only its rows
    B = gen.normal((n, n), 2, device=dev) if rank == 0 else torch.empty((n, n), device=dev)
    if world > 1:
        dist.broadcast(B, 0)
    C = torch.zeros((n, n), device=dev)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            if dist.get_backend() == "nccl":
                dist.barrier(device_ids=[gpu])
            else:
                dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        sharded_gemm(am, lut, A, B, C, world, rank)
    barrier()
    # between timed GEMMs: inputs larger than L2 (B is n^2 * 4 B; A's block rows * n * 4 B)
    clocks = ClockSampler(gpu)
    clocks.start()
    launches0 = am.amsim_launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    barrier()
    for i in range(args.steps):
        ev[2 * i].record()
        sharded_gemm(am, lut, A, B, C, world, rank)
        ev[2 * i + 1].record()
    barrier()
    launches = am.amsim_launch_count() - launches0
    clk = clocks.stop()
    per = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(args.steps)]
    ms_local = sum(per) / args.steps
    ms = max_over_ranks(ms_local, dev)
    macs = n ** 3
    value = macs / (ms * 1e-3) / 1e9
    achieved = rows * n * n / (ms_local * 1e-3) / 1e9     # this rank's kernel rate
    props = torch.cuda.get_device_properties(dev)
    sm_max = clk.get("sm_max_mhz") or 1965.0
    peak = props.multi_processor_count * 32 * sm_max * 1e6 / 1e9
    lut_meas = None
    try:
        idx = np.random.default_rng(0).integers(0, 1 << args.m, 1 << 16).astype(np.uint32)
        lut_meas = am.amsim_bench_lut_lookup(args.m, lut.info()[1], idx, iters=2048) / 1e9
    except Exception as ex:  # noqa: BLE001
        lut_meas = f"unavailable: {ex}"

    gather_ms = None
    if world > 1:
        out = torch.empty_like(C)
        gather_rows(C[r0:r0 + rows], n, world, out)
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(args.steps):
            gather_rows(C[r0:r0 + rows], n, world, out)
        g1.record()
        barrier()
        gather_ms = max_over_ranks(g0.elapsed_time(g1) / args.steps, dev)
        del out

    # end to end through the public API: this rank's A rows and B from pinned host
    # memory, the GEMM, this rank's C rows back to pinned host memory, every step
    e2e = None
    if not args.no_e2e:
        hA = torch.empty((rows, n), pin_memory=True)
        hA.copy_(A[r0:r0 + rows])
        hB = torch.empty((n, n), pin_memory=True)
        hB.copy_(B)
        hC = torch.empty((rows, n), pin_memory=True)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            A[r0:r0 + rows].copy_(hA, non_blocking=True)
            B.copy_(hB, non_blocking=True)
            sharded_gemm(am, lut, A, B, C, world, rank)
            hC.copy_(C[r0:r0 + rows], non_blocking=True)
        f1.record()
        barrier()
        ems = max_over_ranks(f0.elapsed_time(f1) / args.steps, dev)
        e2e = {"value": macs / (ems * 1e-3) / 1e9, "unit": "GMAC/s", "h2d_bytes_per_step": 4 * (rows * n + n * n),
               "d2h_bytes_per_step": 4 * rows * n, "ms_per_step": ems}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cm, dt, threads, desc = oracle_gemm_sample(n, args.model, args.m, args.cpu_budget)
            cpu = {"value": cm / dt / 1e9, "unit": "GMAC/s", "cores": threads, "kind": "oracle", "sample": desc,
                   **cpu_info()}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "GMAC/s", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GMAC/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded; A, B ~ N(0,1))",
            "config": {"workload": workload_label("gemm", args.model, args.m, n), "M": n, "N": n, "K": n,
                       "model": args.model, "m": args.m, "rows_per_gpu": [shard_batch(n, world, r)[1]
                                                                          for r in range(world)],
                       "parallelism": f"M-sharded over {world} GPU(s), B replicated",
                       "l2": f"inputs larger than L2 (B = {4 * n * n / 1e6:.0f} MB)" if 4 * n * n > 126e6
                       else "operands fit the 126 MB L2; not flushed"},
            "clocks": clk,
            "comm": comm,
            "e2e": e2e,
            "gpu_launches": launches,
            "allgather_ms": gather_ms,
            "roofline": {"bound": "alu", "kernel": "amsim_mm_kernel [gemm]", "achieved": achieved, "peak": peak,
                         "unit": "GMAC/s", "frac": achieved / peak, "traffic": None,
                         "algorithmic_bytes_per_launch": 4 * (2 * rows * n + n * n),
                         "frac_of_measured_lookup": (achieved / lut_meas) if isinstance(lut_meas, float) else None,
                         "peak_basis": "148 SMs x 32 LUT lookups/clk x max SM clock",
                         "lut_lookup_measured_gps": lut_meas, "ms_per_launch": per},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)


def relaunch(n: int, backend: str):
    """`python bench.py --gpus N` without torchrun: re-exec this command under
    torch.distributed.run with N processes (one per GPU) on 127.0.0.1."""
    import socket

    import torch
    if backend == "nccl" and torch.cuda.device_count() < n:
        raise SystemExit(f"bench.py: --gpus {n} with NCCL needs {n} visible GPUs, found {torch.cuda.device_count()}")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] relaunching as {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    os.execv(sys.executable, cmd)


def communicator_check(dist, world: int, rank: int, gpu: int, backend: str):
    """Force communicator creation with one collective, log it, and gather
    every rank's device (rank 0 reports them in the JSON line)."""
    import torch
    t0 = time.perf_counter()
    t = torch.ones(1, device=torch.device("cuda", gpu) if backend == "nccl" else "cpu")
    dist.all_reduce(t)
    if int(t.item()) != world:
        raise SystemExit(f"bench.py: all-reduce over the communicator gave {int(t.item())}, expected {world}")
    props = torch.cuda.get_device_properties(gpu)
    me = {"rank": rank, "gpu": gpu, "uuid": str(getattr(props, "uuid", "")), "host": os.uname().nodename}
    everyone = [None] * world
    dist.all_gather_object(everyone, me)
    ms = (time.perf_counter() - t0) * 1e3
    print(f"[bench] rank {rank}/{world}: {backend} communicator initialised (nranks={world}, cuda:{gpu}, "
          f"{ms:.0f} ms)", file=sys.stderr, flush=True)
    if backend == "nccl" and len({e["uuid"] for e in everyone}) != world:
        raise SystemExit("bench.py: NCCL ranks share a GPU; one rank per GPU is required")
    return {"backend": backend, "nranks": dist.get_world_size(), "init_ms": ms,
            "devices": [(e["rank"], e["gpu"], e["uuid"]) for e in everyone]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="amsim", choices=["amsim", "reference"])
    ap.add_argument("--workload", default="resnet50", choices=["resnet50", "resnet18", "lenet5", "gemm"],
                    help="gemm = BASELINE.json config 5: one M = N = K = --size approx GEMM, rows sharded over "
                         "the GPUs (strong scaling)")
    ap.add_argument("--size", type=int, default=16384, help="--workload gemm: M = N = K")
    ap.add_argument("--model", default="mbm", choices=["mbm", "exact", "mitchell"])
    ap.add_argument("--m", type=int, default=7)
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--ref-budget", type=float, default=8.0, help="seconds of oracle work per reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-exact-step", action="store_true",
                    help="skip timing the same step with the exact bf16 table (reported next to the MBM number)")
    ap.add_argument("--policy", type=int, default=0, help="amsim_set_path_policy bits (A/B experiments only)")
    ap.add_argument("--no-full-step", action="store_true",
                    help="skip the whole-network training / inference step measurement (net.py)")
    ap.add_argument("--graph", action="store_true",
                    help="N=1: replay the step as one CUDA graph in the timed regions (per-kind kernel times then "
                         "come from one extra eager step)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)

    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    backend = os.environ.get("AMSIM_DIST_BACKEND", "nccl")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch(args.gpus, backend)           # one process per GPU; does not return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: launched with WORLD_SIZE={world} but --gpus {args.gpus}")
    ndev = torch.cuda.device_count()
    comm = None
    if world > 1:
        # production: NCCL, one rank per GPU.  AMSIM_DIST_BACKEND=gloo lets ranks share
        # GPUs (gpu = local % count) to exercise the multi-rank path on a 1-GPU box
        if backend == "nccl" and ndev < world:
            raise SystemExit(f"bench.py: --gpus {world} with NCCL needs {world} visible GPUs, found {ndev} "
                             f"(AMSIM_DIST_BACKEND=gloo shares GPUs for functional tests only)")
        gpu = local % ndev
        torch.cuda.set_device(gpu)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
        comm = communicator_check(dist, world, rank, gpu, backend)
    else:
        if ndev < 1:
            raise SystemExit("bench.py: no CUDA device visible (no CPU fallback)")
        gpu = 0
        torch.cuda.set_device(0)
    dev = torch.device("cuda", gpu)

    import paper_2209_04161_b200 as am
    from paper_2209_04161_b200.dp import max_over_ranks, shard_batch
    from paper_2209_04161_b200.train_step import TrainStep

    if args.workload == "gemm":
        run_gemm(args, world, rank, gpu, dev, comm)
        if world > 1:
            dist.destroy_process_group()
        return

    gb = global_batch(args.workload)
    _, nb = shard_batch(gb, world, rank)
    layers, _ = workload_layers(args.workload, nb)
    lut = am.Lut.build(args.model, args.m)
    am.amsim_set_path_policy(args.policy)
    step = TrainStep(layers, lut, device=dev, seed=1000, first_input="mnist" if args.workload == "lenet5" else "relu")
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            if dist.get_backend() == "nccl":
                dist.barrier(device_ids=[gpu])
            else:
                dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step.step()
    barrier()
    use_graph = args.graph and world == 1
    run = step.step
    if use_graph:
        n0 = am.amsim_launch_count()
        step.step()
        launches_per_step = am.amsim_launch_count() - n0
        run = step.capture()
        for _ in range(max(args.warmup, 1)):
            run()
        barrier()

    # ---- timed region (device-resident inputs) ----
    clocks = ClockSampler(gpu)
    clocks.start()
    step.timers = None if use_graph else []
    launches0 = am.amsim_launch_count()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        run()
    e1.record()
    barrier()
    # graph replays bypass the library's launch counter: count the captured launches
    launches = launches_per_step * args.steps if use_graph else am.amsim_launch_count() - launches0
    clk = clocks.stop()
    if use_graph:   # per-kind kernel times from one extra eager step
        step.timers = []
        step.step()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms, dev)
    total_macs = sum(l.macs() * (2 if l.first else 3) for l in workload_layers(args.workload, gb)[0])
    value = total_macs / (ms * 1e-3) / 1e9

    # per-kernel-kind device time (events around every launch, same stream)
    kinds = {}
    for kind, macs, a, b in step.timers:
        t = a.elapsed_time(b)
        k = kinds.setdefault(kind, [0.0, 0, 0])
        k[0] += t
        k[1] += macs
        k[2] += 1
    step.timers = None
    dom = max(kinds.items(), key=lambda kv: kv[1][0])
    dom_kind, (dom_ms, dom_macs, dom_n) = dom
    achieved = dom_macs / (dom_ms * 1e-3) / 1e9
    props = torch.cuda.get_device_properties(dev)
    sm_max = clk.get("sm_max_mhz") or 1965.0
    peak = props.multi_processor_count * 32 * sm_max * 1e6 / 1e9   # 32 LUT lookups/clk/SM

    # measured LUT-lookup rate (same m, 16-bit layout, warp-shared row, data-like index mix)
    lut_meas = None
    try:
        import numpy as np
        idx = np.random.default_rng(0).integers(0, 1 << args.m, 1 << 16).astype(np.uint32)
        lut_meas = am.amsim_bench_lut_lookup(args.m, lut.info()[1], idx, iters=2048) / 1e9
    except Exception as ex:  # noqa: BLE001
        lut_meas = f"unavailable: {ex}"

    # ---- the same step with the exact (bfloat16-by-truncation) table: every
    # product pinned to the IEEE product of truncated operands,
    # so this rate has no stand-in model behind it ----
    exact_step = None
    zero_frac = step.activation_zero_fraction()
    if not args.no_exact_step and args.model != "exact" and not use_graph:
        step.set_lut(am.Lut.build("exact", args.m))
        for _ in range(2):
            step.step()
        barrier()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record()
        for _ in range(args.steps):
            step.step()
        x1.record()
        barrier()
        xms = max_over_ranks(x0.elapsed_time(x1) / args.steps, dev)
        exact_step = {"model": "exact", "m": args.m, "ms_per_step": xms,
                      "value": total_macs / (xms * 1e-3) / 1e9, "unit": "GMAC/s",
                      "note": "same step, exact table: products pinned to the IEEE product of bf16-truncated operands"}
        step.set_lut(lut)

    # ---- end to end: pinned host input -> device, step, gradients -> host ----
    e2e = None
    if not args.no_e2e:
        xin = step.input_tensor()
        host_in = torch.empty(xin.shape, dtype=xin.dtype, pin_memory=True)
        host_in.copy_(xin)
        host_out = torch.empty(step.flat_grad.shape, dtype=torch.float32, pin_memory=True)
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            xin.copy_(host_in, non_blocking=True)
            run()
            host_out.copy_(step.flat_grad, non_blocking=True)
        f1.record()
        barrier()
        ems = max_over_ranks(f0.elapsed_time(f1) / args.steps, dev)
        e2e = {"value": total_macs / (ems * 1e-3) / 1e9, "unit": "GMAC/s",
               "h2d_bytes_per_step": host_in.numel() * 4, "d2h_bytes_per_step": host_out.numel() * 4,
               "ms_per_step": ems}

    # ---- whole training step (NEXT(1)): the same approximate passes plus BN, ReLU,
    # pooling, residual adds, loss and SGD (net.py); graph replay on one GPU,
    # eager with the bucketed all-reduce on several ----
    full = None
    if not args.no_full_step:
        from paper_2209_04161_b200 import net as netmod
        del step, run
        torch.cuda.empty_cache()
        net = netmod.BUILDERS[args.workload](lut, batch=nb, device=dev, seed=1000)
        net.train_step()
        tr = net.capture(net.train_step) if world == 1 else net.train_step
        for _ in range(args.warmup):
            tr()
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(args.steps):
            tr()
        g1.record()
        barrier()
        full_ms = max_over_ranks(g0.elapsed_time(g1) / args.steps, dev)
        net.infer_step()
        inf = net.capture(net.infer_step) if world == 1 else net.infer_step
        inf()
        barrier()
        g0.record()
        for _ in range(args.steps):
            inf()
        g1.record()
        barrier()
        infer_ms = max_over_ranks(g0.elapsed_time(g1) / args.steps, dev)
        full = {"train_ms": full_ms, "infer_ms": infer_ms, "approx_passes_share": ms / full_ms,
                "loss": float(net.loss_value.item()), "cuda_graph": world == 1,
                "what": "forward + softmax-xent + backward + SGD-momentum of the whole network (BN, ReLU, pooling, "
                        "residual adds in native FP32 kernels, include/amsim_nn.h); infer = forward with running "
                        "BN statistics"}
        del net, tr, inf
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            macs, dt, threads, desc, kept = oracle_sample(args.workload, args.model, args.m, args.cpu_budget, keep=6)
            cpu = {"value": macs / dt / 1e9, "unit": "GMAC/s", "cores": threads, "kind": "oracle", "sample": desc,
                   **cpu_info(), "sample_parity": sample_parity(am, lut, kept)}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "GMAC/s", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"failed: {ex}", **cpu_info()}

    # DRAM traffic of the dominant kernel kind per layer pass, from the committed
    # ncu launch list of this same command (profiles/; tools/summarize_launches.py)
    traffic, traffic_note = None, None
    tpath = next((os.path.join(ROOT, "profiles", f) for f in ("r02c_traffic.json", "r02b_traffic.json", "r02_traffic.json", "r01_traffic.json")
                  if os.path.exists(os.path.join(ROOT, "profiles", f))), "")
    if args.workload == "resnet50" and os.path.exists(tpath):
        t = json.load(open(tpath)).get(dom_kind)
        if t:
            traffic = t["dram_bytes_per_pass"]
            traffic_note = (f"ncu dram bytes per {dom_kind} pass (avg over {t['layer_passes']} passes) from "
                            f"profiles/{os.path.basename(tpath)}; algorithmic 4(|X|+|W|+|Y|) = "
                            f"{t['algorithmic_bytes_per_pass']:.4g} B/pass (ratio {t['ratio']:.3f})")

    ws_bytes = 0
    for l in layers:
        if hasattr(l, "H"):
            ws_bytes += 4 * (l.N * l.H * l.W * l.C + l.R * l.S * l.C * l.K + l.N * l.OH * l.OW * l.K)
        else:
            ws_bytes += 4 * (l.N * l.IN + l.IN * l.OUT + l.N * l.OUT)
    l2_note = (f"inputs larger than L2 (per-step working set {ws_bytes / 1e9:.1f} GB per GPU)" if ws_bytes > 126e6
               else f"per-step working set {ws_bytes / 1e6:.1f} MB fits the 126 MB L2; not flushed (latency-bound "
                    f"workload)")

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GMAC/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded; ReLU(N(0,1)) activations, He-normal weights, N(0,2^-10) errors)",
            "config": {"workload": workload_label(args.workload, args.model, args.m), "global_batch": gb,
                       "per_gpu_batch": nb, "model": args.model, "m": args.m,
                       "macs_per_step": total_macs, "parallelism": f"dp{world}",
                       "activation_zero_fraction": zero_frac,
                       "l2": l2_note,
                       "cuda_graph": use_graph},
            "clocks": clk,
            "comm": comm,
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": {"bound": "alu", "kernel": f"amsim_mm_kernel [{dom_kind}]", "achieved": achieved,
                         "peak": peak, "unit": "GMAC/s", "frac": achieved / peak, "traffic": traffic,
                         "traffic_note": traffic_note,
                         "frac_of_measured_lookup": (achieved / lut_meas) if isinstance(lut_meas, float) else None,
                         "peak_basis": "148 SMs x 32 LUT lookups/clk (conflict-free LDS = 4-instr/MAC issue "
                                       "ceiling) x max SM clock",
                         "lut_lookup_measured_gps": lut_meas,
                         "per_kind_ms_per_step": {k: v[0] / args.steps for k, v in kinds.items()},
                         "per_kind_gmacs": {k: v[1] / (v[0] * 1e-3) / 1e9 for k, v in kinds.items()}},
            "cpu_baseline": cpu,
            "exact_bf16_step": exact_step,
            "full_train_step": full,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
