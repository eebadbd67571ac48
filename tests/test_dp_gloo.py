"""Data-parallel host logic on CPU with torch.distributed gloo, world size 2
(the N > 1 path of bench.py: batch sharding, bucketed weight-gradient
all-reduce, max-over-ranks timing).  No GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_04161_b200.dp import GradAllReducer, max_over_ranks, plan_buckets, shard_batch


def test_shard_batch_covers_every_sample_once():
    for gb in (1, 7, 64, 128, 255, 256):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                s, c = shard_batch(gb, world, r)
                seen += list(range(s, s + c))
            assert seen == list(range(gb))


def test_plan_buckets_ready_order_and_contiguity():
    numels = [100, 5, 5000, 70, 3000, 1, 1]
    offsets, buckets, total = plan_buckets(numels, 4000)
    assert total == sum(numels)
    # laid out in reverse layer order (the order backward produces them)
    order = sorted(range(len(numels)), key=lambda i: offsets[i])
    assert order == list(range(len(numels)))[::-1]
    covered = []
    for b in buckets:
        assert sum(numels[i] for i in b.layers) == b.numel
        assert b.offset == min(offsets[i] for i in b.layers)
        covered += b.layers
    assert covered == list(range(len(numels)))[::-1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        numels = [7, 300, 11, 4096, 3]
        offsets, buckets, total = plan_buckets(numels, 512)
        flat = torch.zeros(total)
        red = GradAllReducer(flat, buckets)
        assert red.world == world
        # "backward": gradients become ready in reverse layer order
        for li in range(len(numels) - 1, -1, -1):
            flat.narrow(0, offsets[li], numels[li]).fill_(float((rank + 1) * (li + 1)))
            red.ready(li)
        red.finish()
        expect = torch.cat([torch.full((numels[li],), float(sum(r + 1 for r in range(world)) * (li + 1)))
                            for li in sorted(range(len(numels)), key=lambda i: offsets[i])])
        ok_sum = torch.equal(flat, expect)
        mx = max_over_ranks(10.0 + rank)

        # sharded wgrad through the oracle + all-reduce == full-batch wgrad
        import amsim_inputs as inp
        import oracle
        N, H, W, C, K, R, S, st, pd = 4, 6, 6, 3, 5, 3, 3, 2, 1
        d = oracle.conv_desc(N, H, W, C, K, R, S, st, pd)
        x = inp.relu_normal((N, H, W, C), 1)
        dy = inp.normal((N, d.OH, d.OW, K), 2)
        s0, cnt = shard_batch(N, world, rank)
        ds = oracle.conv_desc(cnt, H, W, C, K, R, S, st, pd)
        part = oracle.conv_bwd_filter(ds, x[s0:s0 + cnt], dy[s0:s0 + cnt], "mitchell")
        g = torch.from_numpy(part.c64.copy())
        dist.all_reduce(g)
        full = oracle.conv_bwd_filter(d, x, dy, "mitchell")
        ok_dp = bool(np.all(np.abs(g.numpy() - full.c64) <= 1e-5 * full.abs64 + np.finfo(np.float32).tiny))
        q.put((rank, ok_sum, mx, ok_dp))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_allreduce_and_timing():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_sum, mx, ok_dp in res:
        assert ok_sum, f"rank {rank}: bucketed all-reduce gave a wrong sum"
        assert mx == 11.0, "max over ranks"
        assert ok_dp, f"rank {rank}: sharded + all-reduced wgrad differs from full batch"


def test_single_process_reducer_is_noop():
    offsets, buckets, total = plan_buckets([3, 4], 100)
    flat = torch.arange(total, dtype=torch.float32)
    red = GradAllReducer(flat, buckets)
    red.ready(1)
    red.ready(0)
    red.finish()
    assert torch.equal(flat, torch.arange(total, dtype=torch.float32))


class _OracleGemm:
    """Stand-in for the binding's amsim_gemm on CPU tensors (test-only): the
    oracle's FP32 c32 result of the same rows."""

    @staticmethod
    def amsim_gemm(lut, A, B, C, stream=None):
        import oracle
        C.copy_(torch.from_numpy(oracle.gemm(A.numpy(), B.numpy(), "mitchell", 7).c32))
        return C


def _gemm_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import amsim_inputs as inp
        import oracle
        from paper_2209_04161_b200.dp import gather_rows, sharded_gemm
        M, N, K = 7, 5, 9          # ragged: 4 + 3 rows
        A = torch.from_numpy(inp.normal((M, K), 1))
        B = torch.from_numpy(inp.normal((K, N), 2))
        C = torch.full((M, N), float("nan"))
        r0, n = sharded_gemm(_OracleGemm, None, A, B, C, world, rank)
        untouched = bool(torch.isnan(torch.cat([C[:r0], C[r0 + n:]])).all())
        full = gather_rows(C[r0:r0 + n], M, world)
        ref = oracle.gemm(A.numpy(), B.numpy(), "mitchell", 7).c32
        same = np.array_equal(full.numpy().view(np.uint32), ref.view(np.uint32))
        q.put((rank, r0, n, untouched, same))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_gemm_rows_and_gather():
    """SURVEY.md §8(e) GEMM: M rows partitioned over 2 ranks, each writes only
    its rows, the all-gather reassembles the single-process result bit-exactly."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gemm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(r0, n) for _, r0, n, _, _ in res] == [(0, 4), (4, 3)]
    for rank, _, _, untouched, same in res:
        assert untouched, f"rank {rank} wrote rows outside its shard"
        assert same, f"rank {rank}: gathered rows differ from the single-process GEMM"
