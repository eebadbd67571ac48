"""Data-parallel plumbing: batch sharding and the bucketed weight-gradient
all-reduce (the paper's multi-GPU runs used Horovod gradient all-reduce,
PAPER.md:733; here NCCL via torch.distributed over NVLink / NVSwitch).

Device-agnostic torch.distributed code (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass, field


def shard_batch(global_batch: int, world: int, rank: int):
    """Contiguous batch shard of `rank`: (start, count).  Remainders go to the
    lowest ranks so every sample is processed exactly once."""
    base, rem = divmod(global_batch, world)
    count = base + (1 if rank < rem else 0)
    start = rank * base + min(rank, rem)
    return start, count


def sharded_gemm(am, lut, A, B, C, world: int, rank: int, stream=None):
    """SURVEY.md §8(e), GEMM (config 5): rows of A and C are partitioned into
    `world` contiguous blocks (shard_batch); B and the table are replicated.
    Rank `rank` computes C[r0:r0+n] = A[r0:r0+n] · B through amsim_gemm.  The
    rows of an AMSim GEMM are independent and the per-row summation order does
    not depend on M, so the blocks are bit-identical to the same rows of the
    single-GPU result (tests/test_gpu_parity.py::test_gemm_row_shards_bit_identical).
    A [M, K] and C [M, N] are the full row-major matrices (only this rank's
    rows of A are read and of C written).  Returns (r0, n)."""
    if C.shape[0] != A.shape[0]:
        raise ValueError("A and C must have the same number of rows")
    r0, n = shard_batch(C.shape[0], world, rank)
    if n:
        am.amsim_gemm(lut, A[r0:r0 + n], B, C[r0:r0 + n], stream=stream)
    return r0, n


def gather_rows(C_local, M: int, world: int, out=None):
    """All-gather the row blocks of sharded_gemm into the full M-row matrix on
    every rank (NCCL all_gather_into_tensor on equal, padded blocks; the
    optional, separately timed step of §8(e)).  C_local holds this rank's
    shard_batch rows.  Returns the gathered [M, N] tensor."""
    import torch
    import torch.distributed as dist
    rows = -(-M // world)
    N = C_local.shape[1]
    pad = torch.zeros((rows, N), dtype=C_local.dtype, device=C_local.device)
    pad[:C_local.shape[0]].copy_(C_local)
    full = torch.empty((rows * world, N), dtype=C_local.dtype, device=C_local.device)
    dist.all_gather_into_tensor(full, pad)
    if out is None:
        out = torch.empty((M, N), dtype=C_local.dtype, device=C_local.device)
    for r in range(world):
        s, n = shard_batch(M, world, r)
        out[s:s + n].copy_(full[r * rows:r * rows + n])
    return out


@dataclass
class Bucket:
    layers: list            # layer indices (in the order their gradients become ready)
    offset: int             # element offset in the flat gradient buffer
    numel: int
    pending: set = field(default_factory=set)


def plan_buckets(grad_numels, bucket_elems: int):
    """Lay gradients out in READY order (reverse layer order: backward
    finishes the last layer first) and group consecutive ones into buckets of
    about `bucket_elems` elements.  Returns (offsets per layer, buckets)."""
    order = list(range(len(grad_numels)))[::-1]
    offsets = [0] * len(grad_numels)
    buckets = []
    cur, cur_off, off = [], 0, 0
    for li in order:
        offsets[li] = off
        cur.append(li)
        off += grad_numels[li]
        if off - cur_off >= bucket_elems:
            buckets.append(Bucket(cur, cur_off, off - cur_off))
            cur, cur_off = [], off
    if cur:
        buckets.append(Bucket(cur, cur_off, off - cur_off))
    return offsets, buckets, off


class GradAllReducer:
    """Launches one all-reduce (SUM) per bucket as soon as every gradient in it
    is ready, on a dedicated communication stream so it overlaps the rest of
    the backward pass.  With world == 1 it is a no-op."""

    def __init__(self, flat, buckets, group=None, comm_stream=None):
        import torch.distributed as dist
        self.flat = flat
        self.buckets = buckets
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.comm_stream = comm_stream
        self.layer_to_bucket = {li: bi for bi, b in enumerate(buckets) for li in b.layers}
        self.works = []
        self.reset()

    def reset(self):
        for b in self.buckets:
            b.pending = set(b.layers)
        self.works = []

    def ready(self, layer: int):
        """Gradient of `layer` has been enqueued on the current stream."""
        if self.world == 1:
            return
        b = self.buckets[self.layer_to_bucket[layer]]
        b.pending.discard(layer)
        if not b.pending:
            self._launch(b)

    def _launch(self, b: Bucket):
        import torch
        import torch.distributed as dist
        view = self.flat.narrow(0, b.offset, b.numel)
        if self.flat.is_cuda and self.comm_stream is not None:
            self.comm_stream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(self.comm_stream):
                self.works.append(dist.all_reduce(view, op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        else:
            self.works.append(dist.all_reduce(view, op=dist.ReduceOp.SUM, group=self.group, async_op=True))

    def finish(self):
        """Make the current stream wait for every launched all-reduce."""
        for w in self.works:
            w.wait()
        self.works = []


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the bench's slowest-rank timing rule)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
