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
