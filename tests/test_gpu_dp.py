"""Data-parallel path on CUDA tensors:
2 / 3 / 4 ranks on ONE GPU (torch.distributed gloo, every rank on cuda:0 --
this pool's boxes have one GPU, NCCL refuses two ranks per device) run the
real multi-rank code -- batch shards, TrainStep / Net with the bucketed
all-reduce launched on the communication stream as gradients become ready,
Work.wait() before the update -- and the all-reduced gradients are compared
with the single-process full batch:

  * TrainStep (the bench's approximate passes): every weight gradient against
    the ORACLE's full-batch wgrad, |g - c64| <= 1e-5 * sum|p| + FLT_MIN
    (reading C12; the shard sum only reorders the FP32 accumulation), and the
    ranks' reduced buffers bit-identical to each other;
  * Net (whole LeNet-5 training step: bias / ReLU / pooling / loss / SGD):
    the reduced gradient and the SGD-updated weights against a world-1 run of
    the same global batch, within an accumulation-order tolerance -- with
    uneven shards at world 3 (the loss gradient is divided by the global
    batch, so no rank's shard size biases the mean; weight decay unscaled).
"""
import os
import socket

import numpy as np
import pytest

import amsim_inputs as inp

pytestmark = pytest.mark.gpu

FLT_MIN = np.finfo(np.float32).tiny
GB = 64                                   # LeNet-5 global batch (BASELINE.json config 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, what, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2209_04161_b200 as am
        from amsim_inputs import device as gen
        from paper_2209_04161_b200.dp import shard_batch
        lut = am.Lut.build("mbm", 7)
        s0, c = shard_batch(GB, world, rank)
        if what == "trainstep":
            from paper_2209_04161_b200.train_step import TrainStep
            layers = inp.lenet5_layers(GB)
            full = TrainStep(layers, lut, device="cuda", seed=5, first_input="mnist")   # inputs only
            step = TrainStep([l.with_batch(c) for l in layers], lut, device="cuda", seed=5, first_input="mnist")
            assert step.reducer.world == world
            for ly, lf in zip(step.layers, full.layers):
                ly.x.copy_(lf.x[s0:s0 + c])
                ly.dy.copy_(lf.dy[s0:s0 + c])
            del full
            step.step()
            torch.cuda.synchronize()
            q.put((rank, step.flat_grad.cpu().numpy(), None))
        else:
            from paper_2209_04161_b200 import net as netmod
            net = netmod.lenet5(lut, batch=c, device="cuda", seed=1)
            assert net.reducer.world == world and net.global_batch == GB
            x = gen.mnist_like((GB, 28, 28, 1), 1 + 101, device="cuda")
            g = torch.Generator(device="cuda")
            g.manual_seed(1 + 202)
            labels = torch.randint(0, 10, (GB,), generator=g, device="cuda", dtype=torch.int32)
            net.input.data.copy_(x[s0:s0 + c])
            net.labels.copy_(labels[s0:s0 + c])
            net.train_step()
            torch.cuda.synchronize()
            q.put((rank, net.flat_g.cpu().numpy(), net.flat_w.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def _spawn(world, what):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, what, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0, f"rank process exited with {p.exitcode}"
    return res


@pytest.fixture(scope="module")
def am():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"
    from paper_2209_04161_b200 import build
    build.build()
    import paper_2209_04161_b200 as am
    return am


@pytest.mark.parametrize("world", [2, 4])
def test_trainstep_allreduce_equals_full_batch_oracle(am, orc, world):
    import torch

    from paper_2209_04161_b200.train_step import TrainStep
    res = _spawn(world, "trainstep")
    for r in range(1, world):   # every rank holds the same reduced buffer
        assert np.array_equal(res[r][1].view(np.uint32), res[0][1].view(np.uint32)), f"rank {r} differs"
    flat = res[0][1]
    lut = am.Lut.build("mbm", 7)
    full = TrainStep(inp.lenet5_layers(GB), lut, device="cuda", seed=5, first_input="mnist")
    for ly in full.layers:
        l = ly.spec
        off = ly.dw.storage_offset()
        got = flat[off:off + ly.dw.numel()]
        x, dy = ly.x.cpu().numpy(), ly.dy.cpu().numpy()
        if ly.kind == "conv":
            d = orc.conv_desc(l.N, l.H, l.W, l.C, l.K, l.R, l.S, l.stride, l.pad)
            ref = orc.conv_bwd_filter(d, x, dy, "mbm")
        else:
            ref = orc.gemm(np.ascontiguousarray(x.T), dy, "mbm")
        got = got.reshape(ref.c64.shape).astype(np.float64)
        err = np.abs(got - ref.c64)
        tol = 1e-5 * ref.abs64 + FLT_MIN
        assert np.all(err <= tol), f"{l.name}: worst |err|/tol = {np.max(err / tol):.3g}"
    del full
    torch.cuda.empty_cache()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_net_train_step_allreduce_equals_world1(am, world):
    import torch

    from paper_2209_04161_b200 import net as netmod
    res = _spawn(world, "net")
    lut = am.Lut.build("mbm", 7)
    ref = netmod.lenet5(lut, batch=GB, device="cuda", seed=1)
    w0 = ref.flat_w.clone()
    ref.train_step()
    torch.cuda.synchronize()
    g1, w1 = ref.flat_g.cpu().numpy().astype(np.float64), ref.flat_w.cpu().numpy().astype(np.float64)
    for r in range(world):
        g, w = res[r][1].astype(np.float64), res[r][2].astype(np.float64)
        for p in ref.params:
            off, n = p.grad.storage_offset(), p.numel
            scale = np.max(np.abs(g1[off:off + n])) + FLT_MIN
            dg = np.max(np.abs(g[off:off + n] - g1[off:off + n]))
            assert dg <= 2e-5 * scale, f"rank {r} {p.name}: gradient |diff| {dg:.3g} vs max|g| {scale:.3g}"
            dw = np.max(np.abs(w[off:off + n] - w1[off:off + n]))
            assert dw <= ref.lr * 2e-5 * scale * 2 + 1e-7 * np.max(np.abs(w1[off:off + n])), \
                f"rank {r} {p.name}: updated weights differ by {dw:.3g}"
    # the update moved the weights (the comparison is not vacuous)
    assert torch.max(torch.abs(ref.flat_w - w0)).item() > 0
    del ref
    torch.cuda.empty_cache()
