"""Full training / inference steps: the native-FP32
layer kernels of include/amsim_nn.h against PyTorch FP64 references, and whole
networks (net.py) against a PyTorch FP64 autograd model of the same graph.

The whole-network check runs the AMSim passes in AMSIM_MUL_NATIVE mode, so the
reference is plain FP32 / FP64 arithmetic and the tolerance can be tight; the
AMSim passes themselves are pinned against the oracle in test_gpu_parity.py.
"""
import math

import numpy as np
import pytest

import amsim_inputs as inp


# ---------------------------------------------------------------------------
# CPU: graph structure

@pytest.mark.parametrize("name,layers", [("lenet5", inp.lenet5_layers), ("resnet18", inp.resnet18_cifar_layers),
                                         ("resnet50", inp.resnet50_layers)])
def test_net_approx_layers_match_workloads(name, layers):
    """The full networks' Conv2D / Dense layers are exactly the bench's
    approximate layer lists (same shapes, same MACs per step)."""
    from paper_2209_04161_b200 import net as netmod
    batch = {"lenet5": 64, "resnet18": 128, "resnet50": 256}[name]
    net = netmod.BUILDERS[name](None, batch=batch, build_only=True)
    want = layers(batch)
    convs = [n for n in net.nodes if type(n).__name__ in ("_Conv", "_Dense")]
    assert len(convs) == len(want)
    assert net.approx_macs == inp.workloads.step_macs(want)
    for n, l in zip(convs, want):
        if type(n).__name__ == "_Conv":
            d = n.d
            assert (d.N, d.H, d.W, d.C, d.K, d.R, d.S, d.stride_h, d.pad_h) == \
                   (l.N, l.H, l.W, l.C, l.K, l.R, l.S, l.stride, l.pad), l.name
        else:
            assert (n.x.shape[0], n.IN, n.w.shape[1]) == (l.N, l.IN, l.OUT), l.name


# ---------------------------------------------------------------------------
# GPU: layer kernels vs PyTorch FP64

def _t(a):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a, np.float32)).cuda()


@pytest.fixture(scope="module")
def am():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"
    from paper_2209_04161_b200 import build
    build.build()
    import paper_2209_04161_b200 as am
    return am


def _close(got, want, rtol, what=""):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    scale = max(np.abs(want).max(), 1e-30)
    err = np.abs(got - want).max()
    assert err <= rtol * scale, f"{what}: max err {err:.3g} vs scale {scale:.3g}"


@pytest.mark.gpu
@pytest.mark.parametrize("P,C,relu,res", [(1000, 64, True, False), (777, 6, True, True), (4096, 256, False, True),
                                          (50, 2048, True, True), (3, 5, False, False)])
def test_bn_train_fwd_bwd_vs_torch(am, P, C, relu, res):
    import torch
    from paper_2209_04161_b200 import _lib as L
    g = np.random.default_rng(P + C)
    x = g.normal(0.5, 2.0, (P, C)).astype(np.float32)
    gam = g.normal(1.0, 0.3, C).astype(np.float32)
    bet = g.normal(0.0, 0.3, C).astype(np.float32)
    r = g.normal(0, 1, (P, C)).astype(np.float32) if res else None
    dy = g.normal(0, 1, (P, C)).astype(np.float32)
    # device
    X, G, B, Y = _t(x), _t(gam), _t(bet), torch.empty(P, C, device="cuda")
    R = _t(r) if res else None
    mean, invstd = torch.empty(C, device="cuda"), torch.empty(C, device="cuda")
    rm, rv = torch.zeros(C, device="cuda"), torch.ones(C, device="cuda")
    ws = torch.empty(L.amsim_nn_workspace_bytes(P, C) // 4 + 1, device="cuda")
    L.amsim_bn_fwd_train(X, P, C, G, B, 1e-5, R, relu, Y, mean, invstd, rm, rv, 0.1, ws)
    DX, DG, DB = torch.empty(P, C, device="cuda"), torch.empty(C, device="cuda"), torch.empty(C, device="cuda")
    DR = torch.empty(P, C, device="cuda") if res else None
    L.amsim_bn_bwd(_t(dy), Y, X, P, C, G, mean, invstd, relu, DX, DR, DG, DB, ws)
    torch.cuda.synchronize()
    # reference
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    gt = torch.tensor(gam, dtype=torch.float64, requires_grad=True)
    bt = torch.tensor(bet, dtype=torch.float64, requires_grad=True)
    rt = torch.tensor(r, dtype=torch.float64, requires_grad=True) if res else None
    m = xt.mean(0)
    v = xt.var(0, unbiased=False)
    yt = (xt - m) / torch.sqrt(v + 1e-5) * gt + bt
    if res:
        yt = yt + rt
    if relu:
        yt = torch.relu(yt)
    yt.backward(torch.tensor(dy, dtype=torch.float64))
    _close(Y.cpu(), yt.detach(), 2e-5, "y")
    _close(mean.cpu(), m.detach(), 1e-5, "mean")
    _close(rm.cpu(), 0.1 * m.detach(), 1e-5, "running mean")
    _close(rv.cpu(), 0.9 + 0.1 * xt.var(0, unbiased=True).detach() if P > 1 else rv.cpu(), 1e-5, "running var")
    _close(DX.cpu(), xt.grad, 1e-4, "dx")
    _close(DG.cpu(), gt.grad, 1e-4, "dgamma")
    _close(DB.cpu(), bt.grad, 1e-4, "dbeta")
    if res:
        _close(DR.cpu(), rt.grad, 1e-6, "dres")
    # inference mode with the running statistics
    Y2 = torch.empty(P, C, device="cuda")
    L.amsim_bn_fwd_infer(X, P, C, G, B, rm, rv, 1e-5, R, relu, Y2)
    yi = (torch.tensor(x, dtype=torch.float64) - torch.tensor(rm.cpu().numpy(), dtype=torch.float64)) / \
        torch.sqrt(torch.tensor(rv.cpu().numpy(), dtype=torch.float64) + 1e-5) * gt.detach() + bt.detach()
    if res:
        yi = yi + torch.tensor(r, dtype=torch.float64)
    if relu:
        yi = torch.relu(yi)
    _close(Y2.cpu(), yi, 2e-5, "infer")


@pytest.mark.gpu
def test_bn_deterministic(am):
    import torch
    from paper_2209_04161_b200 import _lib as L
    P, C = 20000, 96
    X = torch.randn(P, C, device="cuda")
    G, B = torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")
    ws = torch.empty(L.amsim_nn_workspace_bytes(P, C) // 4 + 1, device="cuda")
    outs = []
    for _ in range(2):
        Y, m, s = torch.empty(P, C, device="cuda"), torch.empty(C, device="cuda"), torch.empty(C, device="cuda")
        L.amsim_bn_fwd_train(X, P, C, G, B, 1e-5, None, True, Y, m, s, None, None, 0.1, ws)
        outs.append((Y.clone(), m.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.gpu
@pytest.mark.parametrize("relu", [True, False])
def test_bias_act_vs_torch(am, relu):
    import torch
    from paper_2209_04161_b200 import _lib as L
    P, C = 3000, 84
    x = torch.randn(P, C, device="cuda")
    b = torch.randn(C, device="cuda")
    y = torch.empty_like(x)
    L.amsim_bias_act_fwd(x, P, C, b, relu, y)
    want = x + b
    if relu:
        want = torch.relu(want)
    assert torch.allclose(y, want, atol=0, rtol=0)
    dy = torch.randn(P, C, device="cuda")
    dx, db = torch.empty_like(x), torch.empty(C, device="cuda")
    ws = torch.empty(L.amsim_nn_workspace_bytes(P, C) // 4 + 1, device="cuda")
    L.amsim_bias_act_bwd(dy, y, P, C, relu, dx, db, ws)
    dz = dy * (y > 0) if relu else dy
    assert torch.equal(dx, dz)
    _close(db.cpu(), dz.double().sum(0).cpu(), 1e-5, "dbias")


@pytest.mark.gpu
@pytest.mark.parametrize("geom", [(2, 9, 11, 5, 3, 2, 1), (3, 8, 8, 16, 2, 2, 0), (1, 7, 7, 3, 3, 1, 1)])
def test_maxpool_vs_torch(am, geom):
    import torch
    from paper_2209_04161_b200 import _lib as L
    N, H, W, C, R, st, pad = geom
    x = torch.randn(N, H, W, C, device="cuda")
    OH, OW = (H + 2 * pad - R) // st + 1, (W + 2 * pad - R) // st + 1
    y = torch.empty(N, OH, OW, C, device="cuda")
    am_ = torch.empty(N, OH, OW, C, device="cuda", dtype=torch.uint8)
    L.amsim_maxpool_fwd(x, N, H, W, C, R, R, st, pad, y, am_)
    xt = x.double().permute(0, 3, 1, 2).clone().requires_grad_(True)
    yt = torch.nn.functional.max_pool2d(xt, R, st, pad)
    assert torch.equal(y, yt.detach().permute(0, 2, 3, 1).float())
    dy = torch.randn(N, OH, OW, C, device="cuda")
    dx = torch.empty_like(x)
    L.amsim_maxpool_bwd(dy, am_, N, H, W, C, R, R, st, pad, dx)
    yt.backward(dy.double().permute(0, 3, 1, 2))
    _close(dx.cpu(), xt.grad.permute(0, 2, 3, 1).cpu(), 1e-6, "dx")


@pytest.mark.gpu
def test_avgpool_softmax_add_sgd_vs_torch(am):
    import torch
    from paper_2209_04161_b200 import _lib as L
    N, HW, C = 6, 49, 40
    x = torch.randn(N, HW, C, device="cuda")
    y = torch.empty(N, C, device="cuda")
    L.amsim_avgpool_fwd(x, N, HW, C, y)
    _close(y.cpu(), x.double().mean(1).cpu(), 1e-6, "avgpool")
    dy = torch.randn(N, C, device="cuda")
    dx = torch.empty_like(x)
    L.amsim_avgpool_bwd(dy, N, HW, C, dx)
    _close(dx.cpu(), (dy.double()[:, None, :] / HW).expand(N, HW, C).cpu(), 1e-6, "avgpool bwd")
    # softmax cross-entropy
    K = 1000
    z = torch.randn(N, K, device="cuda") * 3
    lab = torch.randint(0, K, (N,), device="cuda", dtype=torch.int32)
    loss, dz = torch.empty(1, device="cuda"), torch.empty(N, K, device="cuda")
    ws = torch.empty(L.amsim_nn_workspace_bytes(N, 1) // 4 + 1, device="cuda")
    L.amsim_softmax_xent(z, lab, N, K, loss, dz, ws)
    zt = z.double().cpu().requires_grad_(True)
    lt = torch.nn.functional.cross_entropy(zt, lab.long().cpu())
    lt.backward()
    _close(loss.cpu(), lt.detach().reshape(1), 1e-5, "loss")
    _close(dz.cpu(), zt.grad, 1e-5, "dlogits")
    # add, sgd
    a, b, o = torch.randn(1001, device="cuda"), torch.randn(1001, device="cuda"), torch.empty(1001, device="cuda")
    L.amsim_add(a, b, o, 1001)
    assert torch.equal(o, a + b)
    w, g, v = torch.randn(999, device="cuda"), torch.randn(999, device="cuda"), torch.randn(999, device="cuda")
    w0, v0 = w.clone(), v.clone()
    L.amsim_sgd_momentum(w, g, v, 999, 0.1, 0.9, 1e-3)
    v_want = 0.9 * v0 + g + 1e-3 * w0
    _close(v.cpu(), v_want.cpu(), 1e-6, "v")
    _close(w.cpu(), (w0 - 0.1 * v_want).cpu(), 1e-6, "w")


# ---------------------------------------------------------------------------
# GPU: whole networks vs a PyTorch FP64 autograd model of the same graph

def _reference_grads(net):
    """Evaluate the Net's graph with torch FP64 autograd from its parameters
    and input; returns (loss, {param name: grad})."""
    import torch
    F = torch.nn.functional
    vals = {}
    params = {p.name: p.data.detach().double().cpu().clone().requires_grad_(True) for p in net.params}
    vals[id(net.tensors[0])] = net.tensors[0].data.detach().double().cpu()
    for n in net.nodes:
        kind = type(n).__name__
        if kind == "_Conv":
            x = vals[id(n.x)].permute(0, 3, 1, 2)
            w = params[n.w.name].permute(3, 2, 0, 1)
            y = F.conv2d(x, w, None, n.d.stride_h, n.d.pad_h).permute(0, 2, 3, 1)
            vals[id(n.out)] = y
        elif kind == "_Dense":
            x = vals[id(n.x)].reshape(n.x.shape[0], -1)
            vals[id(n.out)] = x @ params[n.w.name]
        elif kind == "_BN":
            x = vals[id(n.x)]
            dims = tuple(range(x.dim() - 1))
            m = x.mean(dims)
            v = x.var(dims, unbiased=False)
            y = (x - m) / torch.sqrt(v + n.EPS) * params[n.g.name] + params[n.b.name]
            if n.res is not None:
                y = y + vals[id(n.res)]
            vals[id(n.out)] = torch.relu(y) if n.relu else y
        elif kind == "_BiasAct":
            y = vals[id(n.x)] + params[n.b.name]
            vals[id(n.out)] = torch.relu(y) if n.relu else y
        elif kind == "_MaxPool":
            x = vals[id(n.x)].permute(0, 3, 1, 2)
            vals[id(n.out)] = F.max_pool2d(x, n.R, n.stride, n.pad).permute(0, 2, 3, 1)
        elif kind == "_AvgPool":
            x = vals[id(n.x)]
            vals[id(n.out)] = x.mean((1, 2))
        elif kind == "_Loss":
            loss = F.cross_entropy(vals[id(n.logits)], net.labels.long().cpu())
    loss.backward()
    return loss.detach().item(), {k: v.grad for k, v in params.items()}


@pytest.mark.gpu
@pytest.mark.parametrize("arch", ["lenet5", "resnet18_mini", "resnet50_mini"])
def test_full_step_native_mode_vs_torch(am, arch):
    """The whole training step's wiring -- forward, loss, backward through BN /
    ReLU / bias / pooling / residual adds, gradient accumulation, SGD -- against
    FP64 autograd, with the Conv2D / Dense passes in native-multiply mode."""
    import torch
    from paper_2209_04161_b200 import net as netmod
    lut = am.Lut.build("mbm", 7)
    if arch == "lenet5":
        net = netmod.lenet5(lut, batch=8, seed=3)
    elif arch == "resnet18_mini":
        net = netmod.resnet18_cifar(lut, batch=4, seed=4, widths=(8, 16, 16, 32), hw=16)
    else:
        net = netmod.resnet50(lut, batch=2, seed=5, widths=(8, 8, 16, 16), blocks=(1, 2, 1, 1), hw=64, classes=20)
    with am.multiply_mode(am.AMSIM_MUL_NATIVE):
        net.forward(True)
        net.backward()
        torch.cuda.synchronize()
        loss_ref, grads = _reference_grads(net)
        assert abs(net.loss_value.item() - loss_ref) <= 1e-4 * max(1.0, abs(loss_ref))
        for p in net.params:
            _close(p.grad.cpu(), grads[p.name], 2e-3, p.name)
        w0 = net.flat_w.clone()
        g0 = net.flat_g.clone()
        net.update()
        torch.cuda.synchronize()
        want = w0 - net.lr * (g0 + net.weight_decay * w0)
        _close(net.flat_w.cpu(), want.cpu(), 1e-6, "sgd")


@pytest.mark.gpu
@pytest.mark.parametrize("arch", ["lenet5", "resnet18_mini"])
def test_full_step_amsim_graph_replay(am, arch):
    """AMSim mode: a captured CUDA graph of the training step reproduces the
    eager step bit for bit (same parameters after k steps), the loss is finite
    and decreases on a fixed batch."""
    import torch
    from paper_2209_04161_b200 import net as netmod
    lut = am.Lut.build("mbm", 7)

    def make():
        if arch == "lenet5":
            return netmod.lenet5(lut, batch=16, seed=7)
        return netmod.resnet18_cifar(lut, batch=8, seed=8, widths=(8, 16, 16, 32), hw=16)
    a, b = make(), make()
    losses = []
    for _ in range(3):
        a.train_step()
        losses.append(a.loss_value.item())
    b.train_step()                        # step 1, eager (tables, plans)
    replay = b.capture(b.train_step)      # step 2 runs eagerly on a side stream, then the capture
    replay()                              # step 3
    torch.cuda.synchronize()
    assert torch.equal(a.flat_w, b.flat_w)
    assert all(math.isfinite(v) for v in losses)
    assert losses[-1] < losses[0]


@pytest.mark.gpu
def test_inference_step_uses_running_stats(am):
    import torch
    from paper_2209_04161_b200 import net as netmod
    lut = am.Lut.build("exact", 7)
    net = netmod.resnet18_cifar(lut, batch=4, seed=9, widths=(8, 8, 16, 16), hw=8)
    net.train_step()
    net.infer_step()
    a = net.logits.data.clone()
    net.infer_step()
    torch.cuda.synchronize()
    assert torch.equal(a, net.logits.data) and torch.isfinite(a).all()
