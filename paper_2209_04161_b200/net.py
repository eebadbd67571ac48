"""Full ApproxTrain networks on B200: a whole training step (forward, softmax
cross-entropy, backward, SGD-momentum) and an inference step, with every
Conv2D / Dense multiplication through AMSim (include/amsim.h) and the
non-multiplying layers -- batch normalisation, ReLU, bias, pooling, the
residual add, the loss and the optimiser -- through the native FP32 kernels of
include/amsim_nn.h (PAPER.md:480 approximates only the multiplications;
PAPER.md:888-942 time whole training and inference steps).
NEXT(1).

Architectures follow reading C18: LeNet-5 (28x28x1, conv1 pad 2,
ReLU, 2x2 max-pool, dense 400-120-84-10), ResNet-18 for CIFAR (3x3 stem, no
max-pool, basic blocks) and ResNet-50 v1.5 (7x7/2 stem, 3x3/2 max-pool,
bottlenecks with the stride on the 3x3 conv).  Their approximate layers are
exactly amsim_inputs.workloads' layer lists, so the approximate MACs of a step
equal the bench's.  Activations NHWC, weights HWIO, dense weights [in][out].

Python here only sequences library calls (argument marshalling); the step can
be captured into one CUDA graph (single GPU).  With several processes the
weight gradients (conv, dense, BN and bias parameters, one flat buffer) are
all-reduced in buckets as they become ready (dp.GradAllReducer); the loss
gradient is divided by the global batch, so their sum is the global-batch mean
gradient (uneven shards included).  Batch-norm statistics are per rank, as in
data-parallel training without synchronised batch norm.
"""
from __future__ import annotations

import math

from . import _lib as L
from .dp import GradAllReducer, plan_buckets


class T:
    """An activation tensor (device storage allocated by the Net) and its gradient."""

    def __init__(self, name, shape, needs_grad=True):
        self.name, self.shape, self.needs_grad = name, tuple(shape), needs_grad
        self.data = self.grad = None
        self.written = False

    @property
    def numel(self):
        return math.prod(self.shape)


class Param:
    def __init__(self, name, shape, init):
        self.name, self.shape, self.init = name, tuple(shape), init
        self.data = self.grad = None

    @property
    def numel(self):
        return math.prod(self.shape)


class Net:
    """Graph of layer nodes; see the module docstring."""

    def __init__(self, lut, device="cuda", seed=0, group=None, bucket_mb=25.0):
        self.lut, self.device_str, self.seed, self.group, self.bucket_mb = lut, device, seed, group, bucket_mb
        self.nodes, self.tensors, self.params = [], [], []
        self.approx_macs = 0

    # ---- graph construction ------------------------------------------------
    def tensor(self, name, shape, needs_grad=True):
        t = T(name, shape, needs_grad)
        self.tensors.append(t)
        return t

    def param(self, name, shape, init):
        p = Param(name, shape, init)
        self.params.append(p)
        return p

    def conv(self, x, K, R, S, stride, pad, name, first=False):
        N, H, W, C = x.shape
        d = L.conv_desc(N, H, W, C, K, R, S, stride, pad)
        w = self.param(name + ".w", (R, S, C, K), ("he", R * S * C))
        out = self.tensor(name + ".out", (N, d.OH, d.OW, K))
        self.nodes.append(_Conv(self, x, w, d, out, first))
        self.approx_macs += N * d.OH * d.OW * K * R * S * C * (2 if first else 3)
        return out

    def dense(self, x, OUT, name, first=False):
        N = x.shape[0]
        IN = math.prod(x.shape[1:])
        w = self.param(name + ".w", (IN, OUT), ("he", IN))
        out = self.tensor(name + ".out", (N, OUT))
        self.nodes.append(_Dense(self, x, w, out, first))
        self.approx_macs += N * IN * OUT * (2 if first else 3)
        return out

    def bn(self, x, name, relu=True, res=None):
        C = x.shape[-1]
        g = self.param(name + ".gamma", (C,), ("const", 1.0))
        b = self.param(name + ".beta", (C,), ("const", 0.0))
        out = self.tensor(name + ".out", x.shape)
        self.nodes.append(_BN(self, x, g, b, out, relu, res))
        return out

    def bias_act(self, x, name, relu=True):
        C = x.shape[-1]
        b = self.param(name + ".bias", (C,), ("const", 0.0))
        out = self.tensor(name + ".out", x.shape)
        self.nodes.append(_BiasAct(self, x, b, out, relu))
        return out

    def maxpool(self, x, R, stride, pad, name):
        N, H, W, C = x.shape
        OH, OW = (H + 2 * pad - R) // stride + 1, (W + 2 * pad - R) // stride + 1
        out = self.tensor(name + ".out", (N, OH, OW, C))
        self.nodes.append(_MaxPool(self, x, out, R, stride, pad))
        return out

    def avgpool(self, x, name):
        N, H, W, C = x.shape
        out = self.tensor(name + ".out", (N, C))
        self.nodes.append(_AvgPool(self, x, out))
        return out

    def loss(self, logits):
        self.logits = logits
        self.nodes.append(_Loss(self, logits))

    # ---- allocation ----------------------------------------------------------
    def finalize(self, input_kind="normal"):
        import torch

        from amsim_inputs import device as gen
        dev = torch.device(self.device_str)
        self.device = dev
        for t in self.tensors:
            t.data = torch.empty(t.shape, device=dev)
            if t.needs_grad:
                t.grad = torch.empty(t.shape, device=dev)
        # flat parameter / gradient / momentum buffers; plan_buckets lays the
        # parameters out in the order the backward pass completes their
        # gradients (reverse creation order), so all-reduce buckets are contiguous
        offsets, buckets, total = plan_buckets([p.numel for p in self.params], int(self.bucket_mb * 2 ** 20 / 4))
        self.flat_w = torch.empty(total, device=dev)
        self.flat_g = torch.zeros(total, device=dev)
        self.flat_v = torch.zeros(total, device=dev)
        for j, p in enumerate(self.params):
            p.data = self.flat_w.narrow(0, offsets[j], p.numel).view(p.shape)
            p.grad = self.flat_g.narrow(0, offsets[j], p.numel).view(p.shape)
            kind, arg = p.init
            if kind == "he":
                p.data.copy_(gen.normal(p.shape, self.seed + 7 * j + 1, math.sqrt(2.0 / arg), device=dev))
            else:
                p.data.fill_(arg)
        self.param_index = {id(p): j for j, p in enumerate(self.params)}
        self.reducer = GradAllReducer(self.flat_g, buckets, group=self.group,
                                      comm_stream=torch.cuda.Stream(device=dev) if dev.type == "cuda" else None)
        # the loss gradient is divided by the GLOBAL batch (sum of the ranks'
        # shards), so the all-reduce SUM is the gradient of the global-batch
        # mean loss -- also with uneven shards -- and the update uses lr as is
        self.global_batch = self.tensors[0].shape[0]
        if self.reducer.world > 1:
            import torch.distributed as dist
            nb = torch.tensor([self.global_batch], dtype=torch.int64,
                              device=dev if dist.get_backend(self.group) == "nccl" else "cpu")
            dist.all_reduce(nb, group=self.group)
            self.global_batch = int(nb.item())
        # scratch: two gradient temporaries, the per-channel reduction workspace, wgrad split-K workspace
        maxn = max(t.numel for t in self.tensors)
        self.scratch = [torch.empty(maxn, device=dev), torch.empty(maxn, device=dev)]
        nn_ws = 1
        wg_ws = 1
        for n in self.nodes:
            nn_ws = max(nn_ws, n.nn_ws_bytes())
            wg_ws = max(wg_ws, n.wg_ws_bytes())
        self.nn_ws = torch.empty((nn_ws + 15) // 4, device=dev)
        self.wg_ws = torch.empty((wg_ws + 15) // 4, device=dev)
        for n in self.nodes:
            n.alloc(dev)
        # synthetic input batch and labels (seeded)
        x0 = self.tensors[0]
        if input_kind == "mnist":
            x0.data.copy_(gen.mnist_like(x0.shape, self.seed + 101, device=dev))
        else:
            x0.data.copy_(gen.normal(x0.shape, self.seed + 101, device=dev))
        g = torch.Generator(device=dev)
        g.manual_seed(self.seed + 202)
        self.labels = torch.randint(0, self.logits.shape[1], (self.logits.shape[0],), generator=g, device=dev,
                                    dtype=torch.int32)
        self.loss_value = torch.zeros(1, device=dev)
        self.lr, self.momentum, self.weight_decay = 0.01, 0.9, 5e-5
        return self

    @property
    def input(self):
        return self.tensors[0]

    # ---- gradient plumbing ---------------------------------------------------
    def grad_target(self, t, k=0):
        """Where to write the next gradient contribution of t: its gradient
        buffer if nothing has been written this step, else scratch k."""
        if not t.written:
            return t.grad
        return self.scratch[k][: t.numel].view(t.shape)

    def grad_done(self, t, target):
        if target is t.grad:
            t.written = True
        else:
            L.amsim_add(t.grad, target, t.grad, t.numel)

    # ---- steps ---------------------------------------------------------------
    def forward(self, train=True):
        for n in self.nodes:
            n.fwd(train)

    def backward(self):
        for t in self.tensors:
            t.written = False
        self.reducer.reset()
        for n in reversed(self.nodes):
            n.bwd()
            for p in n.params():
                self.reducer.ready(self.param_index[id(p)])
        self.reducer.finish()

    def update(self):
        # flat_g holds the global-batch mean gradient (see finalize), so weight
        # decay and lr apply unscaled whatever the world size
        L.amsim_sgd_momentum(self.flat_w, self.flat_g, self.flat_v, self.flat_w.numel(), self.lr,
                             self.momentum, self.weight_decay)

    def train_step(self):
        self.forward(True)
        self.backward()
        self.update()

    def infer_step(self):
        self.forward(False)

    def capture(self, fn):
        """CUDA graph of `fn` (single process); returns its replay."""
        import torch
        if self.reducer.world != 1:
            raise RuntimeError("graph capture is single-GPU only")
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            fn()
        if not hasattr(self, "_graphs"):
            self._graphs = []
        self._graphs.append(g)
        return g.replay


# ---------------------------------------------------------------------------
# nodes

class _Node:
    def __init__(self, net):
        self.net = net

    def params(self):
        return []

    def nn_ws_bytes(self):
        return 0

    def wg_ws_bytes(self):
        return 0

    def alloc(self, dev):
        pass


class _Conv(_Node):
    def __init__(self, net, x, w, d, out, first):
        super().__init__(net)
        self.x, self.w, self.d, self.out, self.first = x, w, d, out, first

    def params(self):
        return [self.w]

    def wg_ws_bytes(self):
        return L.amsim_conv2d_bwd_filter_workspace(self.net.lut, self.d)

    def fwd(self, train):
        L.amsim_conv2d_fwd(self.net.lut, self.d, self.x.data, self.w.data, self.out.data)

    def bwd(self):
        net = self.net
        L.amsim_conv2d_bwd_filter(net.lut, self.d, self.x.data, self.out.grad, self.w.grad, net.wg_ws)
        if self.x.needs_grad and not self.first:
            tgt = net.grad_target(self.x)
            L.amsim_conv2d_bwd_data(net.lut, self.d, self.out.grad, self.w.data, tgt)
            net.grad_done(self.x, tgt)


class _Dense(_Node):
    def __init__(self, net, x, w, out, first):
        super().__init__(net)
        self.x, self.w, self.out, self.first = x, w, out, first
        self.IN = w.shape[0]

    def params(self):
        return [self.w]

    def fwd(self, train):
        x2 = self.x.data.view(self.x.shape[0], self.IN)
        L.amsim_gemm(self.net.lut, x2, self.w.data, self.out.data)

    def bwd(self):
        net = self.net
        x2 = self.x.data.view(self.x.shape[0], self.IN)
        L.amsim_gemm(net.lut, x2, self.out.grad, self.w.grad, trans_a=True)          # a = x, b = dy
        if self.x.needs_grad and not self.first:
            tgt = net.grad_target(self.x)
            L.amsim_gemm(net.lut, self.out.grad, self.w.data, tgt.view(self.x.shape[0], self.IN), trans_b=True)
            net.grad_done(self.x, tgt)


class _BN(_Node):
    EPS, MOMENTUM = 1e-5, 0.1

    def __init__(self, net, x, g, b, out, relu, res):
        super().__init__(net)
        self.x, self.g, self.b, self.out, self.relu, self.res = x, g, b, out, relu, res
        self.C = x.shape[-1]
        self.P = x.numel // self.C

    def params(self):
        return [self.g, self.b]

    def nn_ws_bytes(self):
        return L.amsim_nn_workspace_bytes(self.P, self.C)

    def alloc(self, dev):
        import torch
        self.mean = torch.zeros(self.C, device=dev)
        self.invstd = torch.zeros(self.C, device=dev)
        self.rmean = torch.zeros(self.C, device=dev)
        self.rvar = torch.ones(self.C, device=dev)

    def fwd(self, train):
        res = self.res.data if self.res is not None else None
        if train:
            L.amsim_bn_fwd_train(self.x.data, self.P, self.C, self.g.data, self.b.data, self.EPS, res, self.relu,
                                 self.out.data, self.mean, self.invstd, self.rmean, self.rvar, self.MOMENTUM,
                                 self.net.nn_ws)
        else:
            L.amsim_bn_fwd_infer(self.x.data, self.P, self.C, self.g.data, self.b.data, self.rmean, self.rvar,
                                 self.EPS, res, self.relu, self.out.data)

    def bwd(self):
        net = self.net
        tx = net.grad_target(self.x, 0)
        tr = net.grad_target(self.res, 1) if self.res is not None else None
        L.amsim_bn_bwd(self.out.grad, self.out.data, self.x.data, self.P, self.C, self.g.data, self.mean,
                       self.invstd, self.relu, tx, tr, self.g.grad, self.b.grad, net.nn_ws)
        net.grad_done(self.x, tx)
        if tr is not None:
            net.grad_done(self.res, tr)


class _BiasAct(_Node):
    def __init__(self, net, x, b, out, relu):
        super().__init__(net)
        self.x, self.b, self.out, self.relu = x, b, out, relu
        self.C = x.shape[-1]
        self.P = x.numel // self.C

    def params(self):
        return [self.b]

    def nn_ws_bytes(self):
        return L.amsim_nn_workspace_bytes(self.P, self.C)

    def fwd(self, train):
        L.amsim_bias_act_fwd(self.x.data, self.P, self.C, self.b.data, self.relu, self.out.data)

    def bwd(self):
        net = self.net
        tx = net.grad_target(self.x)
        L.amsim_bias_act_bwd(self.out.grad, self.out.data, self.P, self.C, self.relu, tx, self.b.grad, net.nn_ws)
        net.grad_done(self.x, tx)


class _MaxPool(_Node):
    def __init__(self, net, x, out, R, stride, pad):
        super().__init__(net)
        self.x, self.out, self.R, self.stride, self.pad = x, out, R, stride, pad

    def alloc(self, dev):
        import torch
        self.argmax = torch.empty(self.out.shape, device=dev, dtype=torch.uint8)

    def fwd(self, train):
        N, H, W, C = self.x.shape
        L.amsim_maxpool_fwd(self.x.data, N, H, W, C, self.R, self.R, self.stride, self.pad, self.out.data,
                            self.argmax)

    def bwd(self):
        N, H, W, C = self.x.shape
        tx = self.net.grad_target(self.x)
        L.amsim_maxpool_bwd(self.out.grad, self.argmax, N, H, W, C, self.R, self.R, self.stride, self.pad, tx)
        self.net.grad_done(self.x, tx)


class _AvgPool(_Node):
    def __init__(self, net, x, out):
        super().__init__(net)
        self.x, self.out = x, out

    def fwd(self, train):
        N, H, W, C = self.x.shape
        L.amsim_avgpool_fwd(self.x.data, N, H * W, C, self.out.data)

    def bwd(self):
        N, H, W, C = self.x.shape
        tx = self.net.grad_target(self.x)
        L.amsim_avgpool_bwd(self.out.grad, N, H * W, C, tx)
        self.net.grad_done(self.x, tx)


class _Loss(_Node):
    def __init__(self, net, logits):
        super().__init__(net)
        self.logits = logits

    def nn_ws_bytes(self):
        return L.amsim_nn_workspace_bytes(self.logits.shape[0], 1)

    def fwd(self, train):
        if train:   # fused loss + gradient; the backward pass starts from logits.grad
            N, K = self.logits.shape
            L.amsim_softmax_xent(self.logits.data, self.net.labels, N, K, self.net.loss_value, self.logits.grad,
                                 self.net.nn_ws, grad_denominator=self.net.global_batch)

    def bwd(self):
        self.logits.written = True


# ---------------------------------------------------------------------------
# architectures (reading C18)

def lenet5(lut, batch=64, device="cuda", seed=0, group=None, build_only=False):
    net = Net(lut, device, seed, group)
    x = net.tensor("input", (batch, 28, 28, 1), needs_grad=False)
    h = net.bias_act(net.conv(x, 6, 5, 5, 1, 2, "c1", first=True), "c1.act")
    h = net.maxpool(h, 2, 2, 0, "p1")
    h = net.bias_act(net.conv(h, 16, 5, 5, 1, 0, "c2"), "c2.act")
    h = net.maxpool(h, 2, 2, 0, "p2")
    h = net.bias_act(net.dense(h, 120, "f3"), "f3.act")
    h = net.bias_act(net.dense(h, 84, "f4"), "f4.act")
    logits = net.bias_act(net.dense(h, 10, "f5"), "f5.bias", relu=False)
    net.loss(logits)
    return net if build_only else net.finalize("mnist")


def resnet18_cifar(lut, batch=128, device="cuda", seed=0, group=None, widths=(64, 128, 256, 512), hw=32,
                   classes=10, build_only=False):
    net = Net(lut, device, seed, group)
    x = net.tensor("input", (batch, hw, hw, 3), needs_grad=False)
    h = net.bn(net.conv(x, widths[0], 3, 3, 1, 1, "stem", first=True), "stem.bn")
    C = widths[0]
    for stage, (K, stride) in enumerate(zip(widths, (1, 2, 2, 2))):
        for blk in range(2):
            s = stride if blk == 0 else 1
            p = f"l{stage + 1}.{blk}"
            o = net.bn(net.conv(h, K, 3, 3, s, 1, p + ".conv1"), p + ".bn1")
            o2 = net.conv(o, K, 3, 3, 1, 1, p + ".conv2")
            if blk == 0 and (s != 1 or C != K):
                sc = net.bn(net.conv(h, K, 1, 1, s, 0, p + ".down"), p + ".down.bn", relu=False)
            else:
                sc = h
            h = net.bn(o2, p + ".bn2", relu=True, res=sc)
            C = K
    logits = net.bias_act(net.dense(net.avgpool(h, "pool"), classes, "fc"), "fc.bias", relu=False)
    net.loss(logits)
    return net if build_only else net.finalize()


def resnet50(lut, batch=256, device="cuda", seed=0, group=None, widths=(64, 128, 256, 512), blocks=(3, 4, 6, 3),
             hw=224, classes=1000, build_only=False):
    net = Net(lut, device, seed, group)
    x = net.tensor("input", (batch, hw, hw, 3), needs_grad=False)
    h = net.bn(net.conv(x, widths[0], 7, 7, 2, 3, "stem", first=True), "stem.bn")
    h = net.maxpool(h, 3, 2, 1, "stem.pool")
    C = widths[0]
    for stage, (width, nb, stride) in enumerate(zip(widths, blocks, (1, 2, 2, 2))):
        out = width * 4
        for blk in range(nb):
            s = stride if blk == 0 else 1
            p = f"l{stage + 1}.{blk}"
            o = net.bn(net.conv(h, width, 1, 1, 1, 0, p + ".conv1"), p + ".bn1")
            o = net.bn(net.conv(o, width, 3, 3, s, 1, p + ".conv2"), p + ".bn2")
            o3 = net.conv(o, out, 1, 1, 1, 0, p + ".conv3")
            if blk == 0:
                sc = net.bn(net.conv(h, out, 1, 1, s, 0, p + ".down"), p + ".down.bn", relu=False)
            else:
                sc = h
            h = net.bn(o3, p + ".bn3", relu=True, res=sc)
            C = out
    logits = net.bias_act(net.dense(net.avgpool(h, "pool"), classes, "fc"), "fc.bias", relu=False)
    net.loss(logits)
    return net if build_only else net.finalize()


BUILDERS = {"lenet5": lenet5, "resnet18": resnet18_cifar, "resnet50": resnet50}
