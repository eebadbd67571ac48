"""One approximate training step of a layer list, through the C ABI.

"Train step": every approximate Conv2D / Dense pass at its
real shape in dependency order -- forward for all layers, then in reverse
order the weight gradient (Alg. 4 l.4-5) and, except for the first layer, the
preceding-layer gradient (Alg. 4 l.6-8) -- plus, on several GPUs, the NCCL
all-reduce of the weight gradients, bucketed and overlapped with backward.
The non-multiplying layers (BN, ReLU, pooling, residual add, loss, SGD) are
not approximated by the paper and are NOT part of this step:
each layer reads its own seeded synthetic input / error tensors resident in
HBM, and its outputs go to scratch buffers.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import _lib as L
from .dp import GradAllReducer, plan_buckets


@dataclass
class _Layer:
    spec: object
    kind: str          # "conv" | "dense"
    x: object
    w: object
    dy: object
    dw: object         # view into the flat gradient buffer
    desc: object = None


class TrainStep:
    def __init__(self, layers, lut, device="cuda", seed: int = 0, bucket_mb: float = 25.0, group=None,
                 first_input: str = "relu"):
        import torch

        from amsim_inputs import device as gen
        from amsim_inputs import workloads as wl

        self.lut = lut
        self.device = torch.device(device)
        self.specs = list(layers)
        self.layers = []
        numels = []
        for l in self.specs:
            numels.append(l.R * l.S * l.C * l.K if isinstance(l, wl.ConvLayer) else l.IN * l.OUT)
        offsets, buckets, total = plan_buckets(numels, int(bucket_mb * 2 ** 20 / 4))
        self.flat_grad = torch.zeros(total, device=self.device)
        ymax = dxmax = wsmax = 1
        for i, l in enumerate(self.specs):
            s = seed + 16 * i
            dwv = self.flat_grad.narrow(0, offsets[i], numels[i])
            if isinstance(l, wl.ConvLayer):
                xin = (gen.mnist_like if (l.first and first_input == "mnist") else gen.relu_normal)(
                    (l.N, l.H, l.W, l.C), s, device=self.device)
                w = gen.he_normal((l.R, l.S, l.C, l.K), l.R * l.S * l.C, s + 1, device=self.device)
                dy = gen.normal((l.N, l.OH, l.OW, l.K), s + 2, 2 ** -10, device=self.device)
                d = L.conv_desc(l.N, l.H, l.W, l.C, l.K, l.R, l.S, l.stride, l.pad)
                self.layers.append(_Layer(l, "conv", xin, w, dy, dwv.view(l.R, l.S, l.C, l.K), d))
                ymax = max(ymax, l.N * l.OH * l.OW * l.K)
                dxmax = max(dxmax, l.N * l.H * l.W * l.C)
                wsmax = max(wsmax, L.amsim_conv2d_bwd_filter_workspace(lut, d) // 4)
            else:
                xin = gen.relu_normal((l.N, l.IN), s, device=self.device)
                w = gen.he_normal((l.IN, l.OUT), l.IN, s + 1, device=self.device)
                dy = gen.normal((l.N, l.OUT), s + 2, 2 ** -10, device=self.device)
                self.layers.append(_Layer(l, "dense", xin, w, dy, dwv.view(l.IN, l.OUT)))
                ymax = max(ymax, l.N * l.OUT)
                dxmax = max(dxmax, l.N * l.IN)
        self.y_scratch = torch.empty(ymax, device=self.device)
        self.dx_scratch = torch.empty(dxmax, device=self.device)
        self.workspace = torch.empty(wsmax, device=self.device)
        self.comm_stream = torch.cuda.Stream(device=self.device) if self.device.type == "cuda" else None
        self.reducer = GradAllReducer(self.flat_grad, buckets, group=group, comm_stream=self.comm_stream)
        self.timers = None

    def set_lut(self, lut):
        """Run the same step with another table (e.g. the fully pinned exact
        bf16 table next to MBM); grows the wgrad workspace if its plans need more."""
        import torch
        self.lut = lut
        need = max(L.amsim_conv2d_bwd_filter_workspace(lut, ly.desc) // 4 for ly in self.layers if ly.kind == "conv")
        if need > self.workspace.numel():
            self.workspace = torch.empty(need, device=self.device)

    def activation_zero_fraction(self) -> float:
        """Fraction of exact zeros in the layer inputs (the warp-shared A operand
        of conv fwd / wgrad): zero-row skipping saves their lookups, so the fwd /
        wgrad rates depend on it (ReLU(N(0,1)) inputs: about 1/2)."""
        zeros = total = 0
        for ly in self.layers:
            zeros += int((ly.x == 0).sum().item())
            total += ly.x.numel()
        return zeros / max(total, 1)

    # ------------------------------------------------------------------
    def step_macs(self) -> int:
        return sum(l.spec.macs() * (2 if l.spec.first else 3) for l in self.layers)

    def input_tensor(self):
        """The step's network input (the first layer's activation)."""
        return self.layers[0].x

    def _timed(self, kind, macs, fn):
        if self.timers is None:
            fn()
            return
        import torch
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        self.timers.append((kind, macs, e0, e1))

    def forward(self):
        for ly in self.layers:
            l = ly.spec
            if ly.kind == "conv":
                y = self.y_scratch[: l.N * l.OH * l.OW * l.K]
                self._timed("conv_fwd", l.macs(), lambda: L.amsim_conv2d_fwd(self.lut, ly.desc, ly.x, ly.w, y))
            else:
                y = self.y_scratch[: l.N * l.OUT].view(l.N, l.OUT)
                self._timed("dense", l.macs(), lambda: L.amsim_gemm(self.lut, ly.x, ly.w, y))

    def backward(self):
        self.reducer.reset()
        for i in range(len(self.layers) - 1, -1, -1):
            ly = self.layers[i]
            l = ly.spec
            if ly.kind == "conv":
                self._timed("conv_wgrad", l.macs(),
                            lambda: L.amsim_conv2d_bwd_filter(self.lut, ly.desc, ly.x, ly.dy, ly.dw, self.workspace))
                self.reducer.ready(i)
                if not l.first:
                    dx = self.dx_scratch[: l.N * l.H * l.W * l.C]
                    self._timed("conv_dgrad", l.macs(),
                                lambda: L.amsim_conv2d_bwd_data(self.lut, ly.desc, ly.dy, ly.w, dx))
            else:
                self._timed("dense", l.macs(), lambda: L.amsim_gemm(self.lut, ly.x, ly.dy, ly.dw, trans_a=True))
                self.reducer.ready(i)
                if not l.first:
                    dx = self.dx_scratch[: l.N * l.IN].view(l.N, l.IN)
                    self._timed("dense", l.macs(), lambda: L.amsim_gemm(self.lut, ly.dy, ly.w, dx, trans_b=True))
        self.reducer.finish()

    def step(self):
        self.forward()
        self.backward()

    def capture(self):
        """Capture one step into a CUDA graph (single process: the NCCL
        all-reduce path stays eager) and return its replay function.  Call
        after at least one eager step (table upload and plans happen there)."""
        import torch
        if self.reducer.world != 1:
            raise RuntimeError("graph capture is single-GPU only")
        self.timers = None
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.step()                       # warm the side stream
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            self.step()
        self._graph = g
        return g.replay
