"""Layer shape tables of the paper's workloads (shapes only, no arithmetic).

Architectures follow SURVEY.md 8(c) reading C18 (PAPER.md:720-722 leaves them
under-specified): LeNet-5 on 28x28x1 with conv1 pad 2 (C20); ResNet-18 for
CIFAR-10 with a 3x3 stem and no max-pool; ResNet-50 = torchvision v1.5 (stride
on the 3x3 conv of each bottleneck).  Only Conv2D and Dense multiply
(PAPER.md:480), so only those layers are listed.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ConvLayer:
    name: str
    N: int
    H: int
    W: int
    C: int
    K: int
    R: int
    S: int
    stride: int = 1
    pad: int = 0
    first: bool = False  # no dgrad needed for the network's first layer

    @property
    def OH(self):
        return (self.H + 2 * self.pad - self.R) // self.stride + 1

    @property
    def OW(self):
        return (self.W + 2 * self.pad - self.S) // self.stride + 1

    def macs(self) -> int:
        """Dense-convention MACs of one pass: N*OH*OW*K*R*S*C."""
        return self.N * self.OH * self.OW * self.K * self.R * self.S * self.C

    def with_batch(self, n: int) -> "ConvLayer":
        return ConvLayer(self.name, n, self.H, self.W, self.C, self.K, self.R, self.S, self.stride, self.pad,
                         self.first)


@dataclass(frozen=True)
class DenseLayer:
    name: str
    N: int      # batch
    IN: int
    OUT: int
    first: bool = False

    def macs(self) -> int:
        return self.N * self.IN * self.OUT

    def with_batch(self, n: int) -> "DenseLayer":
        return DenseLayer(self.name, n, self.IN, self.OUT, self.first)


def lenet5_layers(batch: int = 64):
    return [
        ConvLayer("c1", batch, 28, 28, 1, 6, 5, 5, 1, 2, first=True),
        ConvLayer("c2", batch, 14, 14, 6, 16, 5, 5, 1, 0),
        DenseLayer("f3", batch, 400, 120),
        DenseLayer("f4", batch, 120, 84),
        DenseLayer("f5", batch, 84, 10),
    ]


def resnet18_cifar_layers(batch: int = 128):
    L = [ConvLayer("stem", batch, 32, 32, 3, 64, 3, 3, 1, 1, first=True)]
    H, C = 32, 64
    for stage, (K, stride) in enumerate([(64, 1), (128, 2), (256, 2), (512, 2)]):
        for blk in range(2):
            s = stride if blk == 0 else 1
            OH = (H + 2 - 3) // s + 1
            L.append(ConvLayer(f"l{stage+1}.{blk}.conv1", batch, H, H, C, K, 3, 3, s, 1))
            L.append(ConvLayer(f"l{stage+1}.{blk}.conv2", batch, OH, OH, K, K, 3, 3, 1, 1))
            if blk == 0 and (s != 1 or C != K):
                L.append(ConvLayer(f"l{stage+1}.{blk}.down", batch, H, H, C, K, 1, 1, s, 0))
            H, C = OH, K
    L.append(DenseLayer("fc", batch, 512, 10))
    return L


def resnet50_layers(batch: int = 256):
    L = [ConvLayer("stem", batch, 224, 224, 3, 64, 7, 7, 2, 3, first=True)]
    H, C = 56, 64  # after the 3x3/2 max-pool
    for stage, (width, blocks, stride) in enumerate([(64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)]):
        out = width * 4
        for blk in range(blocks):
            s = stride if blk == 0 else 1
            OH = (H + 2 - 3) // s + 1
            p = f"l{stage+1}.{blk}"
            L.append(ConvLayer(p + ".conv1", batch, H, H, C, width, 1, 1, 1, 0))
            L.append(ConvLayer(p + ".conv2", batch, H, H, width, width, 3, 3, s, 1))
            L.append(ConvLayer(p + ".conv3", batch, OH, OH, width, out, 1, 1, 1, 0))
            if blk == 0:
                L.append(ConvLayer(p + ".down", batch, H, H, C, out, 1, 1, s, 0))
            H, C = OH, out
    L.append(DenseLayer("fc", batch, 2048, 1000))
    return L


def step_macs(layers) -> int:
    """fwd + wgrad for every layer + dgrad for all but the first."""
    tot = 0
    for l in layers:
        tot += l.macs() * (2 if l.first else 3)
    return tot
