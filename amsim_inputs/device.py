"""Seeded synthetic tensors generated directly in device memory (torch CUDA
Philox generator) for the full-size benchmark workloads, with the same
distributions as the numpy generators in ``amsim_inputs``:
layer inputs ReLU(N(0,1)), He-normal weights, errors N(0, 2^-10).  No method
arithmetic here.
"""
from __future__ import annotations

import math


def _gen(seed: int, device):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def normal(shape, seed: int, std: float = 1.0, device="cuda"):
    import torch
    t = torch.randn(shape, generator=_gen(seed, device), device=device, dtype=torch.float32)
    return t.mul_(std) if std != 1.0 else t


def relu_normal(shape, seed: int, device="cuda"):
    return normal(shape, seed, 1.0, device).clamp_(min=0.0)


def he_normal(shape, fan_in: int, seed: int, device="cuda"):
    return normal(shape, seed, math.sqrt(2.0 / fan_in), device)


def mnist_like(shape, seed: int, zero_frac: float = 0.8, device="cuda"):
    import torch
    g = _gen(seed, device)
    v = torch.rand(shape, generator=g, device=device)
    keep = torch.rand(shape, generator=g, device=device) >= zero_frac
    return v.mul_(keep)
