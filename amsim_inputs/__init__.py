"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no truncation, no LUT, no
approximate product): it only draws seeded FP32 tensors with the shapes and
value distributions of the paper's workloads (SURVEY.md 8(d) "Synthetic
inputs"; recipe restated in DESIGN.md) and the operand grids the per-product
tests sweep.  Both sides consume it; neither side's arithmetic lives here.
"""
from __future__ import annotations

import numpy as np

from .workloads import (ConvLayer, DenseLayer, lenet5_layers, resnet18_cifar_layers,  # noqa: F401
                        resnet50_layers, step_macs)


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def normal(shape, seed: int, std: float = 1.0) -> np.ndarray:
    return (rng(seed).standard_normal(shape, dtype=np.float32) * np.float32(std)).astype(np.float32)


def relu_normal(shape, seed: int) -> np.ndarray:
    """Layer inputs ReLU(N(0,1)): ~50% exact zeros (ResNet-shaped configs)."""
    return np.maximum(normal(shape, seed), np.float32(0.0))


def mnist_like(shape, seed: int, zero_frac: float = 0.8) -> np.ndarray:
    """Values in [0,1) with ~80% exact zeros (MNIST-like sparsity, config 2)."""
    g = rng(seed)
    v = g.random(shape, dtype=np.float32)
    v[g.random(shape) < zero_frac] = 0.0
    return v


def he_uniform(shape, fan_in: int, seed: int) -> np.ndarray:
    lim = np.sqrt(6.0 / fan_in)
    return rng(seed).uniform(-lim, lim, shape).astype(np.float32)


def he_normal(shape, fan_in: int, seed: int) -> np.ndarray:
    return normal(shape, seed, float(np.sqrt(2.0 / fan_in)))


def bits_to_f32(u) -> np.ndarray:
    return np.asarray(u, dtype=np.uint32).view(np.float32)


def operand_grid(m: int, exponents=(1, 2, 63, 64, 65, 126, 127, 128, 190, 253, 254),
                 signs=(0, 1), specials: bool = True) -> np.ndarray:
    """Every m-bit mantissa x the exponent grid x signs,
    plus zero / subnormal / Inf / NaN encodings.  Low mantissa bits below the top
    m are filled with a fixed pattern so truncation is exercised."""
    vals = []
    low_fill = (0x5A5A5A & ((1 << (23 - m)) - 1)) if m < 23 else 0
    for s in signs:
        for e in exponents:
            for k in range(1 << m):
                vals.append((s << 31) | (e << 23) | (k << (23 - m)) | low_fill)
    if specials:
        for s in signs:
            vals += [(s << 31), (s << 31) | 0x1234, (s << 31) | 0x7F800000,
                     (s << 31) | 0x7FC00000, (s << 31) | 0x7F801234 | (0x55 << (23 - min(m, 8)))]
    return bits_to_f32(np.array(vals, dtype=np.uint64).astype(np.uint32))
