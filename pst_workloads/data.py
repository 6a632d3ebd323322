"""Seeded synthetic MNIST-/CIFAR-10-shaped mini-batches (recipe in DESIGN.md §Inputs).

The paper trains on MNIST and CIFAR-10; there is no network
access, so batches are synthetic with the datasets' shapes, value range and
normalisation, and are learnable (class-dependent templates) so the loss
falls.  Mini-batch i depends only on (seed, i): any mini-batch can be
regenerated independently, which is what lets the oracle and the GPU see
identical inputs.

    CIFAR-like (C=3, 32x32): T_y = 4x4x3 Gaussian pattern of class y,
        nearest-upsampled to 32x32; x = clip(0.5 + 0.25 T_y + 0.2 N(0,1), 0, 1),
        quantised to 1/255, normalised per channel with
        mean (0.485, 0.456, 0.406), std (0.229, 0.224, 0.225).
    MNIST-like (C=1, 28x28): T_y = 7x7 Bernoulli(0.19) stroke mask of class y,
        upsampled 4x; x = clip(T_y * U(0.7, 1) + 0.1 N(0,1), 0, 1), quantised to
        1/255, normalised (x - 0.1307) / 0.3081.
    Other shapes (tests): x = N(0,1) + 0.5 T_y with T_y a per-class Gaussian image.
Labels are uniform over n_classes.  Everything is returned as float32 NCHW
and int32 labels -- the ABI's input types.
"""
from __future__ import annotations

import numpy as np

_CIFAR_MEAN = np.array([0.485, 0.456, 0.406], dtype=np.float64)
_CIFAR_STD = np.array([0.229, 0.224, 0.225], dtype=np.float64)


def _templates(seed, shape, n_classes):
    c, h, w = shape
    rng = np.random.default_rng([seed, 0x7E3])
    if (c, h, w) == (3, 32, 32):
        t = rng.standard_normal((n_classes, 3, 4, 4))
        return np.kron(t, np.ones((1, 1, 8, 8)))
    if (c, h, w) == (1, 28, 28):
        t = (rng.random((n_classes, 1, 7, 7)) < 0.19).astype(np.float64)
        return np.kron(t, np.ones((1, 1, 4, 4)))
    return rng.standard_normal((n_classes, c, h, w))


def make_batch(shape, batch, i, seed=1234, n_classes=10):
    """Mini-batch i: (x float32 [batch, C, H, W], y int32 [batch])."""
    c, h, w = shape
    T = _templates(seed, shape, n_classes)
    rng = np.random.default_rng([seed, int(i) + 1])
    y = rng.integers(0, n_classes, size=batch)
    if (c, h, w) == (3, 32, 32):
        x = 0.5 + 0.25 * T[y] + 0.2 * rng.standard_normal((batch, c, h, w))
        x = np.round(np.clip(x, 0.0, 1.0) * 255.0) / 255.0
        x = (x - _CIFAR_MEAN[None, :, None, None]) / _CIFAR_STD[None, :, None, None]
    elif (c, h, w) == (1, 28, 28):
        amp = rng.uniform(0.7, 1.0, size=(batch, 1, 1, 1))
        x = T[y] * amp + 0.1 * rng.standard_normal((batch, c, h, w))
        x = np.round(np.clip(x, 0.0, 1.0) * 255.0) / 255.0
        x = (x - 0.1307) / 0.3081
    else:
        x = rng.standard_normal((batch, c, h, w)) + 0.5 * T[y]
    return x.astype(np.float32), y.astype(np.int32)


def batches(shape, batch, n, seed=1234, n_classes=10, start=0):
    return [make_batch(shape, batch, start + i, seed, n_classes) for i in range(n)]
