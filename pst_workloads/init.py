"""Seeded parameter initialisation (reading AMB-17 in DESIGN.md).

Kaiming-normal (fan_in, ReLU gain) for conv and FC weights, the PyTorch
default uniform(-1/sqrt(fan_in), 1/sqrt(fan_in)) for biases, gamma = 1,
beta = 0.  Values are produced as float32 -- the ABI's parameter type -- and
the same array is handed to the oracle (which promotes it to float64) and to
`pst_create`.
"""
from __future__ import annotations

import numpy as np

from .nets import NetSpec, layer_param_shapes


def init_params(net: NetSpec, seed: int = 42) -> np.ndarray:
    rng = np.random.default_rng(seed)
    chunks = []
    for L in net.layers:
        fan_in = L.cin * L.k * L.k if L.kind == "conv" else L.cin
        for name, shp in layer_param_shapes(L):
            if name == "W":
                v = rng.standard_normal(shp) * np.sqrt(2.0 / fan_in)
            elif name == "b":
                bound = 1.0 / np.sqrt(fan_in)
                v = rng.uniform(-bound, bound, size=shp)
            elif name == "gamma":
                v = np.ones(shp)
            else:  # beta
                v = np.zeros(shp)
            chunks.append(np.asarray(v, dtype=np.float32).ravel())
    return np.concatenate(chunks).astype(np.float32)
