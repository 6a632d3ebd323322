"""Seeded synthetic workloads shared by the oracle side and the CUDA side.

This package holds ONLY inputs: network architecture descriptions (which
layers, which shapes), seeded parameter initialisation and seeded synthetic
mini-batches.  It contains none of the method's arithmetic (no forward, no
backward, no update, no schedule) -- see DESIGN.md "Oracle independence".
Both `oracle/` (through the tests) and `paper_1912_12675_b200` (through the
binding) consume what it produces; neither imports the other.
"""
from .nets import (LayerSpec, NetSpec, lenet5, alexnet_cifar, vgg16_cifar,
                   resnet_cifar, tiny_resnet, tiny_cnn, by_name, param_count,
                   layer_param_shapes, weighted_layer_count)
from .init import init_params
from .data import make_batch, batches
from .configs import CONFIGS, Config

__all__ = [
    "LayerSpec", "NetSpec", "lenet5", "alexnet_cifar", "vgg16_cifar",
    "resnet_cifar", "tiny_resnet", "tiny_cnn", "by_name", "param_count",
    "layer_param_shapes", "weighted_layer_count", "init_params", "make_batch",
    "batches", "CONFIGS", "Config",
]
