"""Network architecture descriptions (inputs only, no arithmetic).

A network is a sequence of *weighted* layers (conv or FC).  Every
non-weighted op (BatchNorm, residual add, ReLU, pooling) is attached to the
weighted layer it follows, which is how the paper numbers layers for its
Pipeline Placement Vector: "p_i represents the layer number after which a
pipeline register pair is inserted" (section 3; Table 1
counts LeNet-5 as 5 layers, AlexNet 8, VGG-16 16, ResNet-20 20).  Reading
AMB-13: non-weighted ops belong to the preceding weighted layer.

Per weighted layer, in order of application:
    y = conv_or_fc(x) (+ bias)
    y = BN_train(y)                       if bn
    y = y + shortcut(block_input)         if residual
    y = relu(y)                           if relu
    y = maxpool2x2(y) | mean_{h,w}(y)     if pool == 'max2' | 'gap'
`block_begin` marks a layer whose *input* is the residual block input used
by the next layer that has `residual` set.  The shortcut is the identity
when shapes match, else the CIFAR-ResNet "option A" shortcut (stride-2
subsample, zero-pad channels equally on both sides); Table 6 (PAPER.md
L198-206) weight column pins this choice (DESIGN.md PIN-9).

The four networks follow the paper's experiments (LeNet-5,
AlexNet, VGG-16, ResNet-20/56/110/224/362); the exact LeNet/AlexNet/VGG
layer shapes are not printed in the paper and are the readings AMB-15/16 in
DESIGN.md.
"""
from __future__ import annotations

from dataclasses import dataclass, field, asdict
from typing import List, Tuple


@dataclass(frozen=True)
class LayerSpec:
    kind: str                 # 'conv' | 'fc'
    cin: int                  # conv: input channels; fc: input features (C*H*W)
    cout: int
    k: int = 1
    stride: int = 1
    pad: int = 0
    bias: bool = False
    bn: bool = False
    block_begin: bool = False
    residual: bool = False
    relu: bool = False
    pool: str = "none"        # 'none' | 'max2' | 'gap'
    dropout: float = 0.0      # drop probability, applied after the ReLU (before pooling)

    def as_dict(self):
        return asdict(self)


@dataclass(frozen=True)
class NetSpec:
    name: str
    layers: Tuple[LayerSpec, ...]
    in_shape: Tuple[int, int, int]   # (C, H, W)
    n_classes: int = 10

    @property
    def n_layers(self) -> int:
        return len(self.layers)


def conv(cin, cout, k=3, stride=1, pad=1, **kw) -> LayerSpec:
    return LayerSpec("conv", cin, cout, k, stride, pad, **kw)


def fc(cin, cout, **kw) -> LayerSpec:
    return LayerSpec("fc", cin, cout, 1, 1, 0, **kw)


def lenet5() -> NetSpec:
    """LeNet-5 for 1x28x28 (reading AMB-15): 5 weighted layers (Table 1)."""
    L = [
        conv(1, 6, k=5, pad=2, bias=True, relu=True, pool="max2"),    # 28 -> 14
        conv(6, 16, k=5, pad=0, bias=True, relu=True, pool="max2"),   # 14 -> 10 -> 5
        fc(16 * 5 * 5, 120, bias=True, relu=True),
        fc(120, 84, bias=True, relu=True),
        fc(84, 10, bias=True),
    ]
    return NetSpec("lenet5", tuple(L), (1, 28, 28), 10)


def alexnet_cifar() -> NetSpec:
    """AlexNet for CIFAR-10 (reading AMB-15): 8 weighted layers (Table 1)."""
    L = [
        conv(3, 64, k=5, pad=2, bias=True, relu=True, pool="max2"),     # 32 -> 16
        conv(64, 192, k=5, pad=2, bias=True, relu=True, pool="max2"),   # 16 -> 8
        conv(192, 384, k=3, pad=1, bias=True, relu=True),
        conv(384, 256, k=3, pad=1, bias=True, relu=True),
        conv(256, 256, k=3, pad=1, bias=True, relu=True, pool="max2"),  # 8 -> 4
        fc(256 * 4 * 4, 2048, bias=True, relu=True),
        fc(2048, 2048, bias=True, relu=True),
        fc(2048, 10, bias=True),
    ]
    return NetSpec("alexnet", tuple(L), (3, 32, 32), 10)


def vgg16_cifar(dropout: bool = False) -> NetSpec:
    """VGG-16 with BatchNorm for CIFAR-10 (readings AMB-15/16): 16 weighted layers.
    dropout=True: "batch normalization and dropout are used during training throughout the
    network", placed as in the common CIFAR VGG-BN recipe (reading AMB-16b,
    external): p = 0.3 after the first conv, 0.4 after every other conv not followed by a pool,
    0.5 after each hidden FC."""
    cfg = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]
    L: List[LayerSpec] = []
    c = 3
    for i, v in enumerate(cfg):
        if v == "M":
            continue
        pool = "max2" if i + 1 < len(cfg) and cfg[i + 1] == "M" else "none"
        p = 0.0 if (not dropout or pool != "none") else (0.3 if not L else 0.4)
        L.append(conv(c, v, k=3, pad=1, bn=True, relu=True, pool=pool, dropout=p))
        c = v
    q = 0.5 if dropout else 0.0
    L += [fc(512, 512, bias=True, relu=True, dropout=q), fc(512, 512, bias=True, relu=True, dropout=q),
          fc(512, 10, bias=True)]
    return NetSpec("vgg16_dropout" if dropout else "vgg16", tuple(L), (3, 32, 32), 10)


def resnet_cifar(depth: int) -> NetSpec:
    """ResNet-(6n+2) for CIFAR-10 (option-A shortcut).

    conv1 3->16 + BN + ReLU; three groups of n BasicBlocks with 16/32/64
    channels at 32^2/16^2/8^2; global average pool; FC 64->10.  Weighted
    layers: 1 + 6n + 1 = depth.  Block boundaries are after layers 1+2k.
    """
    assert (depth - 2) % 6 == 0, depth
    n = (depth - 2) // 6
    L: List[LayerSpec] = [conv(3, 16, bn=True, relu=True)]
    cin = 16
    for g, cout in enumerate((16, 32, 64)):
        for b in range(n):
            stride = 2 if (g > 0 and b == 0) else 1
            L.append(conv(cin, cout, stride=stride, bn=True, relu=True, block_begin=True))
            last = (g == 2 and b == n - 1)
            L.append(conv(cout, cout, bn=True, residual=True, relu=True,
                          pool="gap" if last else "none"))
            cin = cout
    L.append(fc(64, 10, bias=True))
    return NetSpec(f"resnet{depth}", tuple(L), (3, 32, 32), 10)


def tiny_resnet(width: int = 8, hw: int = 8, n: int = 1) -> NetSpec:
    """A small option-A ResNet (same structure as resnet_cifar) for fast tests."""
    L: List[LayerSpec] = [conv(3, width, bn=True, relu=True)]
    cin = width
    for g, cout in enumerate((width, 2 * width)):
        for b in range(n):
            stride = 2 if (g > 0 and b == 0) else 1
            L.append(conv(cin, cout, stride=stride, bn=True, relu=True, block_begin=True))
            last = (g == 1 and b == n - 1)
            L.append(conv(cout, cout, bn=True, residual=True, relu=True,
                          pool="gap" if last else "none"))
            cin = cout
    L.append(fc(cin, 10, bias=True))
    return NetSpec(f"tiny_resnet_w{width}_hw{hw}_n{n}", tuple(L), (3, hw, hw), 10)


def tiny_cnn(hw: int = 8, dropout: float = 0.0) -> NetSpec:
    """A small LeNet-like net (bias, ReLU, max-pool, FC) for fast tests; `dropout` > 0 puts dropout
    after the first conv's ReLU (before its pool) and after the hidden FC's ReLU."""
    L = [
        conv(1, 4, k=3, pad=1, bias=True, relu=True, pool="max2", dropout=dropout),
        conv(4, 6, k=3, pad=1, bias=True, relu=True, pool="max2"),
        fc(6 * (hw // 4) * (hw // 4), 12, bias=True, relu=True, dropout=dropout),
        fc(12, 10, bias=True),
    ]
    return NetSpec(f"tiny_cnn_hw{hw}" + (f"_do{dropout}" if dropout else ""), tuple(L), (1, hw, hw), 10)


def by_name(name: str) -> NetSpec:
    if name == "lenet5":
        return lenet5()
    if name == "alexnet":
        return alexnet_cifar()
    if name == "vgg16":
        return vgg16_cifar()
    if name == "vgg16_dropout":
        return vgg16_cifar(dropout=True)
    if name.startswith("resnet"):
        return resnet_cifar(int(name[len("resnet"):]))
    raise KeyError(name)


def weighted_layer_count(net: NetSpec) -> int:
    return len(net.layers)


def layer_param_shapes(L: LayerSpec):
    """Canonical parameter tensors of one weighted layer, in canonical order.

    conv: W (cout, cin, k, k) [OIHW]; FC: W (cout, cin) with cin in the
    NCHW-flatten order of the incoming tensor; then bias (cout,) if bias;
    then BN gamma (cout,), beta (cout,) if bn.
    """
    out = []
    if L.kind == "conv":
        out.append(("W", (L.cout, L.cin, L.k, L.k)))
    else:
        out.append(("W", (L.cout, L.cin)))
    if L.bias:
        out.append(("b", (L.cout,)))
    if L.bn:
        out.append(("gamma", (L.cout,)))
        out.append(("beta", (L.cout,)))
    return out


def param_count(net: NetSpec) -> int:
    tot = 0
    for L in net.layers:
        for _, shp in layer_param_shapes(L):
            n = 1
            for d in shp:
                n *= d
            tot += n
    return tot
