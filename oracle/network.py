"""Stages of a CNN and their forward/backward passes (TEST INFRASTRUCTURE ONLY).

PAPER.md L67 (§3): a Pipeline Placement Vector PPV = (p_1, ..., p_K) inserts
a register pair after weighted layer p_i; "FS_i and BKS_{K-i+2} correspond
to the same set of layers".  Reading AMB-13 (the printed "p_i+1 to p_{i+1}"
is off by one): stage i (1-indexed) holds weighted layers p_{i-1}+1 .. p_i
with p_0 = 0 and p_{K+1} = L.  Here stages are 0-indexed: stage s holds
0-based layer indices [p_s, p_{s+1}) with p_0 = 0, p_K = L.

A layer spec is any object with the attributes of pst_workloads.LayerSpec
(kind, cin, cout, k, stride, pad, bias, bn, block_begin, residual, relu,
pool).  Parameters of a layer are a dict {'W', 'b', 'gamma', 'beta'}.
"""
from __future__ import annotations

import numpy as np

from . import layers as Lx


# --------------------------------------------------------------------------- parameters
def _shapes(L):
    out = [("W", (L.cout, L.cin, L.k, L.k) if L.kind == "conv" else (L.cout, L.cin))]
    if L.bias:
        out.append(("b", (L.cout,)))
    if L.bn:
        out.append(("gamma", (L.cout,)))
        out.append(("beta", (L.cout,)))
    return out


def unflatten(layer_specs, flat):
    """Canonical flat vector -> list of per-layer parameter dicts (float64 copies)."""
    flat = np.asarray(flat, dtype=np.float64)
    out, off = [], 0
    for L in layer_specs:
        d = {}
        for name, shp in _shapes(L):
            n = int(np.prod(shp))
            d[name] = flat[off:off + n].reshape(shp).copy()
            off += n
        out.append(d)
    assert off == flat.size, (off, flat.size)
    return out


def flatten(layer_specs, params):
    chunks = []
    for L, d in zip(layer_specs, params):
        for name, _ in _shapes(L):
            chunks.append(d[name].ravel())
    return np.concatenate(chunks) if chunks else np.zeros(0)


def n_params(layer_specs):
    return sum(int(np.prod(s)) for L in layer_specs for _, s in _shapes(L))


# --------------------------------------------------------------------------- partition
def partition(layer_specs, ppv):
    """PPV -> list of (start, end) 0-based layer ranges, validated: strictly increasing, each p in
    [1, L-1].  A boundary may fall inside a residual block (the paper's ResNet-20 PPV (5,12,17),
    P:L179 section 6.4, and its fine-grained placements "within residual function blocks", P:L135
    section 6.3): the register pair then carries two tensors -- see CNNStage (reading AMB-14)."""
    Lcount = len(layer_specs)
    ppv = [int(p) for p in ppv]
    if any(p < 1 or p > Lcount - 1 for p in ppv):
        raise ValueError(f"PPV entries must be in [1, {Lcount - 1}]: {ppv}")
    if any(b <= a for a, b in zip(ppv, ppv[1:])):
        raise ValueError(f"PPV must be strictly increasing: {ppv}")
    bounds = [0] + ppv + [Lcount]
    return [(bounds[s], bounds[s + 1]) for s in range(len(bounds) - 1)]


def open_block_at(layer_specs):
    """open[p]: True if a residual block is open between layers p-1 and p (0-based), i.e. a
    register pair after 1-based layer p sits inside a residual block (mid-block register)."""
    out, is_open = [], False
    for L in layer_specs:
        out.append(is_open)
        if L.block_begin:
            is_open = True
        if L.residual:
            is_open = False
    out.append(False)
    return out


def stale_weight_percentage(layer_specs, ppv):
    """(sum_{i<=K} N_i) / (sum_{i<=K+1} N_i) -- the share of
    weights outside the last stage."""
    st = partition(layer_specs, ppv)
    counts = [n_params(layer_specs[a:b]) for a, b in st]
    return 100.0 * sum(counts[:-1]) / sum(counts)


# --------------------------------------------------------------------------- stage passes
class CNNStage:
    """One pipeline stage: contiguous weighted layers with their attached ops.

    forward(params, x)  -> (out, cache); updates BN running statistics (state)
    backward(params, cache, g_out) -> (g_in, grads) with the params given
    (the *current* weights, PAPER.md L63/L75 + reading AMB-2).
    """

    def __init__(self, layer_specs, first_stage=False, bn_momentum=0.1, bn_eps=1e-5, dropout_seed=0, layer0=0):
        """Mid-block registers (reading AMB-14): a stage whose first layer lies inside a residual
        block receives (activation, block input) and, in the backward, returns (gradient of the
        activation, gradient of the block input through the shortcut); a stage that ends inside a
        block emits (activation, block input) and receives the same pair of gradients."""
        self.layers = list(layer_specs)
        self.first_stage = first_stage
        self.dropout_seed = dropout_seed   # counter-based dropout masks (layers.dropout_mask)
        self.layer0 = layer0               # network index of this stage's first layer
        self.bn_momentum = bn_momentum
        self.bn_eps = bn_eps
        self.state = [
            {"run_mean": np.zeros(L.cout), "run_var": np.ones(L.cout)} if L.bn else {}
            for L in self.layers
        ]

    def forward(self, params, x, mb=0):
        """mb: the mini-batch index (it selects the dropout masks; nothing else depends on it)."""
        block_in = None
        if isinstance(x, tuple):                 # mid-block register: (activation, block input)
            x, block_in = x
            block_in = np.asarray(block_in, dtype=np.float64)
        a = np.asarray(x, dtype=np.float64)
        caches = []
        for L, P, S in zip(self.layers, params, self.state):
            c = {"x": a}
            if L.block_begin:
                block_in = a
            if L.kind == "conv":
                y = Lx.conv2d_forward(a, P["W"], P.get("b"), L.stride, L.pad)
            else:
                y = Lx.fc_forward(a, P["W"], P.get("b"))
            if L.bn:
                y, c["bn"] = Lx.bn_train_forward(y, P["gamma"], P["beta"], self.bn_eps)
                xhat, invstd, mean, var, M = c["bn"]
                S["run_mean"], S["run_var"] = Lx.bn_running_update(
                    S["run_mean"], S["run_var"], mean, var, M, self.bn_momentum)
            if L.residual:
                assert block_in is not None, "residual without block input in this stage"
                c["block_in_shape"] = block_in.shape
                y = y + Lx.shortcut_forward(block_in, y.shape)
            if L.relu:
                y, c["mask"] = Lx.relu_forward(y)
            if getattr(L, "dropout", 0.0) > 0.0:
                c["drop"] = Lx.dropout_mask(self.dropout_seed, mb, self.layer0 + len(caches), y.shape, L.dropout)
                y = y * c["drop"]
            if L.pool == "max2":
                c["pool_in_shape"] = y.shape
                y, c["arg"] = Lx.maxpool2_forward(y)
            elif L.pool == "gap":
                c["pool_in_shape"] = y.shape
                y = Lx.gap_forward(y)
            if L.residual:
                block_in = None                  # the block is closed
            caches.append(c)
            a = y
        if block_in is not None:                 # the stage ends inside a block
            return (a, block_in), caches
        return a, caches

    def backward(self, params, caches, g_out):
        g_shortcut = None
        if isinstance(g_out, tuple):             # the stage ends inside a block
            g_out, g_shortcut = g_out
            g_shortcut = np.asarray(g_shortcut, dtype=np.float64)
        g = np.asarray(g_out, dtype=np.float64)
        grads = [None] * len(self.layers)
        for idx in range(len(self.layers) - 1, -1, -1):
            L, P, c = self.layers[idx], params[idx], caches[idx]
            if L.pool == "max2":
                g = Lx.maxpool2_backward(g, c["arg"], c["pool_in_shape"])
            elif L.pool == "gap":
                g = Lx.gap_backward(g, c["pool_in_shape"])
            if "drop" in c:
                g = g * c["drop"]
            if L.relu:
                g = Lx.relu_backward(g, c["mask"])
            if L.residual:
                g_shortcut = Lx.shortcut_backward(g, c["block_in_shape"])
            gr = {}
            if L.bn:
                g, gr["gamma"], gr["beta"] = Lx.bn_train_backward(g, c["bn"], P["gamma"])
            need_gx = not (self.first_stage and idx == 0)
            if L.kind == "conv":
                gx, gW, gb = Lx.conv2d_backward(c["x"], P["W"], g, L.stride, L.pad, need_gx)
            else:
                gx, gW, gb = Lx.fc_backward(c["x"], P["W"], g, need_gx)
            gr["W"] = gW
            if L.bias:
                gr["b"] = gb
            if L.block_begin and gx is not None:
                gx = gx + g_shortcut
                g_shortcut = None
            grads[idx] = gr
            g = gx
        if g_shortcut is not None:               # the stage starts inside a block
            return (g, g_shortcut), grads
        return g, grads

    def bn_stats(self):
        return [(S["run_mean"].copy(), S["run_var"].copy()) if S else None for S in self.state]
