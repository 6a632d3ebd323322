"""The oracle with the CUDA path's storage roundings emulated (tests only; reading AMB-21e).

`EmuStage` is oracle.network.CNNStage run through a namespace of oracle.layers whose results are
rounded the way libpst stores them: every activation, gradient and BN output in float32, and the
operands of every convolution / FC product split as 3xTF32 (hi = tf32 truncation, lo = tf32 of the
remainder; the product keeps hi*hi + hi*lo + lo*hi).  Reductions stay in float64 (libpst
accumulates in fp32 TMEM / fp64 BN sums).  The deviation of this emulation from the exact oracle is
the size of error a float32 implementation of the same arithmetic makes -- the yardstick for the
quantities whose per-tensor ratio is ill-conditioned (momentum buffers, BN running statistics):
their tolerance is max(2e-3, K_EMU x that deviation), tests/parity.py.
"""
from __future__ import annotations

import types

import numpy as np

from oracle import layers as Lx
from oracle import network as Net


def _r32(a):
    return np.asarray(np.asarray(a, dtype=np.float64).astype(np.float32), dtype=np.float64)


def _tf32x3(a):
    """a = hi + lo with hi = tf32 truncation of float32(a), lo = tf32 (round) of the remainder."""
    a32 = np.asarray(a, dtype=np.float32)
    hi = (a32.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
    rem = (a32 - hi).astype(np.float32)
    lo = ((rem.view(np.uint32) + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)
    return hi.astype(np.float64) + lo.astype(np.float64)


def _emu_layers():
    ns = types.SimpleNamespace(**{k: getattr(Lx, k) for k in dir(Lx) if not k.startswith("__")})

    def conv2d_forward(x, W, b, stride, pad):
        return _r32(Lx.conv2d_forward(_tf32x3(x), _tf32x3(W), b, stride, pad))

    def conv2d_backward(x, W, gy, stride, pad, need_gx=True):
        gx, gW, gb = Lx.conv2d_backward(_tf32x3(x), _tf32x3(W), _tf32x3(gy), stride, pad, need_gx)
        return (None if gx is None else _r32(gx)), _r32(gW), (None if gb is None else _r32(gb))

    def fc_forward(x, W, b):
        return _r32(Lx.fc_forward(_tf32x3(x), _tf32x3(W), b))

    def fc_backward(x, W, gy, need_gx=True):
        gx, gW, gb = Lx.fc_backward(_tf32x3(x), _tf32x3(W), _tf32x3(gy), need_gx)
        return (None if gx is None else _r32(gx)), _r32(gW), (None if gb is None else _r32(gb))

    def bn_train_forward(y, gamma, beta, eps):
        z, cache = Lx.bn_train_forward(_r32(y), gamma, beta, eps)
        return _r32(z), cache

    def bn_train_backward(gz, cache, gamma):
        g, gg, gb = Lx.bn_train_backward(_r32(gz), cache, gamma)
        return _r32(g), _r32(gg), _r32(gb)

    ns.conv2d_forward, ns.conv2d_backward = conv2d_forward, conv2d_backward
    ns.fc_forward, ns.fc_backward = fc_forward, fc_backward
    ns.bn_train_forward, ns.bn_train_backward = bn_train_forward, bn_train_backward
    return ns


_EMU = _emu_layers()


class EmuStage(Net.CNNStage):
    """CNNStage with libpst's storage roundings (module docstring)."""

    def _swap(self, fn, *a, **k):
        saved = Net.Lx
        Net.Lx = _EMU
        try:
            return fn(*a, **k)
        finally:
            Net.Lx = saved

    def forward(self, params, x, mb=0):
        return self._swap(Net.CNNStage.forward, self, params, x, mb=mb)

    def backward(self, params, caches, g_out):
        return self._swap(Net.CNNStage.backward, self, params, caches, g_out)
