"""Per-operation definitions in float64 (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

PAPER.md §2 (L43-49): the forward pass computes the activations x^(l) of each
layer from x^(l-1) and W^(l); the backward pass computes delta^(l), the
weight gradients de/dW^(l) from x^(l-1) and delta^(l), and delta^(l-1) from
delta^(l).  Each function below is the plain definition of one operation
and of its vector-Jacobian product.  Tensors are NCHW float64.  Conventions
the paper does not state are the readings in DESIGN.md (PyTorch semantics:
AMB-6 BatchNorm, AMB-7 SGD, AMB-18 max-pool ties / ReLU'(0)=0).
"""
from __future__ import annotations

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view


# --------------------------------------------------------------------------- conv
def _cols(x, k, stride, pad):
    """cols[n, c, i, j, r, s] = xpad[n, c, i*stride + r, j*stride + s]."""
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    win = sliding_window_view(xp, (k, k), axis=(2, 3))   # (N, C, Hp-k+1, Wp-k+1, k, k)
    return win[:, :, ::stride, ::stride]


def conv2d_forward(x, W, b, stride, pad):
    """y[n,o,i,j] = sum_{c,r,s} W[o,c,r,s] * xpad[n,c,i*S+r,j*S+s] + b[o]  (cross-correlation)."""
    k = W.shape[2]
    cols = _cols(x, k, stride, pad)
    y = np.tensordot(cols, W, axes=([1, 4, 5], [1, 2, 3]))   # (N, Ho, Wo, O)
    y = np.ascontiguousarray(y.transpose(0, 3, 1, 2))
    if b is not None:
        y = y + b[None, :, None, None]
    return y


def conv2d_backward(x, W, gy, stride, pad, need_gx=True):
    """VJP of conv2d_forward.

    gW[o,c,r,s] = sum_{n,i,j} gy[n,o,i,j] xpad[n,c,iS+r,jS+s]   (uses the saved input x)
    gb[o]       = sum_{n,i,j} gy[n,o,i,j]
    gx          = scatter-add of sum_o gy[n,o,i,j] W[o,c,r,s] into xpad[n,c,iS+r,jS+s], cropped
    """
    k = W.shape[2]
    N, C, H, Wd = x.shape
    _, O, Ho, Wo = gy.shape
    cols = _cols(x, k, stride, pad)
    gW = np.tensordot(gy, cols, axes=([0, 2, 3], [0, 2, 3]))   # (O, C, k, k)
    gb = gy.sum(axis=(0, 2, 3))
    gx = None
    if need_gx:
        gcols = np.tensordot(W, gy, axes=([0], [1]))           # (C, k, k, N, Ho, Wo)
        gxp = np.zeros((N, C, H + 2 * pad, Wd + 2 * pad))
        for r in range(k):
            for s in range(k):
                gxp[:, :, r:r + stride * (Ho - 1) + 1:stride,
                    s:s + stride * (Wo - 1) + 1:stride] += gcols[:, r, s].transpose(1, 0, 2, 3)
        gx = gxp[:, :, pad:pad + H, pad:pad + Wd]
        gx = np.ascontiguousarray(gx)
    return gx, gW, gb


# --------------------------------------------------------------------------- fully connected
def fc_forward(x, W, b):
    """y = flatten(x) W^T + b, flatten in NCHW order."""
    xf = x.reshape(x.shape[0], -1)
    y = xf @ W.T
    if b is not None:
        y = y + b[None, :]
    return y


def fc_backward(x, W, gy, need_gx=True):
    xf = x.reshape(x.shape[0], -1)
    gW = gy.T @ xf
    gb = gy.sum(axis=0)
    gx = (gy @ W).reshape(x.shape) if need_gx else None
    return gx, gW, gb


# --------------------------------------------------------------------------- batch norm (train mode)
def bn_train_forward(y, gamma, beta, eps):
    """Training-mode BatchNorm over (N, H, W) per channel (reading AMB-6).

    mean, biased var over the mini-batch; xhat = (y - mean)/sqrt(var + eps);
    z = gamma * xhat + beta.  Returns z and the cache (xhat, invstd, mean, var, M).
    Works for (N, C) and (N, C, H, W).
    """
    axes = (0,) if y.ndim == 2 else (0, 2, 3)
    M = y.size // y.shape[1]
    mean = y.mean(axis=axes)
    var = ((y - _bc(mean, y)) ** 2).mean(axis=axes)
    invstd = 1.0 / np.sqrt(var + eps)
    xhat = (y - _bc(mean, y)) * _bc(invstd, y)
    z = _bc(gamma, y) * xhat + _bc(beta, y)
    return z, (xhat, invstd, mean, var, M)


def bn_running_update(run_mean, run_var, mean, var, M, momentum):
    """PyTorch running statistics: r <- (1-m) r + m * stat, variance unbiased (M/(M-1))."""
    new_mean = (1.0 - momentum) * run_mean + momentum * mean
    new_var = (1.0 - momentum) * run_var + momentum * var * (M / (M - 1.0))
    return new_mean, new_var


def bn_train_backward(gz, cache, gamma):
    """VJP of bn_train_forward w.r.t. y, gamma, beta.

    `gamma` is the CURRENT gamma (no weight stashing, reading AMB-2/6); the
    cache holds the forward's xhat and invstd.
        dbeta = sum gz ;  dgamma = sum gz*xhat
        gy = gamma*invstd/M * (M*gz - dbeta - xhat*dgamma)
    """
    xhat, invstd, _mean, _var, M = cache
    axes = (0,) if gz.ndim == 2 else (0, 2, 3)
    dbeta = gz.sum(axis=axes)
    dgamma = (gz * xhat).sum(axis=axes)
    gy = _bc(gamma * invstd / M, gz) * (M * gz - _bc(dbeta, gz) - xhat * _bc(dgamma, gz))
    return gy, dgamma, dbeta


def _bc(v, like):
    return v[None, :] if like.ndim == 2 else v[None, :, None, None]


# --------------------------------------------------------------------------- relu
def relu_forward(y):
    mask = y > 0
    return y * mask, mask


def relu_backward(g, mask):
    """ReLU'(y) = 1 if y > 0 else 0 (ReLU'(0) = 0, reading AMB-18)."""
    return g * mask


# --------------------------------------------------------------------------- dropout
def _fmix32(h):
    """MurmurHash3's 32-bit finaliser on uint32 arrays (wrap-around arithmetic)."""
    h = np.asarray(h, dtype=np.uint32).copy()
    h ^= h >> np.uint32(16)
    h *= np.uint32(0x85EBCA6B)
    h ^= h >> np.uint32(13)
    h *= np.uint32(0xC2B2AE35)
    h ^= h >> np.uint32(16)
    return h


def dropout_threshold(p):
    """Integer keep threshold of drop probability p (p read as float32, as the ABI passes it):
    an element is dropped iff its 32-bit hash is < floor(p * 2^32)."""
    return min(2 ** 32 - 1, int(np.floor(float(np.float32(p)) * 2.0 ** 32)))


def dropout_mask(seed, mb, layer, shape, p):
    """Inverted dropout (VGG-16 "batch normalization and dropout ... throughout", PAPER.md L288,
    SURVEY f-3) with a counter-based generator shared by definition with the CUDA path: for
    mini-batch `mb`, 0-based weighted layer `layer` and the element's logical NCHW index e,
        key = fmix32(seed ^ fmix32(mb * 0x9E3779B9 + (layer + 1) * 0x632BE5AB))
        u   = fmix32(e ^ key);   keep iff u >= floor(p * 2^32)
    (uint32 wrap-around arithmetic).  The mask depends only on (seed, mb, layer, e): the stale
    forward of mini-batch i draws exactly the mask a non-pipelined forward of i would.
    Returns 0 or 1/(1-p) per element (float64)."""
    with np.errstate(over="ignore"):
        pre = np.uint32((int(mb) * 0x9E3779B9 + (int(layer) + 1) * 0x632BE5AB) & 0xFFFFFFFF)
        key = _fmix32(np.uint32(int(seed) & 0xFFFFFFFF) ^ _fmix32(pre))
        e = (np.arange(int(np.prod(shape)), dtype=np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        u = _fmix32(e ^ key)
    keep = u >= np.uint32(dropout_threshold(p)) if dropout_threshold(p) > 0 else np.ones(u.shape, bool)
    scale = 1.0 / (1.0 - float(np.float32(p)))
    return (keep.astype(np.float64) * scale).reshape(shape)


# --------------------------------------------------------------------------- pooling
def maxpool2_forward(x):
    """2x2 max-pool, stride 2.  Tie-break: first maximum in row-major window
    order (0,0),(0,1),(1,0),(1,1) with a strict '>' scan (reading AMB-18)."""
    N, C, H, W = x.shape
    assert H % 2 == 0 and W % 2 == 0, (H, W)
    cand = [x[:, :, a::2, b::2] for a in (0, 1) for b in (0, 1)]
    out = cand[0].copy()
    arg = np.zeros(out.shape, dtype=np.int8)
    for q in range(1, 4):
        better = cand[q] > out
        out = np.where(better, cand[q], out)
        arg = np.where(better, q, arg).astype(np.int8)
    return out, arg


def maxpool2_backward(g, arg, in_shape):
    gx = np.zeros(in_shape)
    for q, (a, b) in enumerate(((0, 0), (0, 1), (1, 0), (1, 1))):
        gx[:, :, a::2, b::2] += g * (arg == q)
    return gx


def gap_forward(x):
    """Global average pool over H, W: (N, C, H, W) -> (N, C)."""
    return x.mean(axis=(2, 3))


def gap_backward(g, in_shape):
    N, C, H, W = in_shape
    return np.broadcast_to(g[:, :, None, None] / (H * W), in_shape).copy()


# --------------------------------------------------------------------------- residual shortcut
def shortcut_forward(x, out_shape):
    """Identity when shapes match; otherwise CIFAR-ResNet option A: take
    x[:, :, ::2, ::2] and zero-pad channels by (Cout - Cin)/2 on each side."""
    if x.shape == tuple(out_shape):
        return x
    N, C, H, W = x.shape
    Co = out_shape[1]
    p = (Co - C) // 2
    sub = x[:, :, ::2, ::2]
    assert sub.shape[2:] == tuple(out_shape[2:]) and Co == C + 2 * p
    out = np.zeros(out_shape)
    out[:, p:p + C] = sub
    return out


def shortcut_backward(g, in_shape):
    """Adjoint of shortcut_forward."""
    if g.shape == tuple(in_shape):
        return g
    C = in_shape[1]
    p = (g.shape[1] - C) // 2
    gx = np.zeros(in_shape)
    gx[:, :, ::2, ::2] = g[:, p:p + C]
    return gx


# --------------------------------------------------------------------------- loss
def softmax_ce(z, y):
    """Mean cross-entropy with the true label (the output x^(L)
    "is used with the true data label to obtain a training error e").
        loss = mean_b( logsumexp(z_b) - z_{b, y_b} ),   dz = (softmax(z) - onehot(y)) / B
    """
    B = z.shape[0]
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    ssum = e.sum(axis=1, keepdims=True)
    lse = (m + np.log(ssum))[:, 0]
    loss = float(np.mean(lse - z[np.arange(B), y]))
    p = e / ssum
    onehot = np.zeros_like(z)
    onehot[np.arange(B), y] = 1.0
    return loss, (p - onehot) / B


# --------------------------------------------------------------------------- optimiser
def sgd_caffe(w, v, g, lr, momentum, weight_decay, nesterov=False):
    """Caffe's SGD and Nesterov solvers (the paper's simulated runs use Caffe, PAPER.md L87;
    AlexNet/VGG-16 use Nesterov momentum, L286/L288):
        v_new <- mu * v + lr * (g + lambda * w)
        SGD:      w <- w - v_new
        Nesterov: w <- w - ((1 + mu) * v_new - mu * v)
    Returns (w_new, v_new)."""
    v_new = momentum * v + lr * (g + weight_decay * w)
    if nesterov:
        return w - ((1.0 + momentum) * v_new - momentum * v), v_new
    return w - v_new, v_new


def sgd_nesterov(w, v, g, lr, momentum, weight_decay):
    """PyTorch's Nesterov form: d = g + lambda w; v <- mu v + d; w <- w - lr (d + mu v)."""
    d = g + weight_decay * w
    v_new = momentum * v + d
    return w - lr * (d + momentum * v_new), v_new


def sgd_momentum(w, v, g, lr, momentum, weight_decay):
    """PyTorch SGD (dampening 0, no Nesterov; reading AMB-7):
        v <- mu * v + (g + lambda * w);  w <- w - lr * v
    Returns (w_new, v_new); inputs are not modified."""
    v_new = momentum * v + (g + weight_decay * w)
    w_new = w - lr * v_new
    return w_new, v_new
