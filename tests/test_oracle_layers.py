"""Pins for oracle/layers.py (CPU, no GPU).

Each layer's forward is checked against PyTorch-CPU float64 functional ops
(an independent library routine), and each VJP against central finite
differences in float64 (the mathematics).  A dropped term, wrong sign, wrong
index or transposed operand in any op fails one of these.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import layers as Lx

RNG = np.random.default_rng(0)


def fd_check(f, args, idx, g_analytic, eps=1e-6, n_dirs=3, rtol=1e-6):
    """Directional central differences: <g, v> == (f(x+eps v) - f(x-eps v)) / 2eps
    where f returns sum(out * R) for a fixed random R."""
    x = args[idx]
    for _ in range(n_dirs):
        v = RNG.standard_normal(x.shape)
        ap = list(args); ap[idx] = x + eps * v
        am = list(args); am[idx] = x - eps * v
        num = (f(*ap) - f(*am)) / (2 * eps)
        ana = float(np.sum(g_analytic * v))
        assert abs(num - ana) <= rtol * max(1.0, abs(num)), (num, ana)


@pytest.mark.parametrize("k,stride,pad,H", [(3, 1, 1, 6), (3, 2, 1, 6), (5, 1, 2, 6), (5, 1, 0, 7), (1, 1, 0, 4)])
def test_conv_forward_matches_torch(k, stride, pad, H):
    x = RNG.standard_normal((2, 3, H, H + 1))
    W = RNG.standard_normal((4, 3, k, k))
    b = RNG.standard_normal(4)
    y = Lx.conv2d_forward(x, W, b, stride, pad)
    yt = F.conv2d(torch.from_numpy(x), torch.from_numpy(W), torch.from_numpy(b), stride=stride, padding=pad)
    np.testing.assert_allclose(y, yt.numpy(), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("k,stride,pad,H", [(3, 1, 1, 5), (3, 2, 1, 6), (5, 1, 2, 5), (5, 1, 0, 7)])
def test_conv_backward_finite_differences(k, stride, pad, H):
    x = RNG.standard_normal((2, 3, H, H))
    W = RNG.standard_normal((4, 3, k, k))
    b = RNG.standard_normal(4)
    R = RNG.standard_normal(Lx.conv2d_forward(x, W, b, stride, pad).shape)
    gx, gW, gb = Lx.conv2d_backward(x, W, R, stride, pad)
    f = lambda x_, W_, b_: float(np.sum(Lx.conv2d_forward(x_, W_, b_, stride, pad) * R))
    fd_check(f, [x, W, b], 0, gx)
    fd_check(f, [x, W, b], 1, gW)
    fd_check(f, [x, W, b], 2, gb)


def test_conv_backward_matches_torch_autograd():
    x = torch.from_numpy(RNG.standard_normal((2, 4, 8, 8))).requires_grad_()
    W = torch.from_numpy(RNG.standard_normal((6, 4, 3, 3))).requires_grad_()
    y = F.conv2d(x, W, stride=2, padding=1)
    R = torch.from_numpy(RNG.standard_normal(tuple(y.shape)))
    (y * R).sum().backward()
    gx, gW, gb = Lx.conv2d_backward(x.detach().numpy(), W.detach().numpy(), R.numpy(), 2, 1)
    np.testing.assert_allclose(gx, x.grad.numpy(), rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(gW, W.grad.numpy(), rtol=1e-11, atol=1e-11)


def test_fc_forward_backward():
    x = RNG.standard_normal((3, 2, 2, 2))
    W = RNG.standard_normal((5, 8))
    b = RNG.standard_normal(5)
    y = Lx.fc_forward(x, W, b)
    np.testing.assert_allclose(y, F.linear(torch.from_numpy(x).flatten(1), torch.from_numpy(W), torch.from_numpy(b)).numpy(), rtol=1e-12)
    R = RNG.standard_normal(y.shape)
    gx, gW, gb = Lx.fc_backward(x, W, R)
    f = lambda x_, W_, b_: float(np.sum(Lx.fc_forward(x_, W_, b_) * R))
    fd_check(f, [x, W, b], 0, gx)
    fd_check(f, [x, W, b], 1, gW)
    fd_check(f, [x, W, b], 2, gb)


@pytest.mark.parametrize("shape", [(4, 3, 5, 5), (6, 4)])
def test_bn_forward_matches_torch(shape):
    y = RNG.standard_normal(shape) * 3 + 1
    C = shape[1]
    g, be = RNG.standard_normal(C), RNG.standard_normal(C)
    rm, rv = RNG.standard_normal(C), RNG.random(C) + 0.5
    z, cache = Lx.bn_train_forward(y, g, be, 1e-5)
    xhat, invstd, mean, var, M = cache
    rm2, rv2 = Lx.bn_running_update(rm, rv, mean, var, M, 0.1)
    rmt, rvt = torch.from_numpy(rm.copy()), torch.from_numpy(rv.copy())
    zt = F.batch_norm(torch.from_numpy(y), rmt, rvt, torch.from_numpy(g), torch.from_numpy(be),
                      training=True, momentum=0.1, eps=1e-5)
    np.testing.assert_allclose(z, zt.numpy(), rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(rm2, rmt.numpy(), rtol=1e-12)
    np.testing.assert_allclose(rv2, rvt.numpy(), rtol=1e-12)


@pytest.mark.parametrize("shape", [(4, 3, 3, 3), (5, 4)])
def test_bn_backward_finite_differences(shape):
    y = RNG.standard_normal(shape) * 2 + 0.5
    C = shape[1]
    g, be = RNG.standard_normal(C), RNG.standard_normal(C)
    R = RNG.standard_normal(shape)
    z, cache = Lx.bn_train_forward(y, g, be, 1e-5)
    gy, dg, db = Lx.bn_train_backward(R, cache, g)
    f = lambda y_, g_, b_: float(np.sum(Lx.bn_train_forward(y_, g_, b_, 1e-5)[0] * R))
    fd_check(f, [y, g, be], 0, gy)
    fd_check(f, [y, g, be], 1, dg)
    fd_check(f, [y, g, be], 2, db)


def test_bn_backward_uses_given_gamma_linearly():
    """No stash: the backward's dx scales with the gamma passed in (the current one)."""
    y = RNG.standard_normal((4, 3, 2, 2))
    g0 = RNG.standard_normal(3)
    R = RNG.standard_normal(y.shape)
    _, cache = Lx.bn_train_forward(y, g0, np.zeros(3), 1e-5)
    gy1, dg1, db1 = Lx.bn_train_backward(R, cache, g0)
    gy2, dg2, db2 = Lx.bn_train_backward(R, cache, 2.0 * g0)
    np.testing.assert_allclose(gy2, 2.0 * gy1, rtol=1e-12, atol=1e-14)
    np.testing.assert_array_equal(dg1, dg2)
    np.testing.assert_array_equal(db1, db2)


def test_relu_and_subgradient_at_zero():
    y = np.array([-1.0, 0.0, 2.0])
    z, m = Lx.relu_forward(y)
    np.testing.assert_array_equal(z, [0.0, 0.0, 2.0])
    np.testing.assert_array_equal(Lx.relu_backward(np.ones(3), m), [0.0, 0.0, 1.0])


def test_maxpool_forward_backward():
    x = RNG.standard_normal((2, 3, 6, 4))
    out, arg = Lx.maxpool2_forward(x)
    xt = torch.from_numpy(x).requires_grad_()
    ot = F.max_pool2d(xt, 2, 2)
    np.testing.assert_array_equal(out, ot.detach().numpy())
    R = RNG.standard_normal(out.shape)
    (ot * torch.from_numpy(R)).sum().backward()
    np.testing.assert_array_equal(Lx.maxpool2_backward(R, arg, x.shape), xt.grad.numpy())


def test_maxpool_tie_break_first_max():
    x = np.zeros((1, 1, 2, 2))
    x[0, 0] = [[1.0, 3.0], [3.0, 3.0]]
    out, arg = Lx.maxpool2_forward(x)
    assert out[0, 0, 0, 0] == 3.0 and arg[0, 0, 0, 0] == 1
    g = Lx.maxpool2_backward(np.ones((1, 1, 1, 1)), arg, x.shape)
    np.testing.assert_array_equal(g[0, 0], [[0, 1], [0, 0]])


def test_gap_forward_backward():
    x = RNG.standard_normal((2, 3, 4, 4))
    np.testing.assert_allclose(Lx.gap_forward(x), F.adaptive_avg_pool2d(torch.from_numpy(x), 1).numpy()[:, :, 0, 0], rtol=1e-13)
    R = RNG.standard_normal((2, 3))
    fd_check(lambda x_: float(np.sum(Lx.gap_forward(x_) * R)), [x], 0, Lx.gap_backward(R, x.shape))


def test_shortcut_option_a():
    x = RNG.standard_normal((2, 4, 6, 6))
    y = Lx.shortcut_forward(x, (2, 8, 3, 3))
    assert np.all(y[:, :2] == 0) and np.all(y[:, 6:] == 0)
    np.testing.assert_array_equal(y[:, 2:6], x[:, :, ::2, ::2])
    R = RNG.standard_normal(y.shape)
    fd_check(lambda x_: float(np.sum(Lx.shortcut_forward(x_, (2, 8, 3, 3)) * R)), [x], 0,
             Lx.shortcut_backward(R, x.shape))
    assert Lx.shortcut_forward(x, x.shape) is x


def test_softmax_ce_matches_torch_and_fd():
    z = RNG.standard_normal((5, 10)) * 3
    y = RNG.integers(0, 10, size=5)
    loss, dz = Lx.softmax_ce(z, y)
    zt = torch.from_numpy(z).requires_grad_()
    lt = F.cross_entropy(zt, torch.from_numpy(y).long())
    lt.backward()
    assert abs(loss - lt.item()) < 1e-12
    np.testing.assert_allclose(dz, zt.grad.numpy(), rtol=1e-11, atol=1e-14)


def test_sgd_matches_torch_optim():
    w = RNG.standard_normal(7)
    grads = [RNG.standard_normal(7) for _ in range(4)]
    lrs = [0.1, 0.1, 0.01, 0.01]
    p = torch.nn.Parameter(torch.from_numpy(w.copy()))
    opt = torch.optim.SGD([p], lr=0.1, momentum=0.9, weight_decay=1e-3)
    wv, vv = w.copy(), np.zeros(7)
    for g, lr in zip(grads, lrs):
        for gr in opt.param_groups:
            gr["lr"] = lr
        p.grad = torch.from_numpy(g.copy())
        opt.step()
        wv, vv = Lx.sgd_momentum(wv, vv, g, lr, 0.9, 1e-3)
    np.testing.assert_allclose(wv, p.detach().numpy(), rtol=1e-13, atol=1e-15)
