"""Dropout in the oracle (CPU; SURVEY 8(f) f-3 -- VGG-16 trains "with batch normalization and
dropout ... throughout the network", reading AMB-16b).  The masks come from a
counter-based generator (oracle.layers.dropout_mask) that the CUDA path implements from the same
definition; pinned here by an independent Python-integer implementation (tests/torch_ref.py), the
mask's statistics, finite differences, torch autograd + torch.optim.SGD with the same masks, and
the schedule (a stale forward of mini-batch i draws the same mask as a non-pipelined one)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import pst_workloads as W
from oracle import layers as Lx
from oracle import network as Net
from oracle import pipeline as Pl
from tests.parity import oracle_stages
from tests.torch_ref import _fmix32, dropout_mask_py, train_sgd


def test_fmix32_vectorised_equals_python_ints():
    rng = np.random.default_rng(0)
    x = rng.integers(0, 2 ** 32, size=2000, dtype=np.uint64).astype(np.uint32)
    got = Lx._fmix32(x)
    assert [int(v) for v in got] == [_fmix32(int(v)) for v in x]
    assert int(Lx._fmix32(np.uint32(0))) == 0          # fmix32(0) = 0 (every step maps 0 to 0)


@pytest.mark.parametrize("p", [0.3, 0.4, 0.5])
def test_mask_values_keep_rate_and_determinism(p):
    shape = (64, 16, 16, 16)
    m = Lx.dropout_mask(7, 3, 2, shape, p)
    scale = 1.0 / (1.0 - float(np.float32(p)))
    assert set(np.unique(m)) <= {0.0, scale}
    n = m.size
    keep = np.count_nonzero(m) / n
    assert abs(keep - (1 - p)) < 5 * np.sqrt(p * (1 - p) / n)          # binomial 5 sigma
    assert abs(m.mean() - 1.0) < 5 * scale * np.sqrt(p * (1 - p) / n)  # inverted dropout: E[m] = 1
    assert np.array_equal(m, Lx.dropout_mask(7, 3, 2, shape, p))
    # another mini-batch / layer / seed gives an (almost) uncorrelated mask
    for other in [(7, 4, 2), (7, 3, 3), (8, 3, 2)]:
        o = Lx.dropout_mask(*other, shape, p)
        agree = np.mean((m > 0) == (o > 0))
        assert abs(agree - (p * p + (1 - p) * (1 - p))) < 0.01


def test_mask_equals_independent_python_generator():
    shape = (3, 4, 5, 6)
    for seed, mb, layer, p in [(0, 0, 0, 0.5), (12345, 17, 4, 0.3), (2 ** 31 + 5, 1 << 20, 9, 0.4)]:
        a = Lx.dropout_mask(seed, mb, layer, shape, p)
        b = dropout_mask_py(seed, mb, layer, shape, p).numpy()
        assert np.array_equal(a, b)


def test_dropout_stage_finite_differences():
    net = W.tiny_cnn(hw=8, dropout=0.4)
    flat = W.init_params(net, seed=3)
    x, y = W.make_batch(net.in_shape, 4, 0, seed=5)
    st = Net.CNNStage(net.layers, first_stage=False, dropout_seed=11)
    P = Net.unflatten(net.layers, flat)
    out, cache = st.forward(P, x, mb=6)
    _, g = Lx.softmax_ce(out, y)
    gx, G = st.backward(P, cache, g)

    def loss(PP, xx):
        o, _ = Net.CNNStage(net.layers, dropout_seed=11).forward(PP, xx, mb=6)
        return Lx.softmax_ce(o, y)[0]

    rng = np.random.default_rng(1)
    eps = 1e-6
    for li, d in enumerate(P):
        for k in d:
            for _ in range(3):
                idx = tuple(rng.integers(0, n) for n in d[k].shape)
                Pp = [{kk: v.copy() for kk, v in dd.items()} for dd in P]
                Pm = [{kk: v.copy() for kk, v in dd.items()} for dd in P]
                Pp[li][k][idx] += eps
                Pm[li][k][idx] -= eps
                fd = (loss(Pp, x) - loss(Pm, x)) / (2 * eps)
                assert abs(fd - G[li][k][idx]) <= 1e-6 * max(1.0, abs(fd)), (li, k)
    xd = np.asarray(x, dtype=np.float64)
    for _ in range(3):
        idx = tuple(rng.integers(0, n) for n in xd.shape)
        xp, xm = xd.copy(), xd.copy()
        xp[idx] += eps
        xm[idx] -= eps
        assert abs((loss(P, xp) - loss(P, xm)) / (2 * eps) - gx[idx]) <= 1e-6


def test_k1_with_dropout_equals_torch_autograd():
    net = W.tiny_cnn(hw=8, dropout=0.4)
    flat = W.init_params(net, seed=3)
    data = W.batches(net.in_shape, 6, 5, seed=11)
    stages, bounds = oracle_stages(net, (), dropout_seed=99)
    hp = Pl.HParams(lr_pipelined=[0.05], lr_nonpipelined=0.05, momentum=0.9, weight_decay=1e-3)
    res = Pl.run_sgd(stages[0], Net.unflatten(net.layers, flat), data, hp)
    t_losses, t_flat = train_sgd(net, flat, data, 0.05, 0.9, 1e-3, dropout_seed=99)
    np.testing.assert_allclose(res.losses, t_losses, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(Net.flatten(net.layers, res.params[0]), t_flat, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("K,ppv", [(2, (2,)), (4, (1, 2, 3))])
def test_pipelined_dropout_a_equals_b_and_masks_follow_mb(K, ppv):
    net = W.tiny_cnn(hw=8, dropout=0.3)
    flat = W.init_params(net, seed=5)
    data = W.batches(net.in_shape, 6, 9, seed=13)
    hp = Pl.HParams(lr_pipelined=[0.05] * K, lr_nonpipelined=0.05, momentum=0.9, weight_decay=1e-3)
    sa, bounds = oracle_stages(net, ppv, dropout_seed=4)
    sb, _ = oracle_stages(net, ppv, dropout_seed=4)
    per = Net.unflatten(net.layers, flat)
    p0 = [per[a:b] for a, b in bounds]
    ra = Pl.run_versioned(sa, p0, data, hp)
    rb = Pl.run_clocked(sb, p0, data, hp)
    assert ra.losses == rb.losses
    # the hybrid run with n_p = 0 (non-pipelined) draws the same masks as textbook SGD
    sc, _ = oracle_stages(net, ppv, dropout_seed=4)
    rc = Pl.run_clocked(sc, p0, data, hp, n_p=0)
    sd, _ = oracle_stages(net, (), dropout_seed=4)
    rd = Pl.run_sgd(sd[0], per, data, hp)
    assert rc.losses == rd.losses
    # dropout changes the trajectory (the masks are not all ones)
    se, _ = oracle_stages(W.tiny_cnn(hw=8), (), dropout_seed=4)
    re_ = Pl.run_sgd(se[0], per, data, hp)
    assert abs(re_.losses[0] - rd.losses[0]) > 1e-6
