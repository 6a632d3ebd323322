"""Solver variants of the paper's Caffe-simulated runs:
Caffe SGD form, Nesterov momentum (PyTorch and Caffe forms), Caffe "inv" learning-rate policy.
Pinned against torch.optim.SGD (library routine, fp64) and closed-form identities."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import layers as Lx
from oracle import pipeline as Pl


def _torch_traj(w0, grads, lr, mu, wd, nesterov):
    p = torch.nn.Parameter(torch.tensor(w0, dtype=torch.float64))
    opt = torch.optim.SGD([p], lr=lr, momentum=mu, weight_decay=wd, nesterov=nesterov)
    out = []
    for g in grads:
        opt.zero_grad()
        p.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
        out.append(p.detach().numpy().copy())
    return out


def _rand(seed, n=5, shape=(7, 3)):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape), [rng.standard_normal(shape) for _ in range(n)]


def test_torch_nesterov_matches_torch_optim():
    w0, grads = _rand(1)
    ref = _torch_traj(w0, grads, 0.05, 0.9, 1e-3, True)
    w, v = w0.copy(), np.zeros_like(w0)
    for g, r in zip(grads, ref):
        w, v = Lx.sgd_nesterov(w, v, g, 0.05, 0.9, 1e-3)
        np.testing.assert_allclose(w, r, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("nesterov", [False, True])
def test_caffe_form_equals_torch_form_at_constant_lr(nesterov):
    """With a constant rate, Caffe's V equals lr times PyTorch's v and the weight sequences are
    the same (for plain momentum and for Nesterov) -- so both forms pin to torch.optim.SGD."""
    w0, grads = _rand(2)
    lr = 0.03
    ref = _torch_traj(w0, grads, lr, 0.9, 5e-4, nesterov)
    w, V = w0.copy(), np.zeros_like(w0)
    for g, r in zip(grads, ref):
        w, V = Lx.sgd_caffe(w, V, g, lr, 0.9, 5e-4, nesterov)
        np.testing.assert_allclose(w, r, rtol=1e-12, atol=1e-12)


def test_caffe_and_torch_forms_differ_when_lr_changes():
    """The forms are not equivalent once the rate changes (Caffe folds lr into the history) --
    why the solver is a separate switch (reading AMB-7)."""
    w0, grads = _rand(3, n=2)
    w1, V = Lx.sgd_caffe(w0, np.zeros_like(w0), grads[0], 0.1, 0.9, 0.0)
    w2c, _ = Lx.sgd_caffe(w1, V, grads[1], 0.01, 0.9, 0.0)
    u1, v = Lx.sgd_momentum(w0, np.zeros_like(w0), grads[0], 0.1, 0.9, 0.0)
    w2t, _ = Lx.sgd_momentum(u1, v, grads[1], 0.01, 0.9, 0.0)
    np.testing.assert_allclose(w1, u1)
    assert np.abs(w2c - w2t).max() > 1e-3


def test_inv_policy_closed_form():
    """Caffe "inv" (L284): lr(i) = base (1 + gamma i)^(-power)."""
    hp = Pl.HParams(lr_pipelined=[0.01], lr_nonpipelined=0.01, lr_policy="inv", inv_gamma=1e-4, inv_power=0.75)
    assert Pl.learning_rate(hp, 0, 0) == pytest.approx(0.01)
    assert Pl.learning_rate(hp, 0, 10000) == pytest.approx(0.01 * 2 ** -0.75)
    assert Pl.learning_rate(hp, 0, 30000) == pytest.approx(0.01 * 4 ** -0.75)
