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


def test_caffe_form_two_steps_changing_lr_by_hand():
    """Caffe's documented update (V <- mu V + alpha (g + lambda W); W <- W - V; Nesterov:
    W <- W - ((1 + mu) V_new - mu V_old)) with the rate changing between steps, worked by hand:
    w0 = 1, g = 0.5 then 0.25, mu = 0.9, lambda = 0.1, alpha = 0.1 then 0.01.
      step 1: g' = 0.5 + 0.1*1 = 0.6;          V1 = 0.06;   w1 = 0.94       (Nesterov: 1 - 1.9*0.06 = 0.886)
      step 2: g' = 0.25 + 0.1*0.94 = 0.344;    V2 = 0.054 + 0.00344 = 0.05744;  w2 = 0.88256
              Nesterov: g' = 0.25 + 0.0886 = 0.3386; V2 = 0.054 + 0.003386 = 0.057386;
                        w2 = 0.886 - (1.9*0.057386 - 0.9*0.06) = 0.8309666"""
    w, V = Lx.sgd_caffe(np.float64(1.0), np.float64(0.0), 0.5, 0.1, 0.9, 0.1)
    assert (w, V) == pytest.approx((0.94, 0.06), abs=1e-15)
    w, V = Lx.sgd_caffe(w, V, 0.25, 0.01, 0.9, 0.1)
    assert (w, V) == pytest.approx((0.88256, 0.05744), abs=1e-15)
    w, V = Lx.sgd_caffe(np.float64(1.0), np.float64(0.0), 0.5, 0.1, 0.9, 0.1, nesterov=True)
    assert (w, V) == pytest.approx((0.886, 0.06), abs=1e-15)
    w, V = Lx.sgd_caffe(w, V, 0.25, 0.01, 0.9, 0.1, nesterov=True)
    assert (w, V) == pytest.approx((0.8309666, 0.057386), abs=1e-15)


@pytest.mark.parametrize("spe,milestones,gamma,n_p", [(3, (2, 4), 0.1, None), (1, (1, 3, 5), 0.5, None),
                                                       (4, (2,), 0.2, 12), (2, (1, 6), 0.1, 6)])
def test_learning_rate_matches_torch_multisteplr(spe, milestones, gamma, n_p):
    """oracle.pipeline.learning_rate (reading AMB-8: the rate of the update from mini-batch i is the
    stage's base rate x gamma^(#milestones <= epoch(i)), epoch(i) = i // steps_per_epoch; after the
    hybrid switch at n_p every stage uses the non-pipelined base, reading AMB-10)
    against torch.optim.lr_scheduler.MultiStepLR stepped once per epoch, one optimizer per stage.
    At the switch the schedule restarts from the non-pipelined base as a user would: a fresh
    optimizer + MultiStepLR fast-forwarded to the switch epoch."""
    lrs = [0.001, 0.02, 0.1]
    lr_np = 0.05
    hp = Pl.HParams(lr_pipelined=lrs, lr_nonpipelined=lr_np, milestones=milestones, gamma=gamma,
                    steps_per_epoch=spe)
    N = 30

    def make(base, epochs_done=0):
        p = torch.nn.Parameter(torch.zeros(1, dtype=torch.float64))
        opt = torch.optim.SGD([p], lr=base)
        sch = torch.optim.lr_scheduler.MultiStepLR(opt, milestones=list(milestones), gamma=gamma)
        for _ in range(epochs_done):
            opt.step()
            sch.step()
        return opt, sch

    for s in range(len(lrs)):
        opt, sch = make(lrs[s])
        for i in range(N):
            if n_p is not None and i == n_p:
                assert n_p % spe == 0
                opt, sch = make(lr_np, n_p // spe)
            want = opt.param_groups[0]["lr"]
            assert Pl.learning_rate(hp, s, i, n_p) == pytest.approx(want, rel=1e-12), (s, i)
            opt.step()
            if (i + 1) % spe == 0:
                sch.step()
