"""Shared helpers for GPU-vs-oracle parity tests (tests only).

Tolerances are BASELINE.json north_star's, with the reading AMB-21:
  weights: per parameter tensor ||W_gpu - W_ref||_inf / max(||W_ref||_inf, 1e-12) <= 2e-3
  losses:  |l_gpu - l_ref| <= 1e-2 * max(1, |l_ref|)
"""
import numpy as np

from oracle import network as Net
from oracle import pipeline as Pl

W_TOL = 2e-3
L_TOL = 1e-2


def oracle_stages(net, ppv):
    bounds = Net.partition(net.layers, ppv)
    stages = [Net.CNNStage(net.layers[a:b], first_stage=(s == 0)) for s, (a, b) in enumerate(bounds)]
    return stages, bounds


def oracle_run(net, flat, ppv, data, hp, n_p=None, snapshot=False):
    stages, bounds = oracle_stages(net, ppv)
    per_layer = Net.unflatten(net.layers, flat)
    res = Pl.run_clocked(stages, [per_layer[a:b] for a, b in bounds], data, hp, n_p=n_p, snapshot=snapshot)
    return res


def flat_params(net, per_stage):
    return Net.flatten(net.layers, [d for st in per_stage for d in st])


def tensor_errors(net, got_flat, ref_flat):
    """max over parameter tensors of the relative inf-norm error, and the worst tensor's name."""
    g = Net.unflatten(net.layers, got_flat)
    r = Net.unflatten(net.layers, ref_flat)
    worst, where = 0.0, None
    for i, (dg, dr) in enumerate(zip(g, r)):
        for k in dr:
            e = float(np.abs(dg[k] - dr[k]).max() / max(np.abs(dr[k]).max(), 1e-12))
            if e > worst:
                worst, where = e, f"layer{i + 1}.{k}"
    return worst, where


def loss_errors(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))))


def hparams(cfg_lr, K, lr_np, momentum, wd, milestones=(), gamma=0.1, spe=1 << 62):
    return Pl.HParams(lr_pipelined=list(cfg_lr), lr_nonpipelined=lr_np, momentum=momentum,
                      weight_decay=wd, milestones=tuple(milestones), gamma=gamma, steps_per_epoch=spe)
