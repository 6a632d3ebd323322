"""Conditioning of the parity measure (CPU, oracle only) -- pins reading AMB-21b.

BASELINE.json asks for per-step weights within a max relative error of 2e-3.  Read per parameter
tensor (AMB-21), that is ill-posed for deep BatchNorm networks: the BN shift gradient
dbeta_c = sum over N*H*W of dY (P:L47 applied to BN) is a sum of a near-zero-mean field (the next
BN's backward removes the mean, the conv in between only adds border terms), so it carries heavy
cancellation.  The exact (float64) oracle itself moves by far more than 2e-3 relative on those
tensors when its initial weights move by 1e-7 relative -- the size of one float32 rounding.  Over a
stage's whole parameter vector (AMB-21b) the same perturbation stays at the 1e-7 level, so that
reading separates rounding from error and is the one the deep-net GPU parity tests use.
"""
import numpy as np
import pytest

import pst_workloads as W
from oracle import network as Net
from oracle import pipeline as Pl
from tests.parity import stage_errors, tensor_errors


def _one_step(net, flat, B):
    st = Net.CNNStage(net.layers, first_stage=True)
    hp = Pl.HParams(lr_pipelined=[0.01], lr_nonpipelined=0.01, momentum=0.9, weight_decay=1e-4)
    data = W.batches(net.in_shape, B, 1, seed=105)
    r = Pl.run_sgd(st, Net.unflatten(net.layers, flat), data, hp)
    return Net.flatten(net.layers, r.params[0])


def test_bn_shift_gradient_is_ill_conditioned_per_tensor():
    net = W.nets.by_name("resnet20")
    flat = W.init_params(net, seed=5).astype(np.float64)
    pert = flat * (1 + 1e-7 * np.random.default_rng(0).standard_normal(flat.shape))
    a = _one_step(net, flat, 32)
    b = _one_step(net, pert, 32)
    per_tensor, where = tensor_errors(net, b, a)
    per_stage, _ = stage_errors(net, (), b, a)
    # the exact oracle's own beta tensors move beyond the 2e-3 tolerance ...
    assert per_tensor > 2e-3 and where.endswith("beta"), (per_tensor, where)
    # ... while the stage's parameter vector moves at the perturbation's own scale
    assert per_stage < 1e-5, per_stage


def test_stage_error_measure():
    """stage_errors against a hand-made example: stage 1's vector max |W| = 2, error 0.01."""
    net = W.tiny_cnn(hw=8)
    ppv = (2,)
    flat = W.init_params(net, seed=1).astype(np.float64)
    per = Net.unflatten(net.layers, flat)
    bounds = Net.partition(net.layers, ppv)
    a, b = bounds[1]
    for i in range(a, b):
        for k in per[i]:
            per[i][k] = np.zeros_like(per[i][k])
    k0 = next(iter(per[a]))
    per[a][k0].flat[0] = 2.0
    ref = Net.flatten(net.layers, per)
    got = ref.copy()
    got[np.flatnonzero(ref == 2.0)[0]] += 0.01
    e, where = stage_errors(net, ppv, got, ref)
    assert where == "stage1" and e == pytest.approx(0.005)
