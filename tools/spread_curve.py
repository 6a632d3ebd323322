#!/usr/bin/env python3
"""The oracle's own sensitivity along a trajectory (CPU; reading AMB-21c/d).

Runs Oracle B twice -- from the seeded initial weights and from the same weights perturbed by 1e-7
relative (one float32 rounding) -- and prints, after every mini-batch, the loss difference and the
per-tensor weight ratio (W / gamma per tensor, beta per stage; tests/parity.py split measure).
Where this spread exceeds a tenth of the tolerance no float32 implementation can be held to the
exact trajectory step for step; the GPU parity tests switch to segment parity there.

    python tools/spread_curve.py resnet110 2 32 100 > profiles/r2_spread_curve_resnet110_k2_b32.jsonl
    python tools/spread_curve.py resnet110 2 32 100 "" 0.001,0.01   # warm-up rates (lr/10)
"""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import pst_workloads as W
from tests.parity import (flat_params, hparams, loss_errors, oracle_run, perturbed, split_errors, W_TOL, L_TOL)


def main():
    name, K, B, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    ppv = tuple(int(p) for p in sys.argv[5].split(",")) if len(sys.argv) > 5 and sys.argv[5] else None
    lr_over = [float(v) for v in sys.argv[6].split(",")] if len(sys.argv) > 6 else None
    cfg = W.CONFIGS[name]
    net = cfg.netspec()
    ppv = cfg.ppv[K] if ppv is None else ppv
    lr = cfg.lr_vector(K) if lr_over is None else lr_over
    flat = W.init_params(net, seed=5)
    data = W.batches(net.in_shape, B, N, seed=105)
    hp = hparams(lr, K, lr[-1], cfg.momentum, cfg.weight_decay, cfg.milestones, 0.1, cfg.steps_per_epoch)
    ref = oracle_run(net, flat, ppv, data, hp, snapshot=True)
    refp = oracle_run(net, perturbed(flat), ppv, data, hp, snapshot=True)
    print(json.dumps({"config": name, "K": K, "ppv": list(ppv), "B": B, "N": N, "lr": lr,
                      "note": "oracle vs oracle from initial weights perturbed by 1e-7 relative"}), flush=True)
    first_over = None
    for t in range(len(ref.snapshots)):
        sw = split_errors(net, ppv, flat_params(net, refp.snapshots[t]), flat_params(net, ref.snapshots[t]), True)
        done = [i for i in range(N) if i <= t - (K - 1)]          # losses computed by step t
        le = loss_errors([refp.losses[i] for i in done], [ref.losses[i] for i in done]) if done else 0.0
        rec = {"step": t, "weights_tensor_spread": sw["tensor"][1], "where": sw["tensor"][3],
               "beta_stage_spread": sw["beta"][1], "loss_spread_so_far": le,
               "loss": ref.losses[done[-1]] if done else None}
        if first_over is None and (sw["tensor"][1] > W_TOL / 10 or le > L_TOL / 10):
            first_over = t
        print(json.dumps(rec), flush=True)
    print(json.dumps({"first_step_spread_over_tol/10": first_over,
                      "final_loss_spread": loss_errors(refp.losses, ref.losses)}), flush=True)


if __name__ == "__main__":
    main()
