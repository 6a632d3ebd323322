#!/usr/bin/env python3
"""The float32-emulated oracle (tests/emulation.py) against the exact oracle on the tiny test ResNet
(CPU; readings AMB-21e/f).  Some partitions jump by ~1e-3 per tensor where most stay at ~1e-7: a ReLU
pre-activation within float32 rounding of 0 takes the other side in the emulation and moves a whole
pixel's gradient contribution (ReLU'(0) = 0, AMB-18).  The same jumps appear on the GPU for other
partitions (gpurun_out probes, DESIGN.md AMB-21f): a property of the arithmetic, not of either side.

    python tools/flip_probe.py > profiles/r2_flip_probe.txt
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import pst_workloads as W
from tests.parity import flat_params, hparams, oracle_run, split_errors, stage_errors

net = W.tiny_resnet(width=16, hw=8, n=2)
for ppv in [(1, 2, 3, 6), (3, 6), (3, 5), (2, 4, 6, 8), (6,), (), (1,)]:
    for lr0 in (0.05, 0.005):
        K = len(ppv) + 1
        lr = [lr0] * (K - 1) + [2 * lr0]
        flat = W.init_params(net, seed=5)
        data = W.batches(net.in_shape, 32, 10, seed=105)
        hp = hparams(lr, K, lr[-1], 0.9, 1e-4)
        ref = oracle_run(net, flat, ppv, data, hp)
        emu = oracle_run(net, flat, ppv, data, hp, emu=True)
        e = split_errors(net, ppv, flat_params(net, emu.params), flat_params(net, ref.params), True)
        mv = stage_errors(net, ppv, flat_params(net, emu.momentum), flat_params(net, ref.momentum))
        print("ppv %-14s lr %-6g emulated-vs-exact: W/gamma per tensor %.2e (%s), beta per stage %.2e, "
              "momentum per stage %.2e" % (ppv, lr0, e["tensor"][1], e["tensor"][3], e["beta"][1], mv[0]), flush=True)
