"""Diagnostic (GPU): mid-block PPVs of a two-block-per-group tiny ResNet in local mode, concurrent vs
serialised stages (pst_stage_timing), against Oracle B.  Prints the split weight error per case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1912_12675_b200 as pst
import pst_workloads as W
from oracle import network as Net
from tests.parity import hparams, oracle_run, flat_params, split_errors

net = W.tiny_resnet(width=16, hw=8, n=2)
PPVS = [tuple(int(v) for v in a.split(',')) if a else () for a in sys.argv[1:]] or [(1, 2, 3, 6), (3, 6), (2, 3)]
for ppv in PPVS:
    K = len(ppv) + 1
    lr = [0.05] * (K - 1) + [0.1]
    flat = W.init_params(net, seed=5)
    data = W.batches(net.in_shape, 32, 10, seed=105)
    ref = oracle_run(net, flat, ppv, data, hparams(lr, K, lr[-1], 0.9, 1e-4))
    for serial in (False,):
        pipe = pst.Pipeline(net, flat, ppv, 32, lr, lr[-1], momentum=0.9, weight_decay=1e-4)
        if serial:
            pipe.stage_timing(True)
        for x, y in data:
            pipe.step(x, y)
        pipe.flush()
        e = split_errors(net, ppv, pipe.weights(), flat_params(net, ref.params), True)
        n_ = len(flat)
        st_ = pipe.weights(pst.W_PARAMS | pst.W_MOMENTUM)
        from tests.parity import stage_errors
        mv = stage_errors(net, ppv, st_[n_:], flat_params(net, ref.momentum))
        print(ppv, "W/gamma per tensor %.2e at %s; beta per stage %.2e; momentum per stage %.2e" % (
            e["tensor"][1], e["tensor"][3], e["beta"][1], mv[0]), flush=True)
        pipe.close()
