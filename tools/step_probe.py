"""Diagnostic (GPU): per-step weight error by stage, tiny ResNet seed 21 PPV (3,) (and others)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1912_12675_b200 as pst
import pst_workloads as W
from oracle import network as Net
from tests.parity import hparams, oracle_run, flat_params, stage_errors

cases = [(1, 21, (3,), 32, 8), (1, 21, (1,), 32, 8), (1, 21, (3,), 16, 8), (2, 5, (7,), 32, 10)]
for n, seed, ppv, B, N in cases:
    net = W.tiny_resnet(width=16, hw=8, n=n)
    K = len(ppv) + 1
    lr = [0.05] * (K - 1) + [0.1]
    flat = W.init_params(net, seed=seed)
    data = W.batches(net.in_shape, B, N, seed=seed + 100)
    ref = oracle_run(net, flat, ppv, data, hparams(lr, K, lr[-1], 0.9, 1e-4), snapshot=True)
    pipe = pst.Pipeline(net, flat, ppv, B, lr, lr[-1], momentum=0.9, weight_decay=1e-4)
    bounds = Net.partition(net.layers, ppv)
    print("net n=%d seed %d ppv %s B %d" % (n, seed, ppv, B))
    for t, (x, y) in enumerate(data):
        pipe.step(x, y)
        got = pipe.weights()
        want = flat_params(net, ref.snapshots[t])
        per = []
        for s, (a, b) in enumerate(bounds):
            g = Net.unflatten(net.layers, got)[a:b]; r = Net.unflatten(net.layers, want)[a:b]
            per.append(max(float(np.abs(g[i][k] - r[i][k]).max() / max(np.abs(r[i][k]).max(), 1e-12)) for i in range(b - a) for k in r[i] if k != "beta"))
        print("  step %d  per-stage W/gamma err %s  versions %s" % (t, ["%.1e" % e for e in per], pipe.versions().tolist()), flush=True)
    pipe.close()
