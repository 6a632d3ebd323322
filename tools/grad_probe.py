"""Diagnostic: per-tensor first-update gradient error, GPU vs oracle (K=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import pst_workloads as W
import paper_1912_12675_b200 as p
from oracle import network as Net
from tests.parity import oracle_run, flat_params, hparams

def probe(name, net, B, lr=1.0):
    flat = W.init_params(net, seed=5)
    data = W.batches(net.in_shape, B, 1, seed=105)
    hp = hparams([lr], 1, lr, 0.0, 0.0)
    ref = oracle_run(net, flat, (), data, hp)
    pipe = p.Pipeline(net, flat, (), B, [lr], lr, momentum=0.0, weight_decay=0.0)
    pipe.step(*data[0]); pipe.flush()
    g_gpu = Net.unflatten(net.layers, (flat.astype(np.float64) - pipe.weights()) / lr)
    g_ref = Net.unflatten(net.layers, (flat.astype(np.float64) - flat_params(net, ref.params)) / lr)
    print(p.build_info().split()[2], name)
    for i, (a, b) in enumerate(zip(g_gpu, g_ref)):
        for k in b:
            d = np.abs(a[k] - b[k]).max(); m = np.abs(b[k]).max()
            print(f"   layer{i+1}.{k:5s} max|g|={m:.3e} max|err|={d:.3e} rel={d/max(m,1e-30):.2e}  sum(g)={b[k].sum():.3e} gpu={a[k].sum():.3e}")
    pipe.close()

probe("tiny_resnet", W.tiny_resnet(width=16, hw=8, n=1), 32)
