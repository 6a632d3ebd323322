"""Diagnostic (GPU): momentum-buffer parity step by step on the tiny ResNet (seed 21 case of
tests/test_gpu_dist.py) -- per-tensor errors of weights and momentum after every step, K=1 and K=2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1912_12675_b200 as pst
import pst_workloads as W
from oracle import network as Net, pipeline as Pl
from tests.parity import hparams, oracle_stages, flat_params

net = W.tiny_resnet(width=16, hw=8, n=1)
n = Net.n_params(net.layers)
for seed in (21, 5):
    for ppv in [(), (3,)]:
        K = len(ppv) + 1
        lr = [0.05, 0.1][-K:] if K == 2 else [0.1]
        flat = W.init_params(net, seed=seed)
        data = W.batches(net.in_shape, 32, 8, seed=seed + 100)
        hp = hparams(lr, K, lr[-1], 0.9, 1e-4)
        pipe = pst.Pipeline(net, flat, ppv, 32, lr, lr[-1], momentum=0.9, weight_decay=1e-4)
        for i, (x, y) in enumerate(data):
            pipe.step(x, y)
        pipe.flush()
        st = pipe.weights(pst.W_PARAMS | pst.W_MOMENTUM)
        stages, bounds = oracle_stages(net, ppv)
        per = Net.unflatten(net.layers, flat)
        ref = Pl.run_clocked(stages, [per[a:b] for a, b in bounds], data, hp)
        gw, gv = Net.unflatten(net.layers, st[:n]), Net.unflatten(net.layers, st[n:2 * n])
        rw, rv = ref.params, ref.momentum
        rw = [d for s_ in rw for d in s_]
        rv = [d for s_ in rv for d in s_]
        print("seed", seed, "ppv", ppv, "losses gpu", np.round(pipe.losses(0, 8), 5).tolist())
        print("                  oracle", np.round(ref.losses, 5).tolist())
        for li in range(len(net.layers)):
            for k in rw[li]:
                ew = np.abs(gw[li][k] - rw[li][k]).max() / max(np.abs(rw[li][k]).max(), 1e-12)
                ev = np.abs(gv[li][k] - rv[li][k]).max() / max(np.abs(rv[li][k]).max(), 1e-12)
                print("   layer%d.%-5s w %.2e  v %.2e  |v| %.3e" % (li + 1, k, ew, ev, np.abs(rv[li][k]).max()))
        pipe.close()
