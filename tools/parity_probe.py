"""Diagnostic: per-step GPU-vs-oracle errors for small configs (prints, never asserts)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import pst_workloads as W
import paper_1912_12675_b200 as p
from tests.parity import oracle_run, flat_params, tensor_errors, loss_errors, hparams

def probe(name, net, ppv, B, N, lr, wd=1e-4, mom=0.9):
    K = len(ppv) + 1
    flat = W.init_params(net, seed=5)
    data = W.batches(net.in_shape, B, N, seed=105)
    hp = hparams(lr, K, lr[-1], mom, wd)
    ref = oracle_run(net, flat, ppv, data, hp, snapshot=True)
    pipe = p.Pipeline(net, flat, ppv, B, lr, lr[-1], momentum=mom, weight_decay=wd)
    errs = []
    for i, (x, y) in enumerate(data):
        pipe.step(x, y)
        errs.append(tensor_errors(net, pipe.weights(), flat_params(net, ref.snapshots[i])))
    pipe.flush()
    le = loss_errors(pipe.losses(0, N), ref.losses)
    print(f"{p.build_info().split()[2]} {name} K={K}: loss err {le:.2e}; per-step worst W err:",
          " ".join(f"{e:.1e}({w})" for e, w in errs))
    print("   gpu losses", np.round(pipe.losses(0, N), 4).tolist())
    print("   ref losses", np.round(ref.losses, 4).tolist())
    pipe.close()

probe("tiny_cnn", W.tiny_cnn(hw=8), (), 32, 8, [0.05], wd=5e-4)
probe("tiny_cnn_lr0", W.tiny_cnn(hw=8), (), 32, 4, [0.0], wd=0.0)
probe("tiny_resnet", W.tiny_resnet(width=16, hw=8, n=1), (), 32, 8, [0.1])
probe("lenet5", W.lenet5(), (1,), 64, 10, [0.01, 0.01], wd=5e-4)
