"""Diagnostic (CPU): the oracle with the GPU's storage roundings emulated.

Rounds every tensor the CUDA path stores in its compute dtype (activations,
gradients, weight shadows) and keeps float32-like accumulation elsewhere (done
in float64 here).  If GPU-vs-oracle errors match emulated-vs-oracle errors,
the discrepancy is arithmetic precision, not a bug."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import pst_workloads as W
from oracle import layers as Lx, network as Net, pipeline as Pl
from tests.parity import flat_params, tensor_errors, loss_errors, hparams, stage_errors

MODES = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": None, "tf32": "tf32", "bf16x2": "bf16x2", "tf32x3": "tf32x3"}
DT = MODES[sys.argv[1] if __name__ == "__main__" and len(sys.argv) > 1 else "tf32x3"]


def set_mode(name):
    """Select the emulated storage/product precision (importers; the CLI takes it as argv[1])."""
    global DT
    DT = MODES[name]

def _b(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float64)).to(torch.bfloat16).double().numpy()

def _trunc_tf32(a32):
    return (a32.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)

def _rnd_tf32(a32):
    return ((a32.view(np.uint32) + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)

def R(a):
    if DT == "tf32x3":
        a32 = np.asarray(a, dtype=np.float32)
        hi = _trunc_tf32(a32)
        lo = _rnd_tf32((a32 - hi).astype(np.float32))
        return hi.astype(np.float64) + lo.astype(np.float64)
    if DT == "bf16x2":
        a = np.asarray(a, dtype=np.float32).astype(np.float64)
        hi = _b(a)
        return hi + _b(a - hi)
    if DT is None:
        return np.asarray(a, dtype=np.float32).astype(np.float64)
    if DT == "tf32":
        a32 = np.asarray(a, dtype=np.float32).view(np.uint32)
        a32 = (a32 + np.uint32(0x1000)) & np.uint32(0xFFFFE000)
        return a32.view(np.float32).astype(np.float64)
    return torch.from_numpy(np.asarray(a, dtype=np.float64)).to(DT).double().numpy()

class EmuStage(Net.CNNStage):
    def forward(self, params, x, mb=0):
        a = R(x)
        caches, block_in = [], None
        for L, P, S in zip(self.layers, params, self.state):
            c = {"x": a}
            if L.block_begin: block_in = a
            Wr = R(P["W"])
            y = Lx.conv2d_forward(a, Wr, P.get("b"), L.stride, L.pad) if L.kind == "conv" else Lx.fc_forward(a, Wr, P.get("b"))
            if L.bn:
                y = R(y)
                c["y"] = y
                y, c["bn"] = Lx.bn_train_forward(y, P["gamma"], P["beta"], self.bn_eps)
                xh, inv, mean, var, M = c["bn"]
                S["run_mean"], S["run_var"] = Lx.bn_running_update(S["run_mean"], S["run_var"], mean, var, M, self.bn_momentum)
            if L.residual:
                c["block_in_shape"] = block_in.shape
                y = y + Lx.shortcut_forward(block_in, y.shape)
            if L.relu: y, c["mask"] = Lx.relu_forward(y)
            last = L is self.layers[-1] and L.kind == "fc" and not L.relu
            y = y if last else R(y)
            if L.pool == "max2":
                c["pool_in_shape"] = y.shape; y, c["arg"] = Lx.maxpool2_forward(y)
            elif L.pool == "gap":
                c["pool_in_shape"] = y.shape; y = R(Lx.gap_forward(y))
            caches.append(c); a = y
        return a, caches

    def backward(self, params, caches, g_out):
        g = np.asarray(g_out, dtype=np.float64)
        grads = [None] * len(self.layers); gsc = None
        for idx in range(len(self.layers) - 1, -1, -1):
            L, P, c = self.layers[idx], params[idx], caches[idx]
            if L.pool == "max2": g = Lx.maxpool2_backward(g, c["arg"], c["pool_in_shape"])
            elif L.pool == "gap": g = Lx.gap_backward(g, c["pool_in_shape"])
            if L.relu: g = Lx.relu_backward(g, c["mask"])
            g = R(g)
            if L.residual: gsc = Lx.shortcut_backward(g, c["block_in_shape"])
            gr = {}
            if L.bn:
                g, gr["gamma"], gr["beta"] = Lx.bn_train_backward(g, c["bn"], P["gamma"])
                g = R(g)
            need = not (self.first_stage and idx == 0)
            Wr = R(P["W"])
            if L.kind == "conv": gx, gW, gb = Lx.conv2d_backward(c["x"], Wr, g, L.stride, L.pad, need)
            else: gx, gW, gb = Lx.fc_backward(c["x"], Wr, g, need)
            gr["W"] = gW
            if L.bias: gr["b"] = gb
            if gx is not None:
                if L.block_begin: gx = gx + gsc
                gx = R(gx)
            grads[idx] = gr; g = gx
        return g, grads

def run(net, ppv, B, N, lr, wd, emu):
    K = len(ppv) + 1
    flat = W.init_params(net, seed=5)
    data = W.batches(net.in_shape, B, N, seed=105)
    bounds = Net.partition(net.layers, ppv)
    cls = EmuStage if emu else Net.CNNStage
    st = [cls(net.layers[a:b], first_stage=(s == 0)) for s, (a, b) in enumerate(bounds)]
    pl = Net.unflatten(net.layers, flat)
    return Pl.run_clocked(st, [pl[a:b] for a, b in bounds], data, hparams(lr, K, lr[-1], 0.9, wd), snapshot=True)

def main():
    CASES = [("tiny_cnn", W.tiny_cnn(hw=8), (), 32, 8, [0.05], 5e-4),
                                          ("tiny_resnet", W.tiny_resnet(width=16, hw=8, n=1), (), 32, 8, [0.1], 1e-4),
                                          ("lenet5", W.lenet5(), (1,), 64, 10, [0.01, 0.01], 5e-4)]
    if len(sys.argv) > 2 and sys.argv[2] == "deep":   # the deep-BN cases judged per stage (AMB-21b)
        CASES = [("resnet20_k1", W.resnet_cifar(20), (), 32, 8, [0.01], 1e-4),
                 ("resnet110_k2", W.resnet_cifar(110), (47,), 32, 5, [0.01, 0.01], 1e-4)]
    if len(sys.argv) > 2 and sys.argv[2] == "big":
        CASES = [("lenet5_k2_20", W.lenet5(), (1,), 64, 20, [0.01, 0.01], 5e-4),
                 ("resnet20_k2", W.resnet_cifar(20), (7,), 128, 12, [0.001, 0.1], 1e-4)]
    for name, net, ppv, B, N, lr, wd in CASES:
        ref = run(net, ppv, B, N, lr, wd, False)
        emu = run(net, ppv, B, N, lr, wd, True)
        errs = [tensor_errors(net, flat_params(net, e), flat_params(net, r)) for e, r in zip(emu.snapshots, ref.snapshots)]
        serrs = [stage_errors(net, ppv, flat_params(net, e), flat_params(net, r))[0] for e, r in zip(emu.snapshots, ref.snapshots)]
        print(sys.argv[1:], name, "loss err %.2e" % loss_errors(emu.losses, ref.losses), " ".join("%.1e(%s)" % e for e in errs[:N]),
              "| per stage max %.1e" % max(serrs), flush=True)


if __name__ == "__main__":
    main()
