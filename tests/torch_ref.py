"""Independent textbook reference for NON-pipelined training (tests only).

Builds the LayerSpec network with PyTorch-CPU float64 functional ops and
trains it with torch autograd + torch.optim.SGD.  This shares no code with
`oracle/` and pins its K=1 (non-pipelined, §2) special case.
"""
import numpy as np
import torch
import torch.nn.functional as F


def _shapes(L):
    out = [("W", (L.cout, L.cin, L.k, L.k) if L.kind == "conv" else (L.cout, L.cin))]
    if L.bias:
        out.append(("b", (L.cout,)))
    if L.bn:
        out += [("gamma", (L.cout,)), ("beta", (L.cout,))]
    return out


def _fmix32(h):
    h &= 0xFFFFFFFF
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & 0xFFFFFFFF
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & 0xFFFFFFFF
    h ^= h >> 16
    return h


def dropout_mask_py(seed, mb, layer, shape, p):
    """The counter-based dropout generator of DESIGN.md (reading AMB-16b), written independently of
    oracle/ with Python integers: key = fmix32(seed ^ fmix32(mb*0x9E3779B9 + (layer+1)*0x632BE5AB)),
    keep element e iff fmix32(e ^ key) >= floor(float32(p) * 2^32); kept elements scale by 1/(1-p)."""
    p32 = float(np.float32(p))
    thr = min(2 ** 32 - 1, int(np.floor(p32 * 2.0 ** 32)))
    key = _fmix32((seed & 0xFFFFFFFF) ^ _fmix32((mb * 0x9E3779B9 + (layer + 1) * 0x632BE5AB) & 0xFFFFFFFF))
    n = int(np.prod(shape))
    keep = [1.0 if _fmix32((e & 0xFFFFFFFF) ^ key) >= thr else 0.0 for e in range(n)]
    return torch.tensor(keep, dtype=torch.float64).reshape(shape) / (1.0 - p32)


def train_sgd(net, flat_params, batches, lr, momentum, weight_decay, lr_fn=None, dropout_seed=0):
    flat = torch.from_numpy(np.asarray(flat_params, dtype=np.float64))
    params, off = [], 0
    for L in net.layers:
        d = {}
        for name, shp in _shapes(L):
            n = int(np.prod(shp))
            d[name] = torch.nn.Parameter(flat[off:off + n].reshape(shp).clone())
            off += n
        params.append(d)
    running = [(torch.zeros(L.cout, dtype=torch.float64), torch.ones(L.cout, dtype=torch.float64)) if L.bn else None
               for L in net.layers]
    allp = [p for d in params for p in d.values()]
    opt = torch.optim.SGD(allp, lr=lr, momentum=momentum, weight_decay=weight_decay)
    losses = []
    for i, (x, y) in enumerate(batches):
        if lr_fn is not None:
            for g in opt.param_groups:
                g["lr"] = lr_fn(i)
        a = torch.from_numpy(np.asarray(x, dtype=np.float64))
        block_in = None
        for li, (L, P, R) in enumerate(zip(net.layers, params, running)):
            if L.block_begin:
                block_in = a
            if L.kind == "conv":
                a = F.conv2d(a, P["W"], P.get("b"), stride=L.stride, padding=L.pad)
            else:
                a = F.linear(a.flatten(1), P["W"], P.get("b"))
            if L.bn:
                a = F.batch_norm(a, R[0], R[1], P["gamma"], P["beta"], training=True, momentum=0.1, eps=1e-5)
            if L.residual:
                if block_in.shape == a.shape:
                    sc = block_in
                else:
                    p = (a.shape[1] - block_in.shape[1]) // 2
                    sc = F.pad(block_in[:, :, ::2, ::2], (0, 0, 0, 0, p, p))
                a = a + sc
            if L.relu:
                a = F.relu(a)
            if getattr(L, "dropout", 0.0) > 0.0:
                a = a * dropout_mask_py(dropout_seed, i, li, tuple(a.shape), L.dropout)
            if L.pool == "max2":
                a = F.max_pool2d(a, 2, 2)
            elif L.pool == "gap":
                a = a.mean(dim=(2, 3))
        loss = F.cross_entropy(a, torch.from_numpy(np.asarray(y)).long())
        losses.append(loss.item())
        opt.zero_grad()
        loss.backward()
        opt.step()
    flat_out = torch.cat([p.detach().reshape(-1) for d in params for p in d.values()]).numpy()
    return losses, flat_out
