"""Shared helpers for GPU-vs-oracle parity tests (tests only).

Tolerances are BASELINE.json north_star's, with the readings of DESIGN.md section 3:
  weights (AMB-21, per tensor):  ||W_gpu - W_ref||_inf / max(||W_ref||_inf, 1e-12) <= 2e-3 for every
           parameter tensor -- applied where it is well posed (nets without BatchNorm, small nets);
  weights (AMB-21b, per stage):  the same ratio over each stage's whole parameter vector -- for
           deep BatchNorm nets, whose BN-shift gradients are sums with heavy cancellation: a 1e-7
           relative perturbation of the initial weights moves the fp64 oracle's own beta tensors by
           1e-2..3e-2 relative after one step (tests/test_oracle_conditioning.py), so no fp32
           implementation can meet the per-tensor reading there;
  losses:  |l_gpu - l_ref| <= 1e-2 * max(1, |l_ref|)
"""
import numpy as np

from oracle import network as Net
from oracle import pipeline as Pl

W_TOL = 2e-3
L_TOL = 1e-2


def oracle_stages(net, ppv):
    bounds = Net.partition(net.layers, ppv)
    stages = [Net.CNNStage(net.layers[a:b], first_stage=(s == 0)) for s, (a, b) in enumerate(bounds)]
    return stages, bounds


def oracle_run(net, flat, ppv, data, hp, n_p=None, snapshot=False):
    stages, bounds = oracle_stages(net, ppv)
    per_layer = Net.unflatten(net.layers, flat)
    res = Pl.run_clocked(stages, [per_layer[a:b] for a, b in bounds], data, hp, n_p=n_p, snapshot=snapshot)
    return res


def flat_params(net, per_stage):
    return Net.flatten(net.layers, [d for st in per_stage for d in st])


def tensor_errors(net, got_flat, ref_flat):
    """max over parameter tensors of the relative inf-norm error, and the worst tensor's name."""
    g = Net.unflatten(net.layers, got_flat)
    r = Net.unflatten(net.layers, ref_flat)
    worst, where = 0.0, None
    for i, (dg, dr) in enumerate(zip(g, r)):
        for k in dr:
            e = float(np.abs(dg[k] - dr[k]).max() / max(np.abs(dr[k]).max(), 1e-12))
            if e > worst:
                worst, where = e, f"layer{i + 1}.{k}"
    return worst, where


def stage_errors(net, ppv, got_flat, ref_flat):
    """max over stages of ||W_gpu - W_ref||_inf / ||W_ref||_inf over the stage's parameter vector
    (reading AMB-21b), and the worst stage."""
    bounds = Net.partition(net.layers, ppv)
    g = Net.unflatten(net.layers, got_flat)
    r = Net.unflatten(net.layers, ref_flat)
    worst, where = 0.0, None
    for s, (a, b) in enumerate(bounds):
        num = max(float(np.abs(g[i][k] - r[i][k]).max()) for i in range(a, b) for k in r[i])
        den = max(float(np.abs(r[i][k]).max()) for i in range(a, b) for k in r[i])
        e = num / max(den, 1e-12)
        if e > worst:
            worst, where = e, f"stage{s}"
    return worst, where


def loss_errors(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))))


def hparams(cfg_lr, K, lr_np, momentum, wd, milestones=(), gamma=0.1, spe=1 << 62):
    return Pl.HParams(lr_pipelined=list(cfg_lr), lr_nonpipelined=lr_np, momentum=momentum,
                      weight_decay=wd, milestones=tuple(milestones), gamma=gamma, steps_per_epoch=spe)


def run_both(pst, net, ppv, B, N, lr, lr_np=None, mom=0.9, wd=1e-4, n_p=None, spe=1 << 62,
             milestones=(), per_step=True, seed=5, check=None, stage_level=False, solver_kw=None):
    """Train the same seeded mini-batches through libpst (all stages on cuda:0, local mode)
    and through Oracle B; compare the weights after every compared step and after the
    drain, and the loss of every mini-batch.  `check`: None = every step (if per_step),
    else the global step indices t after which the weights are compared (big nets).
    Returns (worst weight error, where) per tensor (AMB-21), or per stage if stage_level (AMB-21b),
    the loss error, the stage versions and the oracle's result."""
    import pst_workloads as W
    K = len(ppv) + 1
    flat = W.init_params(net, seed=seed)
    data = W.batches(net.in_shape, B, N, seed=seed + 100)
    lr_np = lr[-1] if lr_np is None else lr_np
    hp = hparams(lr, K, lr_np, mom, wd, milestones, 0.1, spe)
    skw = dict(solver_kw or {})        # solver / nesterov / lr_policy / inv_gamma / inv_power
    for k, v in skw.items():
        setattr(hp, k, v)
    snap = (True if check is None else set(check)) if per_step else False
    ref = oracle_run(net, flat, ppv, data, hp, n_p=n_p, snapshot=snap)
    pipe = pst.Pipeline(net, flat, ppv, B, lr, lr_np, momentum=mom, weight_decay=wd, milestones=milestones,
                        steps_per_epoch=spe, **skw)
    if n_p is not None:
        assert n_p % spe == 0
        pipe.set_hybrid(n_p // spe)
    worst = (0.0, None)
    worst_stage = (0.0, None)
    compared = 0
    for x, y in data:
        pipe.step(x, y)
        if per_step:
            # a hybrid switch inserts the drain steps before this mini-batch's step
            steps, _ = pipe.progress()
            if check is None or (steps - 1) in ref.snapshots:
                got, want = pipe.weights(), flat_params(net, ref.snapshots[steps - 1])
                worst = max(worst, tensor_errors(net, got, want), key=lambda z: z[0])
                worst_stage = max(worst_stage, stage_errors(net, ppv, got, want), key=lambda z: z[0])
                compared += 1
    pipe.flush()
    got, want = pipe.weights(), flat_params(net, ref.params)
    worst = max(worst, tensor_errors(net, got, want), key=lambda z: z[0])
    worst_stage = max(worst_stage, stage_errors(net, ppv, got, want), key=lambda z: z[0])
    lerr = loss_errors(pipe.losses(0, N), ref.losses)
    vers = pipe.versions()
    pipe.close()
    if per_step and check is not None:
        assert compared == len(set(check)), (compared, sorted(check))
    assert np.all(np.isfinite(ref.losses)), "the oracle's trajectory diverged: pick a smaller lr"
    if stage_level:
        return worst_stage, lerr, vers, ref
    return worst, lerr, vers, ref


def run_segments(pst, net, ppv, B, seg_lens, lr, lr_np=None, mom=0.9, wd=1e-4, seed=5):
    """Segment ("shadowing") parity for trajectories that are chaotic (reading AMB-21c).

    The GPU trains sum(seg_lens) mini-batches; after each segment the pipe is drained
    (pst_flush) and the oracle (Oracle B) is restarted from the GPU's drained state --
    its weights and momentum buffers -- for the next segment's mini-batches, with a fresh
    pipeline fill exactly like the GPU's.  Within a segment every mini-batch's loss and, after
    the drain, every stage's weights are compared.  Returns (worst stage error, where), the
    worst loss error and the oracle's losses (all segments)."""
    import pst_workloads as W
    K = len(ppv) + 1
    flat = W.init_params(net, seed=seed)
    N = int(sum(seg_lens))
    data = W.batches(net.in_shape, B, N, seed=seed + 100)
    lr_np = lr[-1] if lr_np is None else lr_np
    hp = hparams(lr, K, lr_np, mom, wd)
    stages, bounds = oracle_stages(net, ppv)
    pipe = pst.Pipeline(net, flat, ppv, B, lr, lr_np, momentum=mom, weight_decay=wd)
    n = Net.n_params(net.layers)
    w_state = flat.astype(np.float64)
    v_state = np.zeros_like(w_state)
    worst, lworst, losses = (0.0, None), 0.0, []
    i0 = 0
    for M in seg_lens:
        seg = data[i0:i0 + M]
        pw, pv = Net.unflatten(net.layers, w_state), Net.unflatten(net.layers, v_state)
        ref = Pl.run_clocked(stages, [pw[a:b] for a, b in bounds], seg, hp,
                             mom0=[pv[a:b] for a, b in bounds])
        for x, y in seg:
            pipe.step(x, y)
        pipe.flush()
        state = pipe.weights(pst.W_PARAMS | pst.W_MOMENTUM).astype(np.float64)
        w_state, v_state = state[:n], state[n:2 * n]
        e = stage_errors(net, ppv, w_state, flat_params(net, ref.params))
        worst = max(worst, (e[0], f"segment@{i0}:{e[1]}"), key=lambda z: z[0])
        lworst = max(lworst, loss_errors(pipe.losses(i0, M), ref.losses))
        losses += list(ref.losses)
        assert np.all(np.isfinite(ref.losses)), "the oracle's trajectory diverged: pick a smaller lr"
        i0 += M
    pipe.close()
    return worst, lworst, losses
