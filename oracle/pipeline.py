"""Pipelined backpropagation with stale weights: two independent formulations
(TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

Notation: K stages (one per GPU), s = 0..K-1; the
paper's K_p register pairs give K = K_p + 1 under the per-GPU mapping
FS_i + BKS_{K_p-i+2}.  The degree of staleness of stage s is
d_s = 2(K-1-s), the paper's 2(K_p-i+1) with i = s+1.

Oracle A -- the definition, in mini-batch order with a weight-version history
(PAPER.md L63, L65, L75):  the forward of mini-batch i through stage s uses
W_s^(max(0, i-d_s)) ("weights that are 2 execution cycles old", L63; versions
clamp at 0 during fill, reading AMB-11); the backward uses the current
weights W_s^(i) (no stashing, L35/L236, reading AMB-2) and the activations
saved by that forward (L65); the SGD update produces W_s^(i+1).

Oracle B -- the schedule (BASELINE.json north_star):
a step clock t; at each step each stage s first runs the backward+update of
mini-batch b = t-2K+1+s, then the forward of mini-batch f = t-s (reading
AMB-1: backward-before-forward is the only order that gives "2 cycles stale"
for K_p = 1, L63).  Messages produced at step t are visible at step t+1.
No weight history exists; the version read is whatever the stage holds.

Hybrid (§4): pipelined training for mini-batches i < n_p, a
drain of the in-flight mini-batches, then non-pipelined training
(reading AMB-10).  Learning rate of the update from mini-batch i: the stage's
pipelined rate (or the non-pipelined rate once i >= n_p) times
gamma^(#milestones <= epoch(i)), epoch(i) = i // steps_per_epoch (AMB-8).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import layers as Lx


@dataclass
class HParams:
    lr_pipelined: Sequence[float]          # per stage
    lr_nonpipelined: float
    momentum: float = 0.9
    weight_decay: float = 0.0
    milestones: Sequence[int] = ()         # epochs
    gamma: float = 0.1
    steps_per_epoch: int = 1 << 62
    solver: str = "torch"                  # "torch" (AMB-7) | "caffe"
    nesterov: bool = False                 # AlexNet / VGG-16 (L286, L288)
    lr_policy: str = "multistep"           # "multistep" (milestones x gamma) | "inv" (LeNet-5, L284)
    inv_gamma: float = 0.0
    inv_power: float = 0.0


def staleness(K, s):
    """d_s = 2(K-1-s): the paper's degree of staleness 2(K_p - i + 1), i = s+1."""
    return 2 * (K - 1 - s)


def ring_depth(K, s):
    """Saved-activation slots of stage s: a mini-batch stays from its forward
    (step f+s) to its backward (step f+2K-1-s), i.e. 2(K-s)-1 = d_s+1 slots
    (PAPER.md L65, L75)."""
    return 2 * (K - s) - 1


def forward_version(K, s, i, n_p=None):
    """Closed form: the version of W_s read by the forward of mini-batch i."""
    if n_p is not None and i >= n_p:
        return i
    return max(0, i - staleness(K, s))


def learning_rate(hp: HParams, s, i, n_p=None):
    base = hp.lr_pipelined[s] if (n_p is None or i < n_p) else hp.lr_nonpipelined
    if hp.lr_policy == "inv":              # Caffe "inv": base (1 + gamma i)^(-power)  (L284)
        return base * (1.0 + hp.inv_gamma * i) ** (-hp.inv_power)
    epoch = i // hp.steps_per_epoch
    return base * (hp.gamma ** sum(1 for m in hp.milestones if epoch >= m))


def _tree_map(fn, *trees):
    return [{k: fn(*(t[j][k] for t in trees)) for k in trees[0][j]} for j in range(len(trees[0]))]


def _sgd_stage(params, mom, grads, lr, hp):
    new_p, new_v = [], []
    for P, V, G in zip(params, mom, grads):
        dp, dv = {}, {}
        for k in P:
            if hp.solver == "caffe":
                dp[k], dv[k] = Lx.sgd_caffe(P[k], V[k], G[k], lr, hp.momentum, hp.weight_decay, hp.nesterov)
            elif hp.nesterov:
                dp[k], dv[k] = Lx.sgd_nesterov(P[k], V[k], G[k], lr, hp.momentum, hp.weight_decay)
            else:
                dp[k], dv[k] = Lx.sgd_momentum(P[k], V[k], G[k], lr, hp.momentum, hp.weight_decay)
        new_p.append(dp)
        new_v.append(dv)
    return new_p, new_v


def _zeros_like(params):
    return _tree_map(np.zeros_like, params)


@dataclass
class Result:
    losses: List[float]
    params: list                 # per stage: list of per-layer dicts
    momentum: list
    version_log: list = field(default_factory=list)   # (t, s, 'F'|'B', mb, version)
    snapshots: Optional[list] = None                  # per step: per-stage params (Oracle B)
    stages: Optional[list] = None


def run_versioned(stages, params0, batches, hp: HParams, loss_fn=Lx.softmax_ce, n_p=None):
    """Oracle A.  `stages`: objects with forward(params, x) / backward(params, cache, g);
    `params0`: per-stage initial params; `batches`: list of (x, y)."""
    K = len(stages)
    N = len(batches)
    hist = [{0: params0[s]} for s in range(K)]
    mom = [_zeros_like(params0[s]) for s in range(K)]
    losses, log = [], []
    for i in range(N):
        x, y = batches[i]
        a = x
        caches = []
        for s in range(K):
            ver = forward_version(K, s, i, n_p)
            log.append((None, s, "F", i, ver))
            a, c = stages[s].forward(hist[s][ver], a, mb=i)
            caches.append(c)
        loss, g = loss_fn(a, y)
        losses.append(loss)
        for s in range(K - 1, -1, -1):
            log.append((None, s, "B", i, i))
            g, G = stages[s].backward(hist[s][i], caches[s], g)
            lr = learning_rate(hp, s, i, n_p)
            hist[s][i + 1], mom[s] = _sgd_stage(hist[s][i], mom[s], G, lr, hp)
            keep = i + 1 - (staleness(K, s) if (n_p is None or i + 1 < n_p) else 0)
            for v in [v for v in hist[s] if v < keep]:
                del hist[s][v]
    final = [hist[s][N] for s in range(K)]
    return Result(losses, final, mom, log, stages=stages)


def run_clocked(stages, params0, batches, hp: HParams, loss_fn=Lx.softmax_ce, n_p=None,
                snapshot=False, mom0=None):
    """Oracle B: the step-clocked schedule with message passing and no weight history.

    snapshot: False, True (per-stage params after every step, a list indexed by t), or a
    container of step indices t (a dict {t: params} holding only those; for big nets).
    mom0: initial momentum buffers per stage (default zero) -- lets a test restart the schedule
    from a drained state (weights + momentum) taken from elsewhere."""
    K = len(stages)
    N = len(batches)
    n_pipe = N if n_p is None else min(n_p, N)
    W = [params0[s] for s in range(K)]
    mom = [_zeros_like(params0[s]) for s in range(K)] if mom0 is None else [mom0[s] for s in range(K)]
    v = [0] * K
    ring = [dict() for _ in range(K)]
    inbox_f = [dict() for _ in range(K)]
    inbox_b = [dict() for _ in range(K)]
    dz = {}
    losses = [None] * N
    log = []
    snaps = [] if snapshot is True else {}

    def keep(t):
        if snapshot is True:
            snaps.append([W[s] for s in range(K)])
        elif snapshot and t in snapshot:
            snaps[t] = [W[s] for s in range(K)]

    # ---- phase 1: pipelined steps (fill, steady state, drain of mbs < n_pipe)
    t = 0
    last_t = n_pipe - 1 + 2 * K - 1 if n_pipe > 0 else -1
    while t <= last_t:
        out_f, out_b = [], []
        for s in range(K):
            b = t - 2 * K + 1 + s
            if 0 <= b < n_pipe:
                g_in = dz.pop(b) if s == K - 1 else inbox_b[s].pop(b)
                assert v[s] == b, (t, s, v[s], b)
                log.append((t, s, "B", b, v[s]))
                g, G = stages[s].backward(W[s], ring[s].pop(b), g_in)
                W[s], mom[s] = _sgd_stage(W[s], mom[s], G, learning_rate(hp, s, b, n_p), hp)
                v[s] += 1
                if s > 0:
                    out_b.append((s - 1, b, g))
            f = t - s
            if 0 <= f < n_pipe:
                a_in = batches[f][0] if s == 0 else inbox_f[s].pop(f)
                log.append((t, s, "F", f, v[s]))
                out, cache = stages[s].forward(W[s], a_in, mb=f)
                ring[s][f] = cache
                assert len(ring[s]) <= ring_depth(K, s), (t, s, len(ring[s]))
                if s == K - 1:
                    losses[f], dz[f] = loss_fn(out, batches[f][1])
                else:
                    out_f.append((s + 1, f, out))
        for (s, f, a) in out_f:
            inbox_f[s][f] = a
        for (s, b, g) in out_b:
            inbox_b[s][b] = g
        keep(t)
        t += 1
    assert all(len(r) == 0 for r in ring) and not dz

    # ---- phase 2 (hybrid): non-pipelined, one mini-batch per step
    for i in range(n_pipe, N):
        a = batches[i][0]
        caches = []
        for s in range(K):
            log.append((t, s, "F", i, v[s]))
            a, c = stages[s].forward(W[s], a, mb=i)
            caches.append(c)
        losses[i], g = loss_fn(a, batches[i][1])
        for s in range(K - 1, -1, -1):
            assert v[s] == i
            log.append((t, s, "B", i, v[s]))
            g, G = stages[s].backward(W[s], caches[s], g)
            W[s], mom[s] = _sgd_stage(W[s], mom[s], G, learning_rate(hp, s, i, n_p), hp)
            v[s] += 1
        keep(t)
        t += 1
    return Result(losses, W, mom, log, snaps if snapshot else None, stages=stages)


def run_fs_bks(stages, params0, batches, hp: HParams, loss_fn=Lx.softmax_ce):
    """Oracle C: the paper's own accelerator mapping (Fig. 3/4; SURVEY f-4).

    K = K_p + 1 stages; the forward stage FS_s and the backward stage BKS_s of stage s run on
    separate accelerators, except the last stage, whose FS and BKS share one ("FS_{K+1} and BKS_1
    ... are assigned to the same accelerator to reduce weight staleness by an execution cycle",
    L67) -- 2K_p + 1 accelerators in total (L67, L77).  One execution cycle t (L61), all
    accelerators in parallel, messages produced in cycle t visible in cycle t+1:
      FS_s, s < K-1 : forward of mini-batch f = t - s with its copy of the weights; the activation
                      goes to FS_{s+1}, the saved activations (L65) to BKS_s;
      last stage    : forward of f = t - (K-1), the loss, then the backward and update of the SAME
                      mini-batch with the same (current) weights; the error goes to BKS_{K-2};
      BKS_s, s < K-1: backward + update of b = t - 2K + 2 + s with the current weights and the saved
                      activations of b; the error goes to BKS_{s-1}; the new weights go to FS_s
                      (weight forwarding), which uses them from cycle t+1.
    FS_s therefore reads version f - 2(K-1-s) (clamped at 0): the degree of staleness
    2(K_p - i + 1) of L75, the same versions Oracle A defines -- A == C bitwise is the pin."""
    K = len(stages)
    N = len(batches)
    W = [params0[s] for s in range(K)]                # BKS (master) weights; last stage: the only copy
    Wf = [params0[s] for s in range(K)]               # FS copies (forwarded weights)
    mom = [_zeros_like(params0[s]) for s in range(K)]
    v = [0] * K
    saved = [dict() for _ in range(K)]                # BKS_s inbox of saved activations
    inbox_f = [dict() for _ in range(K)]
    inbox_b = [dict() for _ in range(K)]
    losses = [None] * N
    log = []
    t = 0
    last_t = N - 1 + 2 * K - 2 if N > 0 else -1       # stage 0's BKS handles mini-batch N-1 at N-1+2K-2
    while t <= last_t:
        out_f, out_b, out_saved, out_w = [], [], [], []
        for s in range(K):
            f = t - s
            if s == K - 1:
                if 0 <= f < N:
                    a_in = batches[f][0] if s == 0 else inbox_f[s].pop(f)
                    log.append((t, s, "F", f, v[s]))
                    out, cache = stages[s].forward(W[s], a_in, mb=f)
                    losses[f], g = loss_fn(out, batches[f][1])
                    assert v[s] == f, (t, s, v[s], f)
                    log.append((t, s, "B", f, v[s]))
                    g, G = stages[s].backward(W[s], cache, g)
                    W[s], mom[s] = _sgd_stage(W[s], mom[s], G, learning_rate(hp, s, f), hp)
                    v[s] += 1
                    if s > 0:
                        out_b.append((s - 1, f, g))
                continue
            b = t - 2 * K + 2 + s
            if 0 <= b < N:                             # BKS_s
                assert v[s] == b, (t, s, v[s], b)
                log.append((t, s, "B", b, v[s]))
                g, G = stages[s].backward(W[s], saved[s].pop(b), inbox_b[s].pop(b))
                W[s], mom[s] = _sgd_stage(W[s], mom[s], G, learning_rate(hp, s, b), hp)
                v[s] += 1
                out_w.append((s, W[s]))
                if s > 0:
                    out_b.append((s - 1, b, g))
            if 0 <= f < N:                             # FS_s
                a_in = batches[f][0] if s == 0 else inbox_f[s].pop(f)
                log.append((t, s, "F", f, v_fs(s, t, K, N)))
                out, cache = stages[s].forward(Wf[s], a_in, mb=f)
                out_f.append((s + 1, f, out))
                out_saved.append((s, f, cache))
        for (s, f, a) in out_f:
            inbox_f[s][f] = a
        for (s, b, g) in out_b:
            inbox_b[s][b] = g
        for (s, f, c) in out_saved:
            saved[s][f] = c
        for (s, w) in out_w:
            Wf[s] = w
        t += 1
    assert all(not d for d in saved) and all(not d for d in inbox_b)
    return Result(losses, W, mom, log, stages=stages)


def v_fs(s, t, K, N):
    """Version held by FS_s during cycle t of Oracle C: the BKS_s updates of cycles < t."""
    return max(0, min(N, t - 2 * K + 2 + s))


def run_sgd(stage, params0, batches, hp: HParams, loss_fn=Lx.softmax_ce):
    """Textbook non-pipelined mini-batch SGD over the whole network as one stage
    (§2): forward, loss, backward, update -- one mb at a time."""
    W = params0
    mom = _zeros_like(params0)
    losses = []
    for i, (x, y) in enumerate(batches):
        out, cache = stage.forward(W, x, mb=i)
        loss, g = loss_fn(out, y)
        losses.append(loss)
        _, G = stage.backward(W, cache, g)
        W, mom = _sgd_stage(W, mom, G, learning_rate(hp, 0, i), hp)
    return Result(losses, [W], [mom])


# --------------------------------------------------------------------------- analysis formulas
def ideal_speedup_paper(Kp):
    """2K+1 accelerators, potential speedup 2K+1 (K = register pairs)."""
    return 2 * Kp + 1


def hybrid_speedup(n_np, n_p, accel):
    """n_np / (n_p/(2K+1) + (n_np - n_p)) with 2K+1 = accel."""
    return n_np / (n_p / accel + (n_np - n_p))


def hybrid_speedup_bound(n_np, n_p):
    """Amdahl bound n_np / (n_np - n_p)."""
    return n_np / (n_np - n_p)
