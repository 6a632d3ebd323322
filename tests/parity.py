"""Shared helpers for GPU-vs-oracle parity tests (tests only).

Tolerances are BASELINE.json north_star's, with the readings of DESIGN.md section 3:
  weights (AMB-21, per tensor):  ||W_gpu - W_ref||_inf / max(||W_ref||_inf, 1e-12) <= 2e-3 for every
           conv/FC weight, bias and BatchNorm gamma tensor, at every compared step;
  BN beta (AMB-21b, per stage):  the same numerator over the stage's beta tensors, divided by the
           stage's whole parameter vector's inf-norm -- beta alone: its gradient is a sum with heavy
           cancellation, so a 1e-7 relative perturbation of the initial weights moves the fp64
           oracle's own beta tensors by 1e-2..3e-2 of their own norm after one step
           (tests/test_oracle_conditioning.py) and no float32 implementation can meet a per-tensor
           ratio there.  Small test nets (deep=False) keep beta per tensor too;
  derived tolerance (AMB-21d):   for deep nets at settings where the exact trajectory itself is
           sensitive, a tensor's tolerance is max(2e-3, K_SPREAD x spread), spread = the same ratio
           between the oracle and the oracle restarted from initial weights perturbed by 1e-7
           relative (one float32 rounding); K_SPREAD is measured, DESIGN.md AMB-21d;
  momentum buffers:              per stage vector after the drain, against max(M_TOL, allowance):
           a momentum buffer is a recent-gradient average and gradients jump when a ReLU
           pre-activation within rounding of 0 changes side (reading AMB-21f);
  BN running statistics:         per stage vector (running mean and variance of every BN layer of
           the stage) relative to its inf-norm, after the drain (reading AMB-6);
  losses:  |l_gpu - l_ref| <= 1e-2 * max(1, |l_ref|) for every mini-batch.
Every run_both / run_segments call appends its achieved errors, tolerances and spreads to the
parity-margin log (record_margin), so the margin is visible, not just pass/fail.
"""
import json
import os

import numpy as np

from oracle import network as Net
from oracle import pipeline as Pl

W_TOL = 2e-3
L_TOL = 1e-2
# Ratio between the deviation of a float32 implementation of the whole schedule and the deviation
# caused by ONE 1e-7 relative perturbation of the initial weights, measured on the oracle with every
# stored tensor rounded as the CUDA path stores it (tools/spread_ratio.py, DESIGN.md AMB-21d).
K_SPREAD = 10.0
# Ratio allowed between the CUDA path's error and the deviation of the float32-emulated oracle
# (tests/emulation.py) from the exact one: two float32 computations of the same arithmetic with
# different rounding orders differ by up to about twice either one's deviation; x2 margin (AMB-21e).
K_EMU = 4.0
# Momentum buffers are recent-gradient averages, so their error is the gradient's, and a gradient is
# not a smooth function of the rounding: a ReLU pre-activation within rounding of 0 takes the other
# side in a float32 computation (ReLU'(0) = 0, reading AMB-18) and moves one pixel's whole
# contribution.  The fp32-emulated oracle shows such jumps of up to 1.4e-2 per stage on the tiny
# ResNet test nets (tools/flip_probe.py); momentum is compared per stage against 5e-2 (reading AMB-21f).
M_TOL = 5e-2

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MARGIN_LOG = os.environ.get("PST_PARITY_LOG", os.path.join(_ROOT, "gpurun_out", "parity_margins.jsonl"))


def record_margin(tag, fields):
    """Append one JSON line {test, achieved errors, tolerances, spreads ...} to the parity-margin log
    (PST_PARITY_LOG, default gpurun_out/parity_margins.jsonl; copied to profiles/ per round) so the
    margin of every parity test is visible, not just pass/fail."""
    rec = {"test": tag}
    rec.update({k: (float(v) if isinstance(v, (np.floating, float)) else v) for k, v in fields.items()})
    try:
        os.makedirs(os.path.dirname(MARGIN_LOG), exist_ok=True)
        with open(MARGIN_LOG, "a") as f:
            f.write(json.dumps(rec, default=str) + "\n")
    except OSError:
        pass
    print("parity-margin", json.dumps(rec, default=str))


def _test_name():
    return os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]


def oracle_stages(net, ppv, dropout_seed=0, emu=False):
    bounds = Net.partition(net.layers, ppv)
    cls = Net.CNNStage
    if emu:
        from tests.emulation import EmuStage as cls
    stages = [cls(net.layers[a:b], first_stage=(s == 0), dropout_seed=dropout_seed, layer0=a)
              for s, (a, b) in enumerate(bounds)]
    return stages, bounds


def oracle_run(net, flat, ppv, data, hp, n_p=None, snapshot=False, mom0=None, dropout_seed=0, emu=False):
    stages, bounds = oracle_stages(net, ppv, dropout_seed, emu)
    per_layer = Net.unflatten(net.layers, flat)
    m0 = None
    if mom0 is not None:
        pm = Net.unflatten(net.layers, mom0)
        m0 = [pm[a:b] for a, b in bounds]
    return Pl.run_clocked(stages, [per_layer[a:b] for a, b in bounds], data, hp, n_p=n_p, snapshot=snapshot,
                          mom0=m0)


def flat_params(net, per_stage):
    return Net.flatten(net.layers, [d for st in per_stage for d in st])


def oracle_bnstats(ref):
    """Running mean and variance of every BN layer, in network order (pst_weights PST_W_BNSTATS)."""
    out = []
    for st in ref.stages:
        for ms in st.bn_stats():
            if ms is not None:
                out += [ms[0], ms[1]]
    return np.concatenate(out) if out else np.zeros(0)


def bn_layout(net):
    """(stage-independent) list of (layer index, cout) of the BN layers in network order."""
    return [(i, L.cout) for i, L in enumerate(net.layers) if L.bn]


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


def stage_errors(net, ppv, got_flat, ref_flat, keys=None):
    """max over stages of max|W_gpu - W_ref| / ||W_ref||_inf, the numerator over the stage's tensors
    named in `keys` (all if None), the denominator over the stage's whole parameter vector (reading
    AMB-21b), and the worst stage."""
    bounds = Net.partition(net.layers, ppv)
    g = Net.unflatten(net.layers, got_flat)
    r = Net.unflatten(net.layers, ref_flat)
    worst, where = 0.0, None
    for s, (a, b) in enumerate(bounds):
        nums = [float(np.abs(g[i][k] - r[i][k]).max()) for i in range(a, b) for k in r[i]
                if keys is None or k in keys]
        if not nums:
            continue
        den = max(float(np.abs(r[i][k]).max()) for i in range(a, b) for k in r[i])
        e = max(nums) / max(den, 1e-12)
        if e > worst:
            worst, where = e, f"stage{s}"
    return worst, where


def split_errors(net, ppv, got_flat, ref_flat, deep, spread=None):
    """The weight measure of this module's docstring.  Returns
    {"tensor": (worst ratio err/tol, err, tol, name), "beta": (ratio, err, tol, where)}:
    per tensor for W / bias / gamma (and beta when not deep), per stage for beta when deep.
    spread: optional allowance per tensor / per stage (allowances(): K_SPREAD x the perturbation
    spread and K_EMU x the float32-emulation deviation, whichever is larger)."""
    g = Net.unflatten(net.layers, got_flat)
    r = Net.unflatten(net.layers, ref_flat)
    out = {"tensor": (0.0, 0.0, W_TOL, None), "beta": (0.0, 0.0, W_TOL, None)}
    for i, (dg, dr) in enumerate(zip(g, r)):
        for k in dr:
            if deep and k == "beta":
                continue
            name = f"layer{i + 1}.{k}"
            e = float(np.abs(dg[k] - dr[k]).max() / max(np.abs(dr[k]).max(), 1e-12))
            tol = max(W_TOL, spread[name]) if spread else W_TOL
            if e / tol > out["tensor"][0]:
                out["tensor"] = (e / tol, e, tol, name)
    if deep:
        bounds = Net.partition(net.layers, ppv)
        for s, (a, b) in enumerate(bounds):
            nums = [float(np.abs(g[i]["beta"] - r[i]["beta"]).max()) for i in range(a, b) if "beta" in r[i]]
            if not nums:
                continue
            den = max(float(np.abs(r[i][k]).max()) for i in range(a, b) for k in r[i])
            e = max(nums) / max(den, 1e-12)
            tol = max(W_TOL, spread[f"stage{s}.beta"]) if spread else W_TOL
            if e / tol > out["beta"][0]:
                out["beta"] = (e / tol, e, tol, f"stage{s}")
    return out


def tensor_spreads(net, ppv, a_flat, b_flat):
    """Per-tensor ratios (and per-stage beta ratios) between two oracle states: the oracle's own
    sensitivity when a_flat/b_flat come from the perturbed / unperturbed runs."""
    g = Net.unflatten(net.layers, a_flat)
    r = Net.unflatten(net.layers, b_flat)
    sp = {}
    for i, (dg, dr) in enumerate(zip(g, r)):
        for k in dr:
            sp[f"layer{i + 1}.{k}"] = float(np.abs(dg[k] - dr[k]).max() / max(np.abs(dr[k]).max(), 1e-12))
    for s, (a, b) in enumerate(Net.partition(net.layers, ppv)):
        nums = [float(np.abs(g[i]["beta"] - r[i]["beta"]).max()) for i in range(a, b) if "beta" in r[i]]
        den = max(float(np.abs(r[i][k]).max()) for i in range(a, b) for k in r[i])
        sp[f"stage{s}.beta"] = max(nums) / max(den, 1e-12) if nums else 0.0
    return sp


def bnstat_errors(net, ppv, got, ref, spread=None):
    """Per stage: max |Δ| over the stage's BN running means and variances / their inf-norm, against
    max(2e-3, K_SPREAD x the oracle's own spread of the same measure).  Returns (worst err/tol,
    err, tol, where) and the per-stage errors {stage: err}."""
    bounds = Net.partition(net.layers, ppv)
    worst, per, off = (0.0, 0.0, W_TOL, None), {}, 0
    for s, (a, b) in enumerate(bounds):
        n = 2 * sum(L.cout for L in net.layers[a:b] if L.bn)
        if n:
            e = float(np.abs(got[off:off + n] - ref[off:off + n]).max() / max(np.abs(ref[off:off + n]).max(), 1e-12))
            per[s] = e
            tol = max(W_TOL, spread.get(s, 0.0)) if spread else W_TOL
            if e / tol > worst[0]:
                worst = (e / tol, e, tol, f"stage{s}")
        off += n
    return worst, per


def loss_errors(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))))


def hparams(cfg_lr, K, lr_np, momentum, wd, milestones=(), gamma=0.1, spe=1 << 62):
    return Pl.HParams(lr_pipelined=list(cfg_lr), lr_nonpipelined=lr_np, momentum=momentum,
                      weight_decay=wd, milestones=tuple(milestones), gamma=gamma, steps_per_epoch=spe)


class Parity:
    """Outcome of run_both: every measure, its tolerance, and assert_ok()."""

    def __init__(self, tag):
        self.tag = tag
        self.w = {"tensor": (0.0, 0.0, W_TOL, None), "beta": (0.0, 0.0, W_TOL, None)}
        self.mom = (0.0, 0.0, M_TOL, None)   # per stage (ratio, err, tol, where)
        self.bn = (0.0, 0.0, W_TOL, None)
        self.loss = 0.0
        self.stage = (0.0, None)     # the round-1 whole-stage-vector measure, for reference
        self.versions = None
        self.ref = None
        self.compared = 0
        self.extra = {}

    def fold_w(self, d):
        for k in d:
            if d[k][0] > self.w[k][0]:
                self.w[k] = d[k]

    def fields(self):
        f = {"weights_tensor_err": self.w["tensor"][1], "weights_tensor_tol": self.w["tensor"][2],
             "weights_tensor_where": self.w["tensor"][3],
             "beta_stage_err": self.w["beta"][1], "beta_stage_tol": self.w["beta"][2], "beta_where": self.w["beta"][3],
             "momentum_stage_err": self.mom[1], "momentum_stage_tol": self.mom[2], "momentum_where": self.mom[3],
             "bnstats_stage_err": self.bn[1], "bnstats_tol": self.bn[2], "bnstats_where": self.bn[3],
             "loss_err": self.loss, "loss_tol": L_TOL,
             "whole_stage_vector_err": self.stage[0], "steps_compared": self.compared}
        f.update(self.extra)
        return f

    def assert_ok(self):
        record_margin(self.tag, self.fields())
        for k in ("tensor", "beta"):
            assert self.w[k][0] <= 1.0, ("weights", k, self.w[k])
        assert self.mom[0] <= 1.0, ("momentum", self.mom)
        assert self.bn[0] <= 1.0, ("bnstats", self.bn)
        assert self.loss <= L_TOL, ("loss", self.loss)
        return self


def compare_final(P, net, ppv, got, got_v, got_bn, losses, ref, deep, sp=None):
    """Fold the drained state (parameters, momentum, BN running statistics; canonical order) and
    the losses into the Parity P.  sp: the oracle's own spreads {"w", "v", "bn"} (oracle_spreads)."""
    sp = sp or {}
    want = flat_params(net, ref.params)
    P.fold_w(split_errors(net, ppv, got, want, deep, sp.get("w")))
    P.stage = max(P.stage, stage_errors(net, ppv, got, want), key=lambda z: z[0])
    P.mom = momentum_errors(net, ppv, got_v, flat_params(net, ref.momentum), sp.get("vs"))
    P.bn = bnstat_errors(net, ppv, got_bn, oracle_bnstats(ref), sp.get("bn"))[0]
    P.loss = loss_errors(losses, ref.losses)
    return P


def stage_vector_errors(net, ppv, got_flat, ref_flat):
    """{stage: max|Δ| over the stage's vector / its inf-norm}."""
    bounds = Net.partition(net.layers, ppv)
    g = Net.unflatten(net.layers, got_flat)
    r = Net.unflatten(net.layers, ref_flat)
    out = {}
    for s, (a, b) in enumerate(bounds):
        num = max(float(np.abs(g[i][k] - r[i][k]).max()) for i in range(a, b) for k in r[i])
        den = max(float(np.abs(r[i][k]).max()) for i in range(a, b) for k in r[i])
        out[s] = num / max(den, 1e-12)
    return out


def momentum_errors(net, ppv, got_v, ref_v, allow=None):
    """Momentum buffers per stage against max(M_TOL, allowance) (reading AMB-21f)."""
    worst = (0.0, 0.0, M_TOL, None)
    for s, e in stage_vector_errors(net, ppv, got_v, ref_v).items():
        tol = max(M_TOL, (allow or {}).get(s, 0.0))
        if e / tol > worst[0]:
            worst = (e / tol, e, tol, f"stage{s}")
    return worst


def oracle_spreads(net, ppv, ref, refp):
    """Per-tensor ratios between two oracle runs (final weights, momentum buffers, BN running
    statistics): refp from initial weights perturbed by 1e-7 relative (reading AMB-21d), or the
    float32-emulated oracle (tests/emulation.py, reading AMB-21e)."""
    return {"w": tensor_spreads(net, ppv, flat_params(net, refp.params), flat_params(net, ref.params)),
            "v": tensor_spreads(net, ppv, flat_params(net, refp.momentum), flat_params(net, ref.momentum)),
            "vs": stage_vector_errors(net, ppv, flat_params(net, refp.momentum), flat_params(net, ref.momentum)),
            "bn": bnstat_errors(net, ppv, oracle_bnstats(refp), oracle_bnstats(ref))[1]}


def allowances(sp_pert=None, sp_emu=None):
    """max(K_SPREAD x perturbation spread, K_EMU x emulation deviation) per key."""
    out = {}
    for kind in ("w", "v", "vs", "bn"):
        a, b = (sp_pert or {}).get(kind, {}), (sp_emu or {}).get(kind, {})
        out[kind] = {k: max(K_SPREAD * a.get(k, 0.0), K_EMU * b.get(k, 0.0)) for k in set(a) | set(b)}
    return out


def perturbed(flat):
    """Initial weights moved by 1e-7 relative (one float32 rounding), fixed seed."""
    return flat.astype(np.float64) * (1 + 1e-7 * np.random.default_rng(0).standard_normal(flat.shape))


def run_both(pst, net, ppv, B, N, lr, lr_np=None, mom=0.9, wd=1e-4, n_p=None, spe=1 << 62,
             milestones=(), per_step=True, seed=5, check=None, deep=False, spread=True, solver_kw=None,
             tag=None, dropout_seed=0, emu=True):
    """Train the same seeded mini-batches through libpst (all stages on cuda:0, local mode)
    and through Oracle B; compare the weights after every compared step and after the drain
    (split measure, see the module docstring), the momentum buffers and BN running statistics
    after the drain, and the loss of every mini-batch.  `check`: None = every step (if per_step),
    else the global step indices t after which the weights are compared (big nets).
    deep: beta per stage (AMB-21b).  spread: also run the oracle from initial weights perturbed by
    1e-7 relative and derive each tensor's tolerance from that spread (AMB-21d).
    Returns a Parity (call .assert_ok())."""
    import pst_workloads as W
    K = len(ppv) + 1
    flat = W.init_params(net, seed=seed)
    data = W.batches(net.in_shape, B, N, seed=seed + 100)
    lr_np = lr[-1] if lr_np is None else lr_np
    hp = hparams(lr, K, lr_np, mom, wd, milestones, 0.1, spe)
    skw = dict(solver_kw or {})        # solver / nesterov / lr_policy / inv_gamma / inv_power (/ mapping)
    for k, v in skw.items():
        if hasattr(hp, k):
            setattr(hp, k, v)
    snap = (True if check is None else set(check)) if per_step else False
    ref = oracle_run(net, flat, ppv, data, hp, n_p=n_p, snapshot=snap, dropout_seed=dropout_seed)
    P = Parity(tag or _test_name())
    P.ref = ref
    sp_steps, sp = {}, None
    if spread:
        # the oracle's own sensitivity (AMB-21d) and a float32 emulation of the same arithmetic (AMB-21e)
        refp = oracle_run(net, perturbed(flat), ppv, data, hp, n_p=n_p, snapshot=snap, dropout_seed=dropout_seed)
        refe = oracle_run(net, flat, ppv, data, hp, n_p=n_p, snapshot=snap, dropout_seed=dropout_seed, emu=emu)
        snaps = ref.snapshots if ref.snapshots is not None else {}
        idx = range(len(snaps)) if isinstance(snaps, list) else snaps.keys()
        for t in idx:
            a = tensor_spreads(net, ppv, flat_params(net, refp.snapshots[t]), flat_params(net, snaps[t]))
            b = tensor_spreads(net, ppv, flat_params(net, refe.snapshots[t]), flat_params(net, snaps[t]))
            sp_steps[t] = allowances({"w": a}, {"w": b})["w"]
        sp_p, sp_e = oracle_spreads(net, ppv, ref, refp), oracle_spreads(net, ppv, ref, refe)
        sp = allowances(sp_p, sp_e)
        P.extra["spread_final_max"] = max(sp_p["w"].values())
        P.extra["emu_dev_final_max"] = max(sp_e["w"].values())
        P.extra["emu_dev_momentum_max"] = max(sp_e["vs"].values())
        P.extra["k_spread"], P.extra["k_emu"] = K_SPREAD, K_EMU
    pipe = pst.Pipeline(net, flat, ppv, B, lr, lr_np, momentum=mom, weight_decay=wd, milestones=milestones,
                        steps_per_epoch=spe, dropout_seed=dropout_seed, **skw)
    if n_p is not None:
        assert n_p % spe == 0
        pipe.set_hybrid(n_p // spe)
    for x, y in data:
        pipe.step(x, y)
        if per_step:
            # a hybrid switch inserts the drain steps before this mini-batch's step
            steps, _ = pipe.progress()
            if check is None or (steps - 1) in ref.snapshots:
                got, want = pipe.weights(), flat_params(net, ref.snapshots[steps - 1])
                P.fold_w(split_errors(net, ppv, got, want, deep, sp_steps.get(steps - 1)))
                P.stage = max(P.stage, stage_errors(net, ppv, got, want), key=lambda z: z[0])
                P.compared += 1
    pipe.flush()
    n = Net.n_params(net.layers)
    state = pipe.weights(pst.W_PARAMS | pst.W_MOMENTUM | pst.W_BNSTATS)
    compare_final(P, net, ppv, state[:n], state[n:2 * n], state[2 * n:], pipe.losses(0, N), ref, deep, sp)
    P.versions = pipe.versions()
    pipe.close()
    if per_step and check is not None:
        assert P.compared == len(set(check)), (P.compared, sorted(check))
    assert np.all(np.isfinite(ref.losses)), "the oracle's trajectory diverged: pick a smaller lr"
    return P


def run_segments(pst, net, ppv, B, seg_lens, lr, lr_np=None, mom=0.9, wd=1e-4, seed=5, deep=True, tag=None,
                 spread=True, emu=True):
    """Segment ("shadowing") parity for trajectories that are chaotic (reading AMB-21c).

    The GPU trains sum(seg_lens) mini-batches; after each segment the pipe is drained
    (pst_flush) and the oracle (Oracle B) is restarted from the GPU's drained state --
    its weights and momentum buffers -- for the next segment's mini-batches, with a fresh
    pipeline fill exactly like the GPU's.  Within a segment every mini-batch's loss and, after
    the drain, the weights (split measure) and momentum are compared.  Returns a Parity whose
    ref.losses are the oracle's losses of all segments."""
    import pst_workloads as W
    K = len(ppv) + 1
    flat = W.init_params(net, seed=seed)
    N = int(sum(seg_lens))
    data = W.batches(net.in_shape, B, N, seed=seed + 100)
    lr_np = lr[-1] if lr_np is None else lr_np
    hp = hparams(lr, K, lr_np, mom, wd)
    pipe = pst.Pipeline(net, flat, ppv, B, lr, lr_np, momentum=mom, weight_decay=wd)
    n = Net.n_params(net.layers)
    w_state = flat.astype(np.float64)
    v_state = np.zeros_like(w_state)
    P = Parity(tag or _test_name())
    losses = []
    i0 = 0
    for M in seg_lens:
        seg = data[i0:i0 + M]
        ref = oracle_run(net, w_state, ppv, seg, hp, mom0=v_state)
        sp = {}
        if spread:   # the oracle's own sensitivity over this segment and its float32 emulation
            sp = allowances(oracle_spreads(net, ppv, ref, oracle_run(net, perturbed(w_state), ppv, seg, hp, mom0=v_state)),
                            oracle_spreads(net, ppv, ref, oracle_run(net, w_state, ppv, seg, hp, mom0=v_state, emu=True))
                            if emu else None)
        for x, y in seg:
            pipe.step(x, y)
        pipe.flush()
        state = pipe.weights(pst.W_PARAMS | pst.W_MOMENTUM).astype(np.float64)
        w_state, v_state = state[:n], state[n:2 * n]
        P.fold_w(split_errors(net, ppv, w_state, flat_params(net, ref.params), deep, sp.get("w")))
        m = momentum_errors(net, ppv, v_state, flat_params(net, ref.momentum), sp.get("vs"))
        if m[0] > P.mom[0]:
            P.mom = m
        P.stage = max(P.stage, stage_errors(net, ppv, w_state, flat_params(net, ref.params)), key=lambda z: z[0])
        P.loss = max(P.loss, loss_errors(pipe.losses(i0, M), ref.losses))
        P.compared += 1
        losses += list(ref.losses)
        assert np.all(np.isfinite(ref.losses)), "the oracle's trajectory diverged: pick a smaller lr"
        i0 += M
    pipe.close()
    P.extra["segments"] = list(seg_lens)

    class _R:
        pass
    P.ref = _R()
    P.ref.losses = losses
    return P
