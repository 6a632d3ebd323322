"""Pins for oracle/network.py and oracle/pipeline.py (CPU, no GPU).

What pins what:
  * K=1 == textbook SGD: torch autograd + torch.optim.SGD in float64 (library),
  * Oracle A (definition) == Oracle B (schedule) bitwise for K in {1,2,3,4},
  * version log == closed form max(0, i - 2(K-1-s)) forward / i backward,
  * the hand-derived scalar worked example (tests/golden/scalar_pipeline_k2.json),
  * the K=2 occupancy timeline of P:L61,
  * Table 1 / Table 5 PPVs valid; mid-block registers (Table 4's (5,12,17)): non-pipelined
    == torch autograd SGD, pipelined A == B, stage pair == finite differences,
  * Table 6 "Weight" column == 4-byte parameter count in MiB,
  * the speedup formulas of P:L77.
"""
import json
import os

import numpy as np
import pytest

from oracle import layers as Lx
from oracle import network as Net
from oracle import pipeline as Pl
import pst_workloads as W
from tests.torch_ref import train_sgd

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def make_stages(net, ppv):
    bounds = Net.partition(net.layers, ppv)
    return [Net.CNNStage(net.layers[a:b], first_stage=(s == 0)) for s, (a, b) in enumerate(bounds)], bounds


def split_params(net, flat, bounds):
    per_layer = Net.unflatten(net.layers, flat)
    return [per_layer[a:b] for a, b in bounds]


def flat_of(net, bounds, per_stage):
    per_layer = [d for st in per_stage for d in st]
    return Net.flatten(net.layers, per_layer)


def hp_for(K, lr=0.05, wd=1e-3, mom=0.9, **kw):
    return Pl.HParams(lr_pipelined=[lr] * K, lr_nonpipelined=lr, momentum=mom, weight_decay=wd, **kw)


NETS = {
    "tiny_resnet": (W.tiny_resnet(width=4, hw=8, n=1), 6, {1: (), 2: (3,), 3: (1, 3), 4: (1, 3, 5)}),
    "tiny_cnn": (W.tiny_cnn(hw=8), 6, {1: (), 2: (2,), 3: (1, 2), 4: (1, 2, 3)}),
}


@pytest.mark.parametrize("name", list(NETS))
def test_k1_equals_torch_autograd_sgd(name):
    net, B, _ = NETS[name]
    flat = W.init_params(net, seed=3)
    data = W.batches(net.in_shape, B, 6, seed=11)
    stages, bounds = make_stages(net, ())
    res = Pl.run_sgd(stages[0], split_params(net, flat, bounds)[0], data, hp_for(1))
    t_losses, t_flat = train_sgd(net, flat, data, 0.05, 0.9, 1e-3)
    np.testing.assert_allclose(res.losses, t_losses, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(Net.flatten(net.layers, res.params[0]), t_flat, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("name", list(NETS))
@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_versioned_equals_clocked_bitwise(name, K):
    net, B, ppvs = NETS[name]
    flat = W.init_params(net, seed=5)
    data = W.batches(net.in_shape, B, 9, seed=7)
    sa, bounds = make_stages(net, ppvs[K])
    sb, _ = make_stages(net, ppvs[K])
    p0 = split_params(net, flat, bounds)
    hp = hp_for(K, milestones=(1,), steps_per_epoch=5, lr=0.08)
    ra = Pl.run_versioned(sa, p0, data, hp)
    rb = Pl.run_clocked(sb, p0, data, hp)
    assert ra.losses == rb.losses
    assert np.array_equal(flat_of(net, bounds, ra.params), flat_of(net, bounds, rb.params))
    for st_a, st_b in zip(sa, sb):
        for x, y in zip(st_a.bn_stats(), st_b.bn_stats()):
            if x is not None:
                assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])


def test_k1_versioned_equals_plain_sgd_bitwise():
    net, B, _ = NETS["tiny_resnet"]
    flat = W.init_params(net, seed=1)
    data = W.batches(net.in_shape, B, 5, seed=2)
    s1, bounds = make_stages(net, ())
    s2, _ = make_stages(net, ())
    p0 = split_params(net, flat, bounds)
    ra = Pl.run_versioned(s1, p0, data, hp_for(1))
    rs = Pl.run_sgd(s2[0], p0[0], data, hp_for(1))
    assert ra.losses == rs.losses
    assert np.array_equal(Net.flatten(net.layers, ra.params[0]), Net.flatten(net.layers, rs.params[0]))


@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_version_log_closed_form(K):
    net, B, ppvs = NETS["tiny_cnn"]
    flat = W.init_params(net, seed=5)
    data = W.batches(net.in_shape, 2, 12, seed=7)
    st, bounds = make_stages(net, ppvs[K])
    rb = Pl.run_clocked(st, split_params(net, flat, bounds), data, hp_for(K))
    nF = nB = 0
    for t, s, kind, mb, ver in rb.version_log:
        if kind == "F":
            nF += 1
            assert ver == max(0, mb - 2 * (K - 1 - s)), (t, s, mb, ver)
            assert t == mb + s
        else:
            nB += 1
            assert ver == mb
            assert t == mb + 2 * K - 1 - s
    assert nF == nB == 12 * K


def test_forward_before_backward_would_add_one_cycle():
    """AMB-1: with the opposite in-step order stage 0 would read version i-(d_0+1)."""
    K = 2
    for i in range(3, 10):
        # backward of mb b on stage 0 happens at t = b + 2K-1; forward of i at t = i.
        done_before = sum(1 for b in range(i) if b + 2 * K - 1 < i)
        done_same_step = sum(1 for b in range(i) if b + 2 * K - 1 == i)
        assert done_before + done_same_step == Pl.forward_version(K, 0, i)
        assert done_before == max(0, i - 2 * (K - 1) - 1)


def test_k2_occupancy_timeline_p61():
    """cycle 0 FS1 has mb0; cycle 1 FS1 mb1, FS2 mb0; cycle 2 FS1 mb2, FS2 mb1, BKS1 mb0."""
    net, B, ppvs = NETS["tiny_cnn"]
    flat = W.init_params(net, seed=5)
    data = W.batches(net.in_shape, 2, 5, seed=7)
    st, bounds = make_stages(net, ppvs[2])
    rb = Pl.run_clocked(st, split_params(net, flat, bounds), data, hp_for(2))
    at = {}
    for t, s, kind, mb, _ in rb.version_log:
        at.setdefault(t, []).append((s, kind, mb))
    assert at[0] == [(0, "F", 0)]
    assert at[1] == [(0, "F", 1), (1, "F", 0)]
    assert at[2] == [(0, "F", 2), (1, "B", 0), (1, "F", 1)]
    assert at[3] == [(0, "B", 0), (0, "F", 3), (1, "B", 1), (1, "F", 2)]
    assert at[4] == [(0, "B", 1), (0, "F", 4), (1, "B", 2), (1, "F", 3)]


class ScalarStage:
    """h = w * x with params [{'W': w}] -- the net of the worked example."""

    def forward(self, params, x, mb=0):
        return params[0]["W"] * x, x

    def backward(self, params, x, g):
        return params[0]["W"] * g, [{"W": g * x}]


def half_square(y, _label):
    return 0.5 * float(y * y), y


@pytest.mark.parametrize("name", ["scalar_pipeline_k2.json", "scalar_pipeline_k3_momentum.json"])
def test_scalar_worked_example_golden(name):
    """Oracle A and Oracle B against the closed-form scalar recursion of tools/make_golden_scalar.py
    (written from P:L61-L75 without importing oracle/); the K=2 file reproduces SURVEY Appendix B's
    hand-derived table to its 8 printed decimals, the K=3 file adds momentum and weight decay."""
    gold = json.load(open(os.path.join(GOLDEN, name)))
    atol = gold["atol"]
    K = gold["hparams"]["K"]
    N = len(gold["pipelined"]["loss"])
    data = [(1.0, None)] * N
    lr, mu, wd = gold["hparams"]["lr"], gold["hparams"]["momentum"], gold["hparams"]["weight_decay"]
    hp = Pl.HParams(lr_pipelined=[lr] * K, lr_nonpipelined=lr, momentum=mu, weight_decay=wd)
    p0 = [[{"W": np.float64(1.0)}] for _ in range(K)]
    stages = lambda: [ScalarStage() for _ in range(K)]
    rb = Pl.run_clocked(stages(), p0, data, hp, loss_fn=half_square)
    np.testing.assert_allclose(rb.losses, gold["pipelined"]["loss"], atol=atol, rtol=0)
    # per-mini-batch weights after each update: Oracle A's history
    for n in range(1, N + 1):
        ra = Pl.run_versioned(stages(), p0, data[:n], hp, loss_fn=half_square)
        got = [float(ra.params[s][0]["W"]) for s in range(K)]
        np.testing.assert_allclose(got, [gold["pipelined"]["w_after"][s][n - 1] for s in range(K)], atol=atol, rtol=0)
    # non-pipelined (K=1 over the chain == hybrid with n_p = 0)
    rn = Pl.run_clocked(stages(), p0, data, hp, loss_fn=half_square, n_p=0)
    np.testing.assert_allclose(rn.losses, gold["nonpipelined"]["loss"], atol=atol, rtol=0)
    np.testing.assert_allclose([float(rn.params[s][0]["W"]) for s in range(K)],
                               [gold["nonpipelined"]["w_after"][s][-1] for s in range(K)], atol=atol, rtol=0)


def test_golden_files_match_their_generator():
    """The committed golden files are exactly what tools/make_golden_scalar.py writes today, and the
    K=2 file agrees with SURVEY Appendix B's hand-derived 8-decimal table."""
    import subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "make_golden_scalar.py"), "--check"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    gold = json.load(open(os.path.join(GOLDEN, "scalar_pipeline_k2.json")))
    hand = {"loss": [0.5, 0.405, 0.32805, 0.21523361, 0.15053029],
            "a": [0.9, 0.819, 0.75339, 0.70556031, 0.66880078], "b": [0.9, 0.81, 0.729, 0.669951, 0.6250133],
            "np_loss": [0.5, 0.32805, 0.23399258, 0.17623916, 0.13796786]}
    np.testing.assert_allclose(gold["pipelined"]["loss"], hand["loss"], atol=5e-9)
    np.testing.assert_allclose(gold["pipelined"]["w_after"][0], hand["a"], atol=5e-9)
    np.testing.assert_allclose(gold["pipelined"]["w_after"][1], hand["b"], atol=5e-9)
    np.testing.assert_allclose(gold["nonpipelined"]["loss"], hand["np_loss"], atol=5e-9)


@pytest.mark.parametrize("n_p", [0, 1, 3, 7])
def test_hybrid_versioned_equals_clocked(n_p):
    net, B, ppvs = NETS["tiny_resnet"]
    K = 3
    flat = W.init_params(net, seed=9)
    data = W.batches(net.in_shape, B, 8, seed=4)
    sa, bounds = make_stages(net, ppvs[K])
    sb, _ = make_stages(net, ppvs[K])
    p0 = split_params(net, flat, bounds)
    hp = Pl.HParams(lr_pipelined=[0.01, 0.02, 0.05], lr_nonpipelined=0.1, momentum=0.9, weight_decay=1e-4)
    ra = Pl.run_versioned(sa, p0, data, hp, n_p=n_p)
    rb = Pl.run_clocked(sb, p0, data, hp, n_p=n_p)
    assert ra.losses == rb.losses
    assert np.array_equal(flat_of(net, bounds, ra.params), flat_of(net, bounds, rb.params))
    for t, s, kind, mb, ver in rb.version_log:
        if kind == "F":
            assert ver == (mb if mb >= n_p else max(0, mb - 2 * (K - 1 - s)))


def test_hybrid_zero_is_nonpipelined_sgd():
    net, B, ppvs = NETS["tiny_cnn"]
    flat = W.init_params(net, seed=9)
    data = W.batches(net.in_shape, B, 5, seed=4)
    sb, bounds = make_stages(net, ppvs[4])
    p0 = split_params(net, flat, bounds)
    hp = Pl.HParams(lr_pipelined=[0.5] * 4, lr_nonpipelined=0.05, momentum=0.9, weight_decay=1e-3)
    rb = Pl.run_clocked(sb, p0, data, hp, n_p=0)
    t_losses, t_flat = train_sgd(net, flat, data, 0.05, 0.9, 1e-3)
    np.testing.assert_allclose(rb.losses, t_losses, rtol=1e-10)
    np.testing.assert_allclose(flat_of(net, bounds, rb.params), t_flat, rtol=1e-9, atol=1e-12)


def test_ring_depths():
    for K, depths in [(2, [3, 1]), (4, [7, 5, 3, 1]), (8, [15, 13, 11, 9, 7, 5, 3, 1])]:
        assert [Pl.ring_depth(K, s) for s in range(K)] == depths
        assert [Pl.staleness(K, s) + 1 for s in range(K)] == depths


PPV_TABLES = {
    "lenet5": [(1,), (1, 2), (1, 2, 3), (1, 2, 3, 4)],
    "alexnet": [(1,), (1, 2), (1, 2, 3)],
    "vgg16": [(2,), (2, 4), (2, 4, 7), (2, 4, 7, 10)],
    "resnet20": [(7,), (7, 13), (7, 13, 19)],
}


@pytest.mark.parametrize("name", list(PPV_TABLES))
def test_table1_ppvs_valid(name):
    net = W.by_name(name)
    assert W.weighted_layer_count(net) == {"lenet5": 5, "alexnet": 8, "vgg16": 16, "resnet20": 20}[name]
    for ppv in PPV_TABLES[name]:
        assert len(Net.partition(net.layers, ppv)) == len(ppv) + 1


def test_table5_ppvs_and_rejections():
    for depth, p in [(20, 7), (56, 19), (110, 37), (224, 75), (362, 121)]:
        net = W.resnet_cifar(depth)
        assert W.weighted_layer_count(net) == depth
        Net.partition(net.layers, (p,))
    assert len(Net.partition(W.resnet_cifar(20).layers, (5, 12, 17))) == 4   # mid-block 12
    with pytest.raises(ValueError):
        Net.partition(W.resnet_cifar(20).layers, (7, 7))
    with pytest.raises(ValueError):
        Net.partition(W.resnet_cifar(20).layers, (20,))


def test_midblock_register_positions():
    """ResNet-20 weighted layers: conv1, then blocks (2,3), (4,5), ..., (18,19), FC 20.  A register
    after an even layer 2..18 sits inside a block ("inserting pipeline register pairs within
    residual function blocks"); after an odd one it sits between blocks."""
    net = W.resnet_cifar(20)
    opn = Net.open_block_at(net.layers)
    assert [p for p in range(1, 20) if opn[p]] == list(range(2, 19, 2))


MID = {"tiny_resnet2": (W.tiny_resnet(width=4, hw=8, n=2), 6)}


@pytest.mark.parametrize("ppv", [(2,), (6,), (2, 4), (1, 2, 4), (2, 3, 6, 8)])
def test_midblock_nonpipelined_equals_torch_autograd(ppv):
    """A mid-block partition changes nothing in the arithmetic of non-pipelined training (hybrid
    with n_p = 0): the two-tensor registers must reproduce torch autograd + torch.optim.SGD over the
    whole network (library routine, float64) -- a dropped shortcut gradient or a wrong block input
    fails this."""
    net, B = MID["tiny_resnet2"]
    flat = W.init_params(net, seed=13)
    data = W.batches(net.in_shape, B, 5, seed=17)
    K = len(ppv) + 1
    stages, bounds = make_stages(net, ppv)
    assert any(Net.open_block_at(net.layers)[p] for p in ppv)
    res = Pl.run_clocked(stages, split_params(net, flat, bounds), data, hp_for(K), n_p=0)
    t_losses, t_flat = train_sgd(net, flat, data, 0.05, 0.9, 1e-3)
    np.testing.assert_allclose(res.losses, t_losses, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(flat_of(net, bounds, res.params), t_flat, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("ppv", [(2,), (6,), (2, 4), (1, 2, 3, 4)])
def test_midblock_versioned_equals_clocked(ppv):
    """Pipelined with mid-block registers: Oracle A == Oracle B bitwise, versions = closed form."""
    net, B = MID["tiny_resnet2"]
    K = len(ppv) + 1
    flat = W.init_params(net, seed=19)
    data = W.batches(net.in_shape, B, 9, seed=23)
    sa, bounds = make_stages(net, ppv)
    sb, _ = make_stages(net, ppv)
    p0 = split_params(net, flat, bounds)
    ra = Pl.run_versioned(sa, p0, data, hp_for(K))
    rb = Pl.run_clocked(sb, p0, data, hp_for(K))
    assert ra.losses == rb.losses
    assert np.array_equal(flat_of(net, bounds, ra.params), flat_of(net, bounds, rb.params))
    for t, s, kind, mb, ver in rb.version_log:
        if kind == "F":
            assert ver == max(0, mb - 2 * (K - 1 - s))


def test_midblock_stage_pair_finite_differences():
    """The backward of a stage pair split inside a block (tuple registers both ways) against
    central finite differences of the composed loss, for the weights of both stages and the input."""
    net, B = MID["tiny_resnet2"]
    ppv = (2,)
    flat = W.init_params(net, seed=29)
    x, y = W.make_batch(net.in_shape, B, 0, seed=31)
    stages, bounds = make_stages(net, ppv)
    P = split_params(net, flat, bounds)
    s0, s1 = stages
    s0.first_stage = False        # also check the input gradient

    def loss_of(P0, P1, xx):
        st0 = Net.CNNStage(net.layers[bounds[0][0]:bounds[0][1]])
        st1 = Net.CNNStage(net.layers[bounds[1][0]:bounds[1][1]])
        h, _ = st0.forward(P0, xx)
        assert isinstance(h, tuple)
        o, _ = st1.forward(P1, h)
        return Lx.softmax_ce(o, y)[0]

    h, c0 = s0.forward(P[0], x)
    o, c1 = s1.forward(P[1], h)
    _, g = Lx.softmax_ce(o, y)
    gh, G1 = s1.backward(P[1], c1, g)
    assert isinstance(gh, tuple)
    gx, G0 = s0.backward(P[0], c0, gh)
    rng = np.random.default_rng(0)
    eps = 1e-6
    for st, Pst, G in ((0, P[0], G0), (1, P[1], G1)):
        for li, d in enumerate(Pst):
            for k in d:
                for _ in range(2):
                    idx = tuple(rng.integers(0, n) for n in d[k].shape)
                    Pp = [[{kk: v.copy() for kk, v in dd.items()} for dd in ps] for ps in P]
                    Pm = [[{kk: v.copy() for kk, v in dd.items()} for dd in ps] for ps in P]
                    Pp[st][li][k][idx] += eps
                    Pm[st][li][k][idx] -= eps
                    fd = (loss_of(*Pp, x) - loss_of(*Pm, x)) / (2 * eps)
                    assert abs(fd - G[li][k][idx]) <= 1e-6 * max(1.0, abs(fd)), (st, li, k, fd, G[li][k][idx])
    xd = np.asarray(x, dtype=np.float64)
    for _ in range(3):
        idx = tuple(rng.integers(0, n) for n in xd.shape)
        xp, xm = xd.copy(), xd.copy()
        xp[idx] += eps
        xm[idx] -= eps
        fd = (loss_of(P[0], P[1], xp) - loss_of(P[0], P[1], xm)) / (2 * eps)
        assert abs(fd - gx[idx]) <= 1e-6 * max(1.0, abs(fd))


def test_table6_weight_column_param_counts():
    """P:L200-204 Table 6 'Weight' column: 1.03, 3.25, 6.59, 13.64, 22.17 MB."""
    for depth, mib, count in [(20, 1.03, 269722), (56, 3.25, 853018), (110, 6.59, 1727962),
                              (224, 13.64, 3575066), (362, 22.17, 5811034)]:
        net = W.resnet_cifar(depth)
        n = Net.n_params(net.layers)
        assert n == W.param_count(net) == count
        assert round(n * 4 / 2 ** 20, 2) == mib


def test_stale_weight_percentage_resnet110():
    """P:L75 definition; stage 0 of ResNet-110 PPV (37) = conv1+BN + 18 group-1 blocks."""
    stage0 = (16 * 3 * 9 + 32) + 18 * 2 * (16 * 16 * 9 + 32)
    pct = Net.stale_weight_percentage(W.resnet_cifar(110).layers, (37,))
    assert abs(pct - 100.0 * stage0 / 1727962) < 1e-12
    assert round(pct, 2) == 4.89


def test_speedup_formulas():
    assert Pl.ideal_speedup_paper(1) == 3                      # P:L77 with K=1 pair
    assert abs(Pl.hybrid_speedup(200, 100, 2) - 4.0 / 3.0) < 1e-12   # 1.33 bound
    assert abs(Pl.hybrid_speedup_bound(200, 100) - 2.0) < 1e-12
    # Table 5: printed speedups equal the time ratios.
    for tn, tp, sp in [(2421, 1974, 1.23), (6745, 4090, 1.65), (13150, 7570, 1.73),
                       (27231, 14998, 1.81), (44814, 24640, 1.82)]:
        assert abs(tn / tp - sp) < 0.01


@pytest.mark.parametrize("name,K", [("tiny_resnet", 1), ("tiny_resnet", 2), ("tiny_resnet", 3), ("tiny_cnn", 4),
                                    ("tiny_resnet2_mid", 3)])
def test_fs_bks_mapping_equals_versioned(name, K):
    """Oracle C (the paper's 2K_p+1-accelerator mapping; SURVEY f-4) against Oracle A:
    bitwise equal losses and weights (the mapping moves work between accelerators, not the math),
    and the forward-version log equals the closed form of P:L75."""
    if name == "tiny_resnet2_mid":
        net, B, ppv = W.tiny_resnet(width=4, hw=8, n=2), 6, (2, 6)
    else:
        net, B, ppvs = NETS[name]
        ppv = ppvs[K]
    flat = W.init_params(net, seed=21)
    data = W.batches(net.in_shape, B, 9, seed=22)
    sa, bounds = make_stages(net, ppv)
    sc, _ = make_stages(net, ppv)
    p0 = split_params(net, flat, bounds)
    hp = hp_for(K)
    ra = Pl.run_versioned(sa, p0, data, hp)
    rc = Pl.run_fs_bks(sc, p0, data, hp)
    assert ra.losses == rc.losses
    assert np.array_equal(flat_of(net, bounds, ra.params), flat_of(net, bounds, rc.params))
    for t, s, kind, mb, ver in rc.version_log:
        if kind == "F":
            assert ver == max(0, mb - 2 * (K - 1 - s)), (t, s, mb, ver)
        if kind == "B":
            assert ver == mb
    # 2K-1 accelerators busy in the steady state: per cycle K forwards and K backwards, the last
    # stage doing both of the same mini-batch
    per_t = {}
    for t, s, kind, mb, ver in rc.version_log:
        per_t.setdefault(t, []).append((s, kind))
    mid = per_t[2 * K]
    assert sorted(mid) == sorted([(s, "F") for s in range(K)] + [(s, "B") for s in range(K)]) if len(data) > 2 * K else True
