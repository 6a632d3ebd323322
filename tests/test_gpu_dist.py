"""Distributed-mode parity (GPU): libpst.so with one PROCESS per pipeline stage and NCCL
send/recv between neighbouring stages (include/pst.h `pst_dist`; section 5 -- the
paper's stages exchange activations and gradients between devices every cycle; L183 section 6.5 --
one stage pair per GPU), against the oracle's schedule (Oracle B).

The GPU box this suite runs on has ONE B200, so the K ranks share cuda:0.  NCCL refuses two ranks
of one communicator on the same device of the same host ("Duplicate GPU detected"), so each rank
gets its own NCCL_HOSTID: NCCL then treats the ranks as separate hosts and moves the messages over
its socket transport on the loopback interface.  Everything libpst does is the multi-GPU code path
unchanged -- ncclCommInitRank, the eager neighbour warm-up, the grouped ncclSend/ncclRecv captured
in each rank's step graphs, the non-pipelined (hybrid) exchange, per-rank weights and losses --
only NCCL's transport underneath differs from NVLink.

Checked after the drain, per rank: every parameter tensor, the momentum buffers and the BatchNorm
running statistics of that rank's stage, its version counter, and (last rank) every mini-batch's
loss.
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import pst_workloads as W
from oracle import network as Net
from tests.parity import (K_EMU, K_SPREAD, Parity, allowances, compare_final, hparams, oracle_run, oracle_spreads,
                          perturbed)

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_12675_b200 as p
    p.lib()
    return p


def _launch(case, timeout=900):
    K = len(case["ppv"]) + 1
    work = tempfile.mkdtemp(prefix="pst_dist_")
    cpath = os.path.join(work, "case.json")
    json.dump(case, open(cpath, "w"))
    procs = []
    for r in range(K):
        env = dict(os.environ)
        env.update(NCCL_HOSTID=f"pst-test-rank{r}", NCCL_SOCKET_IFNAME="lo", NCCL_IB_DISABLE="1",
                   NCCL_DEBUG=env.get("NCCL_DEBUG", "WARN"), PYTHONPATH=ROOT)
        log = open(os.path.join(work, f"rank{r}.log"), "w")
        procs.append((subprocess.Popen([sys.executable, "-m", "tests.dist_worker", str(r), str(K), work, cpath],
                                       cwd=ROOT, env=env, stdout=log, stderr=subprocess.STDOUT,
                                       start_new_session=True), log))
    failed = []
    for r, (p, log) in enumerate(procs):
        try:
            rc = p.wait(timeout=timeout)
        except subprocess.TimeoutExpired:
            for q, _ in procs:
                try:
                    os.killpg(q.pid, 9)
                except Exception:
                    pass
            rc = "timeout"
        log.close()
        if rc != 0:
            failed.append((r, rc, open(os.path.join(work, f"rank{r}.log")).read()[-3000:]))
    assert not failed, failed
    return [dict(np.load(os.path.join(work, f"rank{r}.npz"))) for r in range(K)], work


def _local(gpu, case, net, flat, data):
    """The same case in local mode (all stages in this process): the distributed run must reproduce
    it up to the run-to-run rounding of the fp64 atomics in the BN-statistics reduction."""
    ppv = tuple(case["ppv"])
    pipe = gpu.Pipeline(net, flat, ppv, case["B"], case["lr"], case.get("lr_np", case["lr"][-1]),
                        momentum=case.get("mom", 0.9), weight_decay=case.get("wd", 1e-4),
                        milestones=case.get("milestones", ()), steps_per_epoch=case.get("spe", 1 << 62),
                        dropout_seed=case.get("dropout_seed", 0))
    if case.get("n_p") is not None:
        pipe.set_hybrid(case["n_p"] // case["spe"])
    for x, y in data:
        pipe.step(x, y)
    pipe.flush()
    out = pipe.weights(gpu.W_PARAMS | gpu.W_MOMENTUM | gpu.W_BNSTATS), pipe.losses(0, case["N"])
    pipe.close()
    return out


def _check(gpu, case, tag):
    net = getattr(W, case["net"])(**case.get("net_kw", {}))
    ppv = tuple(case["ppv"])
    K = len(ppv) + 1
    flat = W.init_params(net, seed=case["seed"])
    data = W.batches(net.in_shape, case["B"], case["N"], seed=case["seed"] + 100)
    hp = hparams(case["lr"], K, case.get("lr_np", case["lr"][-1]), case.get("mom", 0.9), case.get("wd", 1e-4),
                 case.get("milestones", ()), 0.1, case.get("spe", 1 << 62))
    ds = case.get("dropout_seed", 0)
    ref = oracle_run(net, flat, ppv, data, hp, n_p=case.get("n_p"), dropout_seed=ds)
    sp_p = oracle_spreads(net, ppv, ref, oracle_run(net, perturbed(flat), ppv, data, hp, n_p=case.get("n_p"),
                                                      dropout_seed=ds))
    sp_e = oracle_spreads(net, ppv, ref, oracle_run(net, flat, ppv, data, hp, n_p=case.get("n_p"), emu=True,
                                                      dropout_seed=ds))
    sp = allowances(sp_p, sp_e)
    got, work = _launch(case)
    for s in range(K):
        assert list(got[s]["versions"]) == [case["N"]], (s, got[s]["versions"])
    # the ranks' stage blocks concatenated in stage order = the canonical network order
    g_p = np.concatenate([g["params"] for g in got])
    g_v = np.concatenate([g["momentum"] for g in got])
    g_bn = np.concatenate([g["bnstats"] for g in got])
    P = Parity(tag)
    compare_final(P, net, ppv, g_p, g_v, g_bn, got[K - 1]["losses"], ref, deep=case.get("deep", False), sp=sp)
    P.extra.update(spread_final_max=max(sp_p["w"].values()), emu_dev_momentum_max=max(sp_e["vs"].values()),
                   k_spread=K_SPREAD, k_emu=K_EMU)
    # distributed vs local mode on the same GPU: same kernels, same inputs
    loc, loc_loss = _local(gpu, case, net, flat, data)
    mine = np.concatenate([g_p, g_v, g_bn])
    d_local = float(np.abs(mine - loc).max() / max(np.abs(loc).max(), 1e-12))
    dl_local = float(np.abs(got[K - 1]["losses"] - loc_loss).max())
    P.extra.update(dist_vs_local_state_rel=d_local, dist_vs_local_loss_abs=dl_local,
                   transport="NCCL socket (the ranks share cuda:0)", K=K, N=case["N"])
    P.assert_ok()
    assert d_local <= 1e-5 and dl_local <= 1e-5, (d_local, dl_local)


def test_dist_k2_tiny_resnet(gpu):
    """Two ranks, PPV (3): pipelined fill, steady state and drain over NCCL."""
    _check(gpu, dict(net="tiny_resnet", net_kw=dict(width=16, hw=8, n=1), ppv=[3], B=32, N=8, seed=21,
                lr=[0.05, 0.1], deep=True), "dist_k2_tiny_resnet")


def test_dist_k3_hybrid(gpu):
    """Three ranks with the hybrid switch (reading AMB-10): pipelined for 4 mini-batches,
    drain, then the non-pipelined exchange (ungrouped send/recv per mini-batch), lr milestone."""
    _check(gpu, dict(net="tiny_resnet", net_kw=dict(width=16, hw=8, n=1), ppv=[1, 3], B=32, N=9, seed=23,
                lr=[0.02, 0.05, 0.1], lr_np=0.08, n_p=4, spe=2, milestones=[3], deep=True), "dist_k3_hybrid")


def test_dist_k4_tiny_cnn(gpu):
    """Four ranks (every interior rank sends and receives in both directions every step)."""
    _check(gpu, dict(net="tiny_cnn", net_kw=dict(hw=8), ppv=[1, 2, 3], B=32, N=10, seed=25, lr=[0.05] * 4, wd=5e-4),
           "dist_k4_tiny_cnn")


def test_dist_k2_resnet110_b128(gpu):
    """bench.py's 2-GPU workload through the distributed path: ResNet-110, batch 128, the balanced
    PPV (45), Table 7's rate vector [0.001, 0.1]; 4 mini-batches (mini-batch 3's stage-0
    forward reads a stale version).  Deep BN net: beta per stage (AMB-21b)."""
    cfg = W.CONFIGS["resnet110"]
    _check(gpu, dict(net="resnet_cifar", net_kw=dict(depth=110), ppv=list(cfg.ppv[2]), B=128, N=4, seed=31,
                     lr=cfg.lr_vector(2), wd=cfg.weight_decay, deep=True), "dist_k2_resnet110_b128")


def test_dist_k3_midblock(gpu):
    """Mid-block registers over NCCL (reading AMB-14): the block input travels beside the
    activation and the shortcut gradient beside the input gradient; PPV (2, 6) of a two-block-per-
    group tiny ResNet splits a plain block and an option-A block.  Then the hybrid switch."""
    _check(gpu, dict(net="tiny_resnet", net_kw=dict(width=16, hw=8, n=2), ppv=[2, 6], B=32, N=9, seed=27,
                     lr=[0.002, 0.005, 0.01], lr_np=0.008, n_p=4, spe=2, milestones=[3], deep=True),
           "dist_k3_midblock_hybrid")


def test_dist_k2_dropout(gpu):
    """Dropout across processes: each rank's stage draws its masks from the shared counter-based
    generator with its own forward counter (pst.h pst_layer.dropout, reading AMB-16b)."""
    _check(gpu, dict(net="tiny_cnn", net_kw=dict(hw=8, dropout=0.4), ppv=[1], B=32, N=9, seed=29, lr=[0.05] * 2,
                     wd=5e-4, dropout_seed=777), "dist_k2_dropout")
