"""Pipeline parity (GPU): libpst.so's stale-weight pipelined training against the
oracle's schedule (Oracle B), step by step, on identical seeded inputs.

Every K-stage configuration here runs all stages on cuda:0 ("local" mode: the
same scheduler and stage programs as the multi-GPU path; transfers are device
copies instead of NCCL).  Checked after EVERY pipeline step: each parameter
tensor within 2e-3 relative (inf-norm) and every mini-batch loss within 1e-2
(BASELINE.json north_star tolerances, reading AMB-21), plus the stage version
counters against the closed form.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import pst_workloads as W
from tests.parity import L_TOL, W_TOL, run_both

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pst():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_12675_b200 as p
    return p


@pytest.mark.parametrize("K,ppv", [(1, ()), (2, (3,)), (3, (1, 3))])
def test_tiny_resnet_pipeline(pst, K, ppv):
    net = W.tiny_resnet(width=16, hw=8, n=1)
    P = run_both(pst, net, ppv, 32, 8, [0.05] * (K - 1) + [0.1]).assert_ok()
    assert list(P.versions) == [8] * K


@pytest.mark.parametrize("K,ppv", [(1, ()), (2, (2,)), (4, (1, 2, 3))])
def test_tiny_cnn_pipeline(pst, K, ppv):
    net = W.tiny_cnn(hw=8)
    run_both(pst, net, ppv, 32, 8, [0.05] * K, wd=5e-4).assert_ok()


def test_lenet5_config1_k2(pst):
    """BASELINE.json configs[0]: LeNet-5, MNIST-shaped, batch 64, 2 stages, 20 steps."""
    cfg = W.CONFIGS["lenet5"]
    run_both(pst, W.lenet5(), cfg.ppv[2], 64, 20, cfg.lr_vector(2), mom=cfg.momentum,
             wd=cfg.weight_decay).assert_ok()


def test_hybrid_switch(pst):
    """pipelined for n_p mini-batches, drain, then non-pipelined (AMB-10)."""
    net = W.tiny_resnet(width=16, hw=8, n=1)
    P = run_both(pst, net, (1, 3), 32, 9, [0.02, 0.05, 0.1], lr_np=0.08, n_p=4, spe=2,
                 milestones=(3,)).assert_ok()
    assert list(P.versions) == [9, 9, 9]


def test_distributed_mode_single_rank(pst):
    """The one-process-per-GPU code path (pst_dist: ncclCommInitRank, the eager neighbour
    warm-up, the per-rank step program) with world size 1 on cuda:0: it must train exactly like
    local mode and the oracle (more ranks need more GPUs than this box has; the message pattern
    of K > 1 is checked over gloo in test_dist_gloo.py)."""
    import numpy as np
    from oracle import network as Net
    from tests.parity import hparams, oracle_run, flat_params, tensor_errors, loss_errors
    net = W.tiny_resnet(width=16, hw=8, n=1)
    flat = W.init_params(net, seed=11)
    data = W.batches(net.in_shape, 32, 6, seed=12)
    ref = oracle_run(net, flat, (), data, hparams([0.05], 1, 0.05, 0.9, 1e-4))
    pipe = pst.Pipeline(net, flat, (), 32, [0.05], 0.05, momentum=0.9, weight_decay=1e-4, devices=[0], rank=0,
                        nccl_id=pst.nccl_unique_id())
    for x, y in data:
        pipe.step(x, y)
    pipe.flush()
    e = tensor_errors(net, pipe.weights(), flat_params(net, ref.params))
    assert e[0] <= W_TOL, e
    assert loss_errors(pipe.losses(0, 6), ref.losses) <= L_TOL
    pipe.close()


@pytest.mark.parametrize("skw,ppv", [
    (dict(solver="caffe", lr_policy="inv", inv_gamma=1e-4, inv_power=0.75), (2,)),   # LeNet-5's (L284)
    (dict(solver="caffe", nesterov=True), (1, 2, 3)),                                  # AlexNet/VGG (L286-288)
    (dict(nesterov=True), (2,)),                                                        # PyTorch Nesterov
])
def test_solver_variants(pst, skw, ppv):
    """The paper's Caffe-simulated solver settings through the GPU update
    kernel, pipelined, against the oracle's solver of the same form; lr milestones change the rate
    mid-run so the Caffe form (lr folded into the history) differs from the PyTorch form."""
    net = W.tiny_cnn(hw=8)
    K = len(ppv) + 1
    run_both(pst, net, ppv, 32, 10, [0.05] * K, wd=5e-4, milestones=(2,), spe=3, solver_kw=skw).assert_ok()


def test_lenet5_paper_solver_k2(pst):
    """configs[0] with the paper's own LeNet-5 solver: Caffe SGD, momentum 0.9, wd 5e-4, lr 0.01
    with the "inv" policy (L284; gamma 1e-4 / power 0.75, Caffe's LeNet values, external), 2 stages."""
    cfg = W.CONFIGS["lenet5"]
    run_both(pst, W.lenet5(), cfg.ppv[2], 64, 20, cfg.lr_vector(2), mom=cfg.momentum, wd=cfg.weight_decay,
             solver_kw=dict(solver="caffe", lr_policy="inv", inv_gamma=1e-4, inv_power=0.75)).assert_ok()


def test_abi_error_behaviour(pst):
    """include/pst.h's error contract on a live context: invalid arguments return PST_E_INVALID
    without poisoning the context, losses beyond what was fed / a cap that is too small are
    reported, and the size query (out = NULL) returns the block size."""
    import ctypes as C
    import numpy as np
    from paper_1912_12675_b200 import binding as Bd
    L = Bd.lib()
    net = W.tiny_cnn(hw=8)
    flat = W.init_params(net, seed=3)
    with pytest.raises(Bd.PstError) as e:                   # batch out of range
        pst.Pipeline(net, flat, (), 0, [0.1], 0.1)
    assert e.value.code == -1
    with pytest.raises(Bd.PstError):                        # PPV not increasing
        pst.Pipeline(net, flat, (2, 1), 8, [0.1] * 3, 0.1)
    n_s, keep = Bd.net_struct(net, flat)                    # solver enum out of range
    part, keep_p = Bd._partition([], None)
    lrs = (C.c_float * 1)(0.1)
    ms = (C.c_int64 * 1)(0)
    hp = Bd._HParams(8, 0.9, 0.0, C.cast(lrs, C.POINTER(C.c_float)), 0.1, 0, C.cast(ms, C.POINTER(C.c_int64)),
                     0.1, 1 << 62, 7, 0, 0, 0.0, 0.0)
    assert L.pst_create(C.byref(n_s), C.byref(part), C.byref(hp), None, C.byref(C.c_void_p())) == -1
    assert L.pst_create(None, None, None, None, C.byref(C.c_void_p())) == -1
    pipe = pst.Pipeline(net, flat, (), 8, [0.1], 0.1)
    x, y = W.make_batch(net.in_shape, 8, 0, seed=1)
    pipe.step(x, y)
    n = C.c_int64()
    assert L.pst_weights(pipe._ctx, 1, None, 0, C.byref(n)) == 0 and n.value == flat.size   # size query
    small = np.empty(4, dtype=np.float32)
    rc = L.pst_weights(pipe._ctx, 1, small.ctypes.data_as(C.POINTER(C.c_float)), 4, C.byref(n))
    assert rc == -1 and n.value == flat.size                # cap too small: INVALID, size reported
    out = np.empty(4, dtype=np.float32)
    rc = L.pst_losses(pipe._ctx, 5, 1, out.ctypes.data_as(C.POINTER(C.c_float)))
    assert rc == -5                                         # mini-batch 5 was never fed: PST_E_STATE
    assert L.pst_step(pipe._ctx, None) == -1                # null batch
    pipe.step(x, y)                                         # the context is not poisoned
    pipe.flush()
    assert list(pipe.versions()) == [2]
    pipe.close()


@pytest.mark.parametrize("K,ppv", [(1, ()), (2, (1,)), (4, (1, 2, 3))])
def test_dropout_pipeline(pst, K, ppv):
    """Dropout (SURVEY f-3; VGG-16's "batch normalization and dropout") with the counter-based
    masks both sides generate from one definition (pst.h pst_layer.dropout, reading AMB-16b): a conv
    layer with dropout before its max-pool and a hidden FC with dropout, pipelined."""
    net = W.tiny_cnn(hw=8, dropout=0.4)
    P = run_both(pst, net, ppv, 32, 9, [0.05] * K, wd=5e-4, dropout_seed=1234567).assert_ok()
    assert list(P.versions) == [9] * K


def test_dropout_hybrid(pst):
    net = W.tiny_cnn(hw=8, dropout=0.3)
    run_both(pst, net, (2,), 32, 9, [0.05, 0.05], lr_np=0.03, n_p=4, spe=2, wd=5e-4,
             dropout_seed=99).assert_ok()
