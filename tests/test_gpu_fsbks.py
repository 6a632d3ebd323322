"""The paper's 2K_p+1-accelerator mapping on the GPU (include/pst.h PST_MAP_FS_BKS).

PAPER.md L59-L77 (section 3, Fig. 3/4): the forward stage FS_s and the backward stage BKS_s of every
stage but the last run on separate accelerators ("In total 2K+1 accelerators are used", L67; the
potential speedup 2K+1, L77); each cycle BKS_s forwards its new weights to FS_s and FS_s hands the
saved activations to BKS_s (L65); the last stage's FS and BKS share one accelerator (L67).  libpst
runs each FS and BKS as its own stage object with its own stream (local mode; here all 2K-1 on
cuda:0).  The weight versions are those of the per-GPU mapping (Oracle C == Oracle A bitwise,
tests/test_oracle_pipeline.py), so the final weights, momentum, BN running statistics and every loss
are compared with Oracle B after the drain.
"""
import pytest

torch = pytest.importorskip("torch")

import pst_workloads as W
from tests.parity import run_both

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pst():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_12675_b200 as p
    return p


FSBKS = dict(mapping=1)


@pytest.mark.parametrize("K,ppv", [(1, ()), (2, (3,)), (3, (1, 3))])
def test_fsbks_tiny_resnet(pst, K, ppv):
    net = W.tiny_resnet(width=16, hw=8, n=1)
    P = run_both(pst, net, ppv, 32, 9, [0.05] * (K - 1) + [0.1], per_step=False, deep=True,
                 solver_kw=FSBKS).assert_ok()
    assert list(P.versions) == [9] * K


def test_fsbks_tiny_cnn_k4(pst):
    run_both(pst, W.tiny_cnn(hw=8), (1, 2, 3), 32, 10, [0.05] * 4, wd=5e-4, per_step=False,
             solver_kw=FSBKS).assert_ok()


def test_fsbks_midblock(pst):
    net = W.tiny_resnet(width=16, hw=8, n=2)
    run_both(pst, net, (2, 6), 32, 9, [0.005, 0.005, 0.01], per_step=False, deep=True,
             solver_kw=FSBKS).assert_ok()


def test_fsbks_resnet20_paper_ppv(pst):
    """ResNet-20 with the paper's 4-stage PPV (5,12,17): 7 accelerators' worth of stage
    objects (FS_0..FS_3, BKS_0..BKS_2)."""
    P = run_both(pst, W.nets.by_name("resnet20"), (5, 12, 17), 32, 12, [0.001] * 4, per_step=False, deep=True,
                 solver_kw=FSBKS).assert_ok()
    assert list(P.versions) == [12] * 4


def test_fsbks_rejects_hybrid_and_dist(pst):
    net = W.tiny_cnn(hw=8)
    flat = W.init_params(net, seed=1)
    p = pst.Pipeline(net, flat, (2,), 8, [0.1, 0.1], 0.1, mapping=1)
    with pytest.raises(pst.PstError) as e:
        p.set_hybrid(1)
    assert e.value.code == -6
    p.close()
    with pytest.raises(pst.PstError) as e:
        pst.Pipeline(net, flat, (2,), 8, [0.1, 0.1], 0.1, mapping=1, rank=0, nccl_id=pst.nccl_unique_id())
    assert e.value.code in (-6, -1)


def test_fsbks_dropout(pst):
    """Dropout under the FS/BKS mapping: the forward objects draw the masks, the backward objects
    receive the post-dropout activations with the saved state."""
    run_both(pst, W.tiny_cnn(hw=8, dropout=0.4), (1, 2), 32, 9, [0.05] * 3, wd=5e-4, per_step=False,
             solver_kw=FSBKS, dropout_seed=4242).assert_ok()
