"""C-ABI checks that need no GPU: the library loads, exports every symbol the
headers declare, and its host-only logic (PPV validation, parameter counting,
schedule) agrees with the paper's closed forms and with the oracle."""
import os
import re

import numpy as np
import pytest

import pst_workloads as W
from oracle import network as Net
from oracle import pipeline as Pl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pst():
    import paper_1912_12675_b200 as p
    p.lib()
    return p


def _declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(pst_\w+)\s*\(", src)) - {"pst_status"}


def test_exports_every_declared_symbol(pst):
    L = pst.lib()
    names = _declared("pst.h") | _declared("pst_ops.h")
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert "sm_100a" in pst.build_info()


@pytest.mark.parametrize("name", ["lenet5", "alexnet", "vgg16", "resnet20", "resnet110", "resnet362"])
def test_param_count_matches_oracle(pst, name):
    net = W.by_name(name)
    assert pst.param_count(net) == Net.n_params(net.layers) == W.param_count(net)


def test_partition_ranges_match_oracle(pst):
    for name, ppvs in [("lenet5", [(1,), (1, 2, 3, 4)]), ("vgg16", [(2, 4, 7), (1, 2, 4, 6, 7, 9, 10)]),
                       ("resnet110", [(37,), (17, 33, 61), (9, 17, 25, 33, 45, 61, 81)]),
                       ("resnet362", [(121,), (27, 55, 81, 107, 147, 201, 265)]),
                       ("resnet20", [(5, 12, 17), (2,), (3, 5, 7, 9, 11, 13, 15, 17, 19)])]:   # mid-block, Table 3
        net = W.by_name(name)
        for ppv in ppvs:
            assert pst.partition_ranges(net, ppv) == Net.partition(net.layers, ppv)


def test_partition_rejections(pst):
    net = W.resnet_cifar(20)
    for bad, code in [((7, 7), -1), ((20,), -1), ((0,), -1), ((5, 4), -1)]:
        with pytest.raises(pst.PstError) as e:
            pst.partition_ranges(net, bad)
        assert e.value.code == code, (bad, e.value)


@pytest.mark.parametrize("K", [1, 2, 3, 4, 8])
def test_schedule_matches_closed_form(pst, K):
    n_total = 13
    for s in range(K):
        for t in range(n_total + 2 * K):
            b, f, v = pst.schedule(K, s, t, n_total)
            eb = t - 2 * K + 1 + s
            ef = t - s
            assert b == (eb if 0 <= eb < n_total else -1)
            assert f == (ef if 0 <= ef < n_total else -1)
            if f >= 0:
                assert v == Pl.forward_version(K, s, f)   # max(0, f - 2(K-1-s))


def test_nccl_unique_id(pst):
    a = pst.nccl_unique_id()
    assert len(a) == 128 and any(a)


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5, 8, 10])
def test_ring_slots(pst, K):
    """Saved-state rings hold at least the paper's 2(K-s)-1 mini-batches, input rings of
    stages s > 0 at least 2(K-s)+1 (the neighbour's copy of the next mini-batch lands while the stage
    still reads b..f), every size divides the graph-key period 2K+2, and each is the smallest such
    divisor (no memory beyond what the period forces)."""
    P = 2 * K + 2
    for s in range(K):
        saved, inp, period = pst.ring_slots(K, s)
        assert period == P and P % saved == 0 and P % inp == 0
        need_s = 2 * (K - s) - 1
        need_i = need_s if s == 0 else 2 * (K - s) + 1
        assert saved >= need_s and inp >= need_i
        assert all(P % d for d in range(need_s, saved))
        assert all(P % d for d in range(need_i, inp))
    assert pst.ring_slots(1, 0)[:2] == (1, 1)
    assert [pst.ring_slots(8, s)[0] for s in range(8)] == [18, 18, 18, 9, 9, 6, 3, 1]
