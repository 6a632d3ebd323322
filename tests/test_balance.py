"""Profile-driven PPV balancer (pst_workloads/balance.py) -- host logic, CPU."""
import itertools

import numpy as np
import pytest

import pst_workloads as W
from pst_workloads import balance as Bl


def _brute(costs, K, allowed):
    L = len(costs) - 1
    best = (float("inf"), None)
    for ppv in itertools.combinations(sorted(p for p in allowed if 1 <= p < L), K - 1):
        m = max(Bl.stage_costs(costs, ppv))
        if m < best[0] - 1e-12:
            best = (m, ppv)
    return best


@pytest.mark.parametrize("seed", range(12))
def test_dp_matches_brute_force(seed):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(5, 13))
    costs = [0.0] + list(rng.uniform(0.1, 5.0, L))
    allowed = list(range(1, L)) if seed % 2 else [p for p in range(1, L) if p % 2 == 1]
    for K in (2, 3, 4):
        if K - 1 > len([p for p in allowed if p < L]):
            continue
        ppv = Bl.balance_ppv(costs, K, allowed)
        m, ref = _brute(costs, K, allowed)
        assert max(Bl.stage_costs(costs, ppv)) == pytest.approx(m)


def test_uniform_costs_split_evenly():
    costs = [0.0] + [1.0] * 12
    assert Bl.balance_ppv(costs, 4, range(1, 12)) == (3, 6, 9)
    assert Bl.balance_efficiency(costs, (3, 6, 9)) == pytest.approx(1.0)


@pytest.mark.parametrize("name", ["resnet110", "resnet362"])
def test_config_ppvs_are_the_balanced_ones(name):
    """The bench/parity PPVs of ResNet-110/362 are the balancer's output on the measured table,
    valid block boundaries, and at least as balanced as the paper's hand placement (Table 5)."""
    cfg = W.CONFIGS[name]
    net = cfg.netspec()
    costs = Bl.resnet_layer_costs(net, Bl.load_cost_table())
    allowed = Bl.resnet_boundaries(net)
    for K, ppv in cfg.ppv.items():
        if K == 1:
            continue
        assert tuple(ppv) == Bl.balance_ppv(costs, K, allowed), (K, ppv)
        assert all(p in allowed for p in ppv)
        # allowing mid-block points never balances worse than block boundaries alone
        blk = Bl.balance_ppv(costs, K, Bl.resnet_block_boundaries(net))
        assert Bl.balance_efficiency(costs, ppv) >= Bl.balance_efficiency(costs, blk) - 1e-12
    for K, ppv in cfg.paper_ppv.items():
        assert Bl.balance_efficiency(costs, cfg.ppv[K]) >= Bl.balance_efficiency(costs, ppv)


def test_resnet110_balance_numbers():
    net = W.nets.by_name("resnet110")
    costs = Bl.resnet_layer_costs(net, Bl.load_cost_table())
    assert len(costs) == 111
    assert Bl.balance_efficiency(costs, (45,)) > 0.95 > Bl.balance_efficiency(costs, (37,))
    assert Bl.balance_efficiency(costs, W.CONFIGS["resnet110"].ppv[8]) > 0.9
