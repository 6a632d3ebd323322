"""Profile-driven partition balancer.

The paper places its pipeline registers by hand and notes that the early layers dominate the
runtime; the stage time of a K-GPU pipeline is the time of its slowest stage, so
the speedup is bounded by sum(costs) / (K * max stage cost).  Given the measured cost of every
weighted layer (forward + backward + update work on the B200, see b200_costs.json) this module
finds the partition-point vector (PPV) that minimises the maximum stage cost over the
allowed boundaries by dynamic programming -- host logic only, no method arithmetic.  Since round 2
every layer boundary is allowed, including points inside a residual block (two-tensor registers,
SURVEY f-2, reading AMB-14).
"""
from __future__ import annotations

import functools
import json
import os
from typing import Dict, List, Sequence, Tuple

from .nets import NetSpec, weighted_layer_count

_HERE = os.path.dirname(os.path.abspath(__file__))


def load_cost_table(path: str = os.path.join(_HERE, "b200_costs.json")) -> Dict:
    with open(path) as f:
        return json.load(f)


def resnet_layer_costs(net: NetSpec, table: Dict) -> List[float]:
    """Cost (us) of each weighted layer 1..L of a CIFAR ResNet-(6n+2) from the measured table:
    index 0 is unused so that costs[l] is weighted layer l (the PPV numbering)."""
    L = weighted_layer_count(net)
    n = (L - 2) // 6
    t = table["resnet_cifar_b128"]
    c = [0.0] * (L + 1)
    c[1] = t["conv1"]
    for l in range(2, L):
        g = 0 if l < 2 + 2 * n else (1 if l < 2 + 4 * n else 2)
        first_of_group = l in (2 + 2 * n, 2 + 4 * n)       # the stride-2 conv opening groups 2, 3
        c[l] = t["stride2"][g - 1] if first_of_group else t["group"][g]
    c[L] = t["head"]
    return c


def resnet_block_boundaries(net: NetSpec) -> List[int]:
    """PPV entries of an option-A ResNet between residual blocks: after the first conv or after a
    block (odd weighted-layer numbers 1 + 2k below L)."""
    L = weighted_layer_count(net)
    return [p for p in range(1, L) if p % 2 == 1]


def resnet_boundaries(net: NetSpec) -> List[int]:
    """Allowed PPV entries: every weighted layer 1..L-1 (mid-block points carry the block input
    too, SURVEY f-2, reading AMB-14; every block of these nets has two layers, so a partition has
    at most one point inside any block)."""
    return list(range(1, weighted_layer_count(net)))


def stage_costs(costs: Sequence[float], ppv: Sequence[int]) -> List[float]:
    L = len(costs) - 1
    b = [0] + list(ppv) + [L]
    return [float(sum(costs[b[i] + 1:b[i + 1] + 1])) for i in range(len(b) - 1)]


def balance_efficiency(costs: Sequence[float], ppv: Sequence[int]) -> float:
    """sum of stage costs / (K * max stage cost): the fraction of the ideal K-fold speedup the
    partition allows."""
    st = stage_costs(costs, ppv)
    return sum(st) / (len(st) * max(st))


def balance_ppv(costs: Sequence[float], K: int, allowed: Sequence[int]) -> Tuple[int, ...]:
    """Min-max contiguous partition of weighted layers 1..L into K stages with boundaries from
    `allowed` (ties: the lexicographically smallest PPV)."""
    L = len(costs) - 1
    if K == 1:
        return ()
    pre = [0.0]
    for l in range(1, L + 1):
        pre.append(pre[-1] + float(costs[l]))
    allowed = sorted(p for p in set(allowed) if 1 <= p < L)

    @functools.lru_cache(maxsize=None)
    def best(start: int, k: int):
        if k == 1:
            return pre[L] - pre[start - 1], ()
        res = (float("inf"), ())
        for p in allowed:
            if p < start:
                continue
            left = pre[p] - pre[start - 1]
            if left >= res[0]:
                break                          # costs are non-negative: later p only grow `left`
            sub, rest = best(p + 1, k - 1)
            m = max(left, sub)
            if m < res[0]:
                res = (m, (p,) + rest)
        return res

    m, ppv = best(1, K)
    if len(ppv) != K - 1:
        raise ValueError(f"no {K}-stage partition with boundaries {allowed}")
    return ppv
