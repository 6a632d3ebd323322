"""Measure the per-layer cost table of pst_workloads/b200_costs.json on the B200 (profile-driven
PPV balancer): graph-replayed per-launch times of every distinct ResNet-CIFAR
conv shape at batch 128 (forward, dgrad, wgrad; tools/conv_lab.py's method) plus the in-graph
marginal BN costs measured with PST_SKIP (profiles/r1b_inGraph_skip_ms_per_step.txt).
usage (GPU box): python tools/measure_layer_costs.py > pst_workloads/b200_costs.json"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_12675_b200 import ops

N, IT = 128, 50
BN_APPLY_US, BN_BWD_US = 5.0, 3.5        # in-graph marginal cost per launch (0.54 / 0.38 ms over 109)
DILATE_US = 5.0                          # stride-2 dgrad: zero-insertion pass (launch list, r1b)
HEAD_US = 20.0                           # GAP + FC fwd/bwd + softmax-CE (launch list, r1b)


def t(which, Cin, H, Cout, S):
    return ops.time_conv(which, N, Cin, H, H, Cout, 3, S, 1, IT)


def layer(Cin, H, Cout, S=1, dgrad=True):
    # a stride-2 dgrad runs as a stride-1 correlation over the zero-inserted input grid
    f, d, w = t(0, Cin, H, Cout, S), (t(1, Cin, H, Cout, 1) if dgrad else 0.0), t(2, Cin, H, Cout, S)
    return f + d + w + BN_APPLY_US + BN_BWD_US + (DILATE_US if (S == 2 and dgrad) else 0.0)


table = {"resnet_cifar_b128": {
    "conv1": layer(3, 32, 16, dgrad=False),
    "group": [layer(16, 32, 16), layer(32, 16, 32), layer(64, 8, 64)],
    "stride2": [layer(16, 32, 32, S=2), layer(32, 16, 64, S=2)],
    "head": HEAD_US,
    "unit": "us per weighted layer per step (fwd + dgrad + wgrad + BN apply/backward)",
    "source": "tools/measure_layer_costs.py on B200 (graph-replayed launches, batch 128)"}}
print(json.dumps(table, indent=1))
