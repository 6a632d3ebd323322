#!/usr/bin/env python3
"""Writes tests/golden/scalar_pipeline_k{2,3}.json: the paper's stale-weight schedule on a chain of
K scalar "layers", computed by a closed-form recursion written here from the paper -- it imports
nothing from oracle/ (or from the CUDA path), so the oracle can be checked against it.

Net: h_0 = x; h_{s+1} = w_s * h_s for stage s = 0..K-1; loss = 0.5 * h_K^2; x = 1 every mini-batch.
Schedule (section 3): the forward of mini-batch i through stage s reads weight version
max(0, i - 2(K-1-s)) -- "weights that are 2 execution cycles old" for K_p = 1 (L63), degree of
staleness 2(K_p - i + 1) in general (L75), versions clamped at 0 while the pipe fills (reading
AMB-11); the backward of mini-batch i uses the CURRENT weights w_s^(i) (no stash, L35/L236,
reading AMB-2) and the activations its own forward produced (L65).  Update: PyTorch SGD with
momentum (reading AMB-7), v <- mu v + (g + lambda w), w <- w - lr v.
Non-pipelined (L43-49): every stage reads w_s^(i) in the forward.

    python tools/make_golden_scalar.py          # rewrites the JSON files
    python tools/make_golden_scalar.py --check  # exit 1 if the files differ from a fresh run
"""
from __future__ import annotations

import json
import os
import sys

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def chain(K, N, lr, mu, wd, pipelined):
    w = [[1.0] for _ in range(K)]      # w[s][v] = version v of stage s's weight
    vel = [0.0] * K
    losses = []
    for i in range(N):
        # forward of mini-batch i: activations h_0..h_K with the versions the schedule reads
        h = [1.0]
        for s in range(K):
            ver = max(0, i - 2 * (K - 1 - s)) if pipelined else i
            h.append(w[s][ver] * h[s])
        losses.append(0.5 * h[K] * h[K])
        # backward of mini-batch i with the current weights w_s^(i), then the update -> w_s^(i+1)
        delta = h[K]                       # d loss / d h_K
        for s in range(K - 1, -1, -1):
            cur = w[s][i]
            g = delta * h[s]               # d loss / d w_s (saved forward activation h_s)
            delta = delta * cur            # d loss / d h_s through the current weight
            vel[s] = mu * vel[s] + (g + wd * cur)
            w[s].append(cur - lr * vel[s])
    return losses, [ws[1:] for ws in w]


CASES = {
    "scalar_pipeline_k2.json": dict(K=2, N=5, lr=0.1, mu=0.0, wd=0.0),
    "scalar_pipeline_k3_momentum.json": dict(K=3, N=8, lr=0.05, mu=0.9, wd=0.01),
}


def build(name):
    c = CASES[name]
    pl, pw = chain(c["K"], c["N"], c["lr"], c["mu"], c["wd"], True)
    nl, nw = chain(c["K"], c["N"], c["lr"], c["mu"], c["wd"], False)
    return {
        "citation": "PAPER.md section 3 L61 (cycle timeline), L63 ('weights that are 2 execution cycles old'), "
                    "L75 (degree of staleness 2(K_p-i+1)); readings AMB-1/2/7/11.  Written by "
                    "tools/make_golden_scalar.py (closed-form scalar recursion; imports nothing from oracle/).",
        "net": f"chain of {c['K']} scalars h_(s+1) = w_s h_s, h_0 = x = 1, loss = 0.5 h_K^2",
        "init": {"w": [1.0] * c["K"]},
        "hparams": {"lr": c["lr"], "momentum": c["mu"], "weight_decay": c["wd"], "K": c["K"]},
        "pipelined": {"loss": pl, "w_after": pw},
        "nonpipelined": {"loss": nl, "w_after": nw},
        "atol": 1e-12,
    }


def main():
    check = "--check" in sys.argv
    bad = 0
    for name in CASES:
        data = build(name)
        path = os.path.join(GOLDEN, name)
        if check:
            if json.load(open(path)) != json.loads(json.dumps(data)):
                print("stale:", path)
                bad = 1
        else:
            with open(path, "w") as f:
                json.dump(data, f, indent=1)
                f.write("\n")
            print("wrote", path)
    return bad


if __name__ == "__main__":
    sys.exit(main())
