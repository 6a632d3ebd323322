"""Measured per-stage step times of the ResNet-110 b128 pipeline (pst_stage_timing): all K stages
in one process on one GPU, serialised within each step so each stage's device time is measured
alone.  On K GPUs every stage runs on its own device, so max(stage time) is the projected K-GPU
step time before the NVLink exchange; sum/K1 shows the per-stage fixed overhead.  A projection
from measured kernel times, not a multi-GPU measurement.
usage (GPU box): python tools/stage_times.py [steps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pst_workloads as W
import paper_1912_12675_b200 as pst

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = W.CONFIGS["resnet110"]
net = cfg.netspec()
params = W.init_params(net, seed=42)
B = cfg.batch
dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
       for x, y in (W.make_batch(net.in_shape, B, i, seed=1234) for i in range(8))]
k1 = None
for K in (1, 2, 4, 8):
    pipe = pst.Pipeline(net, params, cfg.ppv[K], B, cfg.lr_vector(K), cfg.base_lr, momentum=cfg.momentum,
                        weight_decay=cfg.weight_decay)
    for i in range(4 * K + 20):
        pipe.step(*dev[i % 8])
    pipe.sync()
    pipe.stage_timing(True)
    for i in range(steps):
        pipe.step(*dev[i % 8])
    ms, n = pipe.stage_times()
    pipe.stage_timing(False)
    per = (ms / max(1, n)).tolist()
    k1 = per[0] if K == 1 else k1
    mx = max(per)
    print(json.dumps({"K": K, "ppv": list(cfg.ppv[K]), "stage_ms": [round(x, 4) for x in per],
                      "max_stage_ms": round(mx, 4), "sum_stage_ms": round(sum(per), 4),
                      "projected_speedup_vs_k1": round(k1 / mx, 3), "projected_fraction_of_ideal": round(k1 / mx / K, 3),
                      "note": "per-stage device time measured alone on one GPU; excludes the NVLink exchange"}),
          flush=True)
    pipe.close()
