"""Diagnostic (not the BASELINE metric): ResNet-110 b128 trained as a K-stage pipeline with ALL
stages on one GPU ("local" mode: the same scheduler, stage graphs, rings and per-step boundary
transfers as the multi-GPU path, device copies instead of NCCL).  The GPU does the same total
work per step as K=1, so img/s close to the K=1 figure means the pipeline machinery (graph-key
selection, ring slots, boundary copies, per-stage streams and events) adds little overhead.
Prints one JSON line per K.   usage (GPU box): python tools/local_pipeline_bench.py [steps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pst_workloads as W
import paper_1912_12675_b200 as pst

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
cfg = W.CONFIGS["resnet110"]
net = cfg.netspec()
params = W.init_params(net, seed=42)
B = cfg.batch
host = [W.make_batch(net.in_shape, B, i, seed=1234) for i in range(8)]
dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()) for x, y in host]
for K in (1, 2, 4, 8):
    ppv = cfg.ppv[K]
    pipe = pst.Pipeline(net, params, ppv, B, cfg.lr_vector(K), cfg.base_lr, momentum=cfg.momentum,
                        weight_decay=cfg.weight_decay)
    for i in range(4 * K + 20):
        pipe.step(*dev[i % 8])
    pipe.sync()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        pipe.step(*dev[i % 8])
    pipe.sync()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(json.dumps({"K": K, "ppv": list(ppv), "ms_per_step": ms, "img_s": B / (ms / 1e3),
                      "mode": "local (all stages on one GPU)"}), flush=True)
    pipe.close()
