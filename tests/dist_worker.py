"""One rank of libpst's distributed mode (one process per pipeline stage, NCCL send/recv between
neighbouring stages, include/pst.h `pst_dist`), driven by tests/test_gpu_dist.py.

    python -m tests.dist_worker <rank> <world> <workdir> <case.json>

Rank 0 writes a fresh NCCL unique id to <workdir>/nccl_id; the other ranks wait for it.  Every
rank trains the case's seeded mini-batches through its own stage, drains the pipe, and writes
<workdir>/rank<r>.npz with its stage's parameters, momentum buffers, BatchNorm running statistics
and version counter (and, on the last rank, every mini-batch's loss).  No oracle arithmetic runs
here: the parent test compares these arrays with Oracle B.
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np


def main():
    rank, world, workdir, case_path = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    case = json.load(open(case_path))
    import paper_1912_12675_b200 as pst
    import pst_workloads as W

    net = getattr(W, case["net"])(**case.get("net_kw", {}))
    ppv = tuple(case["ppv"])
    K = len(ppv) + 1
    assert K == world, (K, world)
    flat = W.init_params(net, seed=case["seed"])
    data = W.batches(net.in_shape, case["B"], case["N"], seed=case["seed"] + 100)
    id_path = os.path.join(workdir, "nccl_id")
    if rank == 0:
        nid = pst.nccl_unique_id()
        with open(id_path + ".tmp", "wb") as f:
            f.write(nid)
        os.replace(id_path + ".tmp", id_path)
    else:
        t0 = time.time()
        while not os.path.exists(id_path):
            if time.time() - t0 > 120:
                raise SystemExit("rank %d: no NCCL id from rank 0" % rank)
            time.sleep(0.05)
        nid = open(id_path, "rb").read()
    devices = case.get("devices") or [0] * K
    pipe = pst.Pipeline(net, flat, ppv, case["B"], case["lr"], case.get("lr_np", case["lr"][-1]),
                        momentum=case.get("mom", 0.9), weight_decay=case.get("wd", 1e-4),
                        milestones=case.get("milestones", ()), steps_per_epoch=case.get("spe", 1 << 62),
                        devices=devices, rank=rank, nccl_id=nid, dropout_seed=case.get("dropout_seed", 0))
    if case.get("n_p") is not None:
        pipe.set_hybrid(case["n_p"] // case["spe"])
    for x, y in data:
        # only stage 0 reads the images and only the last stage reads the labels (pst.h pst_batch)
        pipe.step(x if rank == 0 else None, y if rank == K - 1 else None)
    pipe.flush()
    out = {"params": pipe.weights(pst.W_PARAMS), "momentum": pipe.weights(pst.W_MOMENTUM),
           "bnstats": pipe.weights(pst.W_BNSTATS), "versions": pipe.versions(),
           "progress": np.array(pipe.progress())}
    if rank == K - 1:
        out["losses"] = pipe.losses(0, case["N"])
    np.savez(os.path.join(workdir, "rank%d.npz" % rank), **out)
    pipe.close()


if __name__ == "__main__":
    main()
