#!/usr/bin/env python3
"""Benchmark: pipelined stale-weight training throughput on B200 (BASELINE.json metric).

    python bench.py --gpus N --steps K --warmup W            (N>1: under torch.distributed.run)
    python bench.py --impl reference --gpus N --steps K --warmup W

Workload: ResNet-110, CIFAR-10-shaped synthetic data, batch 128 (BASELINE.json
configs[3], the paper's headline ResNet-110 case), split into
K = N pipeline stages, one per GPU (PPV from pst_workloads.CONFIGS; N=1 is
non-pipelined training on one GPU).  One step = one global pipeline step: every
stage runs the backward+update of one mini-batch and the forward of another, so
the job trains `batch` images per step; value = steps * batch / device time
(max over ranks).  Prints ONE JSON line on rank 0.

The reference arm for this tier is the CPU oracle (oracle/, the only other place
bench.py executes it): each step trains a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

METRIC = "train images/sec at 1/2/4/8 B200 stages; speedup vs 1-GPU; conv tensor-pipe %"
PAPER_IMG_S = {1: 760.0, 2: 1321.0}   # ResNet-110 on GTX1060, context only


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="resnet110")
    p.add_argument("--batch", type=int, default=0)
    p.add_argument("--profile-steps", type=int, default=2)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=16, help="images per oracle sample step")
    p.add_argument("--spin-seconds", type=float, default=1.5, help="untimed spin-up before timing (0 under ncu)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def spawn_ranks(n):
    """`python bench.py --gpus N` without a launcher: start N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1 and return their exit code (rank 0 prints the line)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def share_gpu():
    """PST_BENCH_SHARE_GPU=1: every rank on cuda:0 (a functional check of the N-rank path on a one-GPU
    box; NCCL needs a distinct NCCL_HOSTID per rank to accept two ranks on one device and then uses
    its socket transport).  Numbers from such a run are not throughput measurements."""
    return os.environ.get("PST_BENCH_SHARE_GPU") == "1"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        if self.p is None:
            return out
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.count(",") >= 5]
        os.unlink(self.f.name)
        if not rows:
            return out
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].strip().lower() == "active"})
        out.update(sm_mhz=statistics.median(sm) if sm else None, sm_max_mhz=max(mx) if mx else None,
                   reasons=reasons, samples=len(rows))
        return out


# --------------------------------------------------------------------------- CPU oracle (baseline)
def oracle_sample_rate(cfg, sample_b, n_steps=1, seed=42):
    """Train `n_steps` non-pipelined oracle steps on a sample_b-image slice; img/s."""
    import pst_workloads as W
    from oracle import network as Net, pipeline as Pl, layers as Lx
    net = cfg.netspec()
    flat = W.init_params(net, seed=seed)
    st = Net.CNNStage(net.layers, first_stage=True)
    params = Net.unflatten(net.layers, flat)
    hp = Pl.HParams(lr_pipelined=[cfg.base_lr], lr_nonpipelined=cfg.base_lr, momentum=cfg.momentum,
                    weight_decay=cfg.weight_decay)
    data = [W.make_batch(net.in_shape, sample_b, i, seed=1234) for i in range(n_steps)]
    t0 = time.perf_counter()
    Pl.run_sgd(st, params, data, hp)
    dt = time.perf_counter() - t0
    return n_steps * sample_b / dt, dt


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        return int(max(n)) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def oracle_lenet5_config(n_steps=20):
    """BASELINE configs[0] in full through the oracle's schedule: LeNet-5, MNIST-shaped, batch 64,
    2 stages (PPV (1)), n_steps mini-batches (Oracle B, fill and drain included); img/s."""
    import pst_workloads as W
    from oracle import network as Net, pipeline as Pl
    cfg = W.CONFIGS["lenet5"]
    net = cfg.netspec()
    flat = W.init_params(net, seed=42)
    bounds = Net.partition(net.layers, cfg.ppv[2])
    st = [Net.CNNStage(net.layers[a:b], first_stage=(s == 0), layer0=a) for s, (a, b) in enumerate(bounds)]
    per = Net.unflatten(net.layers, flat)
    hp = Pl.HParams(lr_pipelined=cfg.lr_vector(2), lr_nonpipelined=cfg.base_lr, momentum=cfg.momentum,
                    weight_decay=cfg.weight_decay)
    data = [W.make_batch(net.in_shape, cfg.batch, i, seed=1234) for i in range(n_steps)]
    t0 = time.perf_counter()
    Pl.run_clocked(st, [per[a:b] for a, b in bounds], data, hp)
    dt = time.perf_counter() - t0
    return n_steps * cfg.batch / dt, dt


def cpu_baseline(cfg, sample):
    """SURVEY 8(d) oracle timing: the bench workload (one non-pipelined SGD step of the full
    batch-128 mini-batch, fp64 NumPy, BLAS threads = host cores) as `value`; beside it the same step
    on a `sample`-image slice with ONE BLAS thread, and BASELINE configs[0] (LeNet-5 K=2, 20 steps) in
    full.  About 20-40 s of host time."""
    rate, dt = oracle_sample_rate(cfg, cfg.batch, 1)
    out = {"value": rate, "unit": "img/s", "cores": blas_threads(), "kind": "oracle",
           "host_cpus": os.cpu_count(),
           "sample": f"1 non-pipelined SGD step of {cfg.net} on a full {cfg.batch}-image mini-batch "
                     f"({dt:.1f} s, float64 NumPy, BLAS threads = {blas_threads()})"}
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1, user_api="blas"):
            r1, d1 = oracle_sample_rate(cfg, sample, 1)
        out["one_thread"] = {"value": r1, "unit": "img/s", "sample": f"{sample}-image slice, 1 BLAS thread ({d1:.1f} s)"}
    except Exception as e:   # threadpoolctl missing: report, do not fail the bench
        out["one_thread"] = {"unavailable": str(e)[:120]}
    rl, dl = oracle_lenet5_config(20)
    out["lenet5_k2_config0"] = {"value": rl, "unit": "img/s", "seconds": dl,
                                "sample": "BASELINE configs[0] in full: LeNet-5 b64, 2 stages, 20 steps (Oracle B)"}
    return out


def run_reference(args, rank, world):
    import pst_workloads as W
    if rank != 0:
        return
    cfg = W.CONFIGS[args.config]
    B = args.batch or cfg.batch
    sample = args.cpu_sample
    for _ in range(args.warmup):
        oracle_sample_rate(cfg, sample, 1)
    tot = 0.0
    for _ in range(args.steps):
        _, dt = oracle_sample_rate(cfg, sample, 1)
        tot += dt
    rate = args.steps * sample / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "img/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.net}_cifar10_b{B}_pp{world}", "model": cfg.net, "global_batch": B,
                   "stages": world, "parallelism": "none (CPU oracle on the host, rank 0 only)",
                   "sample": f"{sample} of the {B} images per step"},
        "cpu_baseline": {"value": rate, "unit": "img/s", "cores": blas_threads(), "kind": "oracle",
                         "sample": f"1 non-pipelined SGD step of {cfg.net} on a {sample}-image slice per step"},
        "e2e": {"value": rate, "unit": "img/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our arm
def main():
    args = parse()
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import pst_workloads as W
    import paper_1912_12675_b200 as pst

    shared = share_gpu() and world > 1
    if shared:
        local = 0
        os.environ["NCCL_HOSTID"] = f"pst-bench-rank{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
    elif torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    cfg = W.CONFIGS[args.config]
    K = world
    if K in cfg.ppv:
        ppv = cfg.ppv[K]
    elif cfg.net.startswith("resnet"):     # any other stage count: the profile-driven balancer
        from pst_workloads import balance as Bl
        netspec = cfg.netspec()
        ppv = Bl.balance_ppv(Bl.resnet_layer_costs(netspec, Bl.load_cost_table()), K,
                             Bl.resnet_boundaries(netspec))
    else:
        raise SystemExit(f"no PPV for {K} stages in config {cfg.name}")
    B = args.batch or cfg.batch
    net = cfg.netspec()
    params = W.init_params(net, seed=42)
    lr = cfg.lr_vector(K)
    kw = dict(momentum=cfg.momentum, weight_decay=cfg.weight_decay, milestones=cfg.milestones,
              steps_per_epoch=cfg.steps_per_epoch)
    if world > 1:
        nid = [pst.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        pipe = pst.Pipeline(net, params, ppv, B, lr, cfg.base_lr, devices=[0] * K if shared else list(range(K)),
                            rank=rank,
                            nccl_id=nid[0], **kw)
        my_stage = rank
    else:
        pipe = pst.Pipeline(net, params, ppv, B, lr, cfg.base_lr, **kw)
        my_stage = 0
    stream = torch.cuda.ExternalStream(pipe.stream(my_stage))

    n_pool = 8
    host = [W.make_batch(net.in_shape, B, i, seed=1234) for i in range(n_pool)]
    dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()) for x, y in host]
    torch.cuda.synchronize()

    warm = max(args.warmup, 2 * K)   # reach the pipeline's steady state before timing
    for i in range(warm):
        pipe.step(*dev[i % n_pool])
    pipe.sync()
    t_w = time.perf_counter()
    for i in range(10):
        pipe.step(*dev[(warm + i) % n_pool])
    pipe.sync()
    per_step = (time.perf_counter() - t_w) / 10
    warm += 10
    # untimed spin-up: about 1.5 s more of steps so a fresh box's clocks and caches settle (the
    # first bench on a new box otherwise sometimes reads 20-50% slow); the count is agreed on
    # by all ranks, whose stages exchange activations every step
    # clocks: sampled from the start of the spin-up through the end of the timed region (the timed
    # region alone is ~0.1 s, shorter than nvidia-smi's sampling period)
    clocks = ClockSampler(local)
    n_spin = int(max_over_ranks(float(min(2000, int(args.spin_seconds / max(per_step, 1e-4))))))
    for i in range(n_spin):
        pipe.step(*dev[(warm + i) % n_pool])
        if i % 50 == 49:
            pipe.sync()
    pipe.sync()
    warm += n_spin
    torch.cuda.synchronize()
    barrier()

    # ---- device-timed region: inputs resident in HBM
    l0 = pipe.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    e0.record(stream)
    for i in range(args.steps):
        pipe.step(*dev[(warm + i) % n_pool])
    e1.record(stream)
    pipe.sync()
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    launches = int(sum_over_ranks(pipe.launches() - l0))   # every rank's kernels in the timed region
    clk = clocks.stop()
    value = args.steps * B / (ms / 1e3)

    # ---- instrumented window: CUDA events around every kernel (eager launches)
    pipe.profile(True)
    for i in range(args.profile_steps):
        pipe.step(*dev[i % n_pool])
    prof = pipe.profile_read()
    pipe.profile(False)
    pk = peaks()
    cls = max(prof, key=lambda k: prof[k][0])
    kms, kn, kbytes, kflops = prof[cls]
    achieved = kbytes / (kms / 1e3) / 1e9 if kms > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(cls)
        except Exception:
            traffic = None
    step_ms_prof = sum(v[0] for v in prof.values()) / max(1, args.profile_steps)
    # Roofline of the dominant kernel class: the binding resource is the one whose lower-bound
    # time (algorithmic bytes / HBM peak vs algorithmic flops / tensor peak) is larger.
    # Tensor peak for the default build's fp32 contraction: 3 TF32 products per fp32 product
    # (3xTF32), TF32 = measured bf16 peak x the guide's nominal 1.1/2.25 ratio.
    info = pst.build_info()
    hbm_peak = pk.get("hbm_gbs", 6650.0)
    bf16_peak = pk.get("bf16_tflops", 1590.0)
    if "tf32x3" in info:
        tc_peak, tc_note = bf16_peak * (1.1 / 2.25) / 3.0, "bf16_tflops x 1.1/2.25 (tf32) / 3 (3xTF32 products)"
    else:
        tc_peak, tc_note = bf16_peak, "bf16_tflops"
    t_bw = kbytes / (hbm_peak * 1e9) if kbytes else 0.0
    t_tc = kflops / (tc_peak * 1e12) if kflops else 0.0
    tflops = kflops / (kms / 1e3) / 1e12 if kms > 0 else 0.0
    if t_tc > t_bw:
        bound, ach, peak, unit = "tensor", tflops, tc_peak, "TFLOP/s"
        src = "MEASURED_PEAKS.json " + tc_note + ("" if not pk.get("fallback") else " of fallback")
    else:
        bound, ach, peak, unit = "hbm", achieved, hbm_peak, "GB/s"
        src = "MEASURED_PEAKS.json hbm_gbs (burst copy)" + ("" if not pk.get("fallback") else " of fallback")
    roofline = {"bound": bound, "kernel": cls, "achieved": ach, "peak": peak, "unit": unit,
                "frac": ach / peak if peak else None, "traffic": traffic,
                "alg_bytes_per_launch": kbytes / max(1, kn), "alg_flops_per_launch": kflops / max(1, kn),
                "launches": kn, "avg_launch_us": 1e3 * kms / max(1, kn),
                "share_of_step": (kms / max(1, args.profile_steps)) / step_ms_prof if step_ms_prof else None,
                "hbm_gbs": achieved, "tensor_tflops": tflops,
                "frac_of_roofline_time": (max(t_bw, t_tc) / (kms / 1e3)) if kms > 0 else None,
                "peak_source": src}
    # BASELINE metric's "conv tensor-pipe %": all conv work (fwd + dgrad + wgrad) against the
    # contraction peak over the conv kernels' own (serially timed) device time
    conv = [prof[k] for k in ("conv_fwd", "conv_dgrad", "conv_wgrad") if k in prof]
    conv_ms = sum(v[0] for v in conv)
    conv_tflops = (sum(v[3] for v in conv) / (conv_ms / 1e3) / 1e12) if conv_ms > 0 else 0.0
    conv_pipe = {"tflops": conv_tflops, "peak_tflops": tc_peak, "pct": 100.0 * conv_tflops / tc_peak if tc_peak else None,
                 "conv_ms_per_step": conv_ms / max(1, args.profile_steps),
                 "note": "sum of conv FLOPs / conv kernel time (per-kernel CUDA events, serial) / " + tc_note,
                 "ncu_counter": "sm__pipe_tensor_cycles_active 9.5-12.9% on the ResNet-110 conv kernels "
                                "(tcgen05 UTCHMMA issue; profiles/r2_tc_counters.txt)"}
    def class_roofline(v):
        # each class against its own binding resource: the larger of its algorithmic bytes at the HBM
        # peak and its flops at the contraction peak, over its event-timed device time
        tb = v[2] / (hbm_peak * 1e9) if v[2] else 0.0
        tt = v[3] / (tc_peak * 1e12) if v[3] else 0.0
        return ("tensor" if tt > tb else "hbm"), (max(tb, tt) / (v[0] / 1e3) if v[0] > 0 else None)
    kernel_table = {k: {"ms_per_step": v[0] / max(1, args.profile_steps), "launches_per_step": v[1] / max(1, args.profile_steps),
                        "GBps": (v[2] / (v[0] / 1e3) / 1e9) if v[0] > 0 else 0.0,
                        "TFLOPs": (v[3] / (v[0] / 1e3) / 1e12) if v[0] > 0 else 0.0,
                        "bound": class_roofline(v)[0], "roofline_frac": class_roofline(v)[1]}
                    for k, v in prof.items() if v[1] > 0}

    # ---- end-to-end through the public API: host buffers, H2D + loss readback every step
    e2e = None
    if not args.no_e2e:
        last = (rank == K - 1) if world > 1 else True
        torch.cuda.synchronize()
        barrier()
        steps0, fed0 = pipe.progress()
        t0 = time.perf_counter()
        for i in range(args.steps):
            x, y = host[i % n_pool]
            pipe.step(x, y)
            if last:
                mb = fed0 + i - (K - 1)
                if mb >= 0:
                    pipe.losses(mb, 1)
        pipe.sync()
        dt = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": args.steps * B / dt, "unit": "img/s",
               "h2d_bytes_per_step": int(host[0][0].nbytes + host[0][1].nbytes), "d2h_bytes_per_step": 4}

    # ---- per-stage device memory (pst_memory; the paper's activation storage P:L65/L75, Table 6)
    mine = [dict(stage=s_, **pipe.memory(s_)) for s_ in ([my_stage] if world > 1 else range(K))]
    if dist is not None:
        allm = [None] * world
        dist.all_gather_object(allm, mine)
        mine = [m for part in allm for m in part]
    memory = {"per_stage": mine,
              "note": "bytes_per_slot = saved forward state of one mini-batch; ring_slots kept vs the paper's "
                      "2(K-s)-1 (paper_slots); total = every device buffer of the stage"}
    tot = sum(m["bytes_per_slot"] for m in mine)
    extra_paper = sum((m["paper_slots"] - 1) * m["bytes_per_slot"] for m in mine)
    extra_kept = sum((m["ring_slots"] - 1) * m["bytes_per_slot"] for m in mine)
    pbytes = sum(m["param_bytes"] for m in mine)
    memory["increase_pct_paper_depth"] = 100.0 * extra_paper / (tot + pbytes) if tot else None
    memory["increase_pct_as_built"] = 100.0 * extra_kept / (tot + pbytes) if tot else None

    # ---- CPU oracle baseline (rank 0, N == 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.cpu_sample)

    if shared:
        placement = ("all ranks on cuda:0, NCCL socket transport (PST_BENCH_SHARE_GPU=1): a functional check "
                     "of the N-rank path, not a throughput measurement")
    else:
        placement = "one process per GPU, NCCL send/recv" if world > 1 else "one GPU"
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "img/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "warmup_steps_run": warm, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": (value / PAPER_IMG_S[world]) if world in PAPER_IMG_S else None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg.net}_cifar10_b{B}_pp{K}", "model": cfg.net, "global_batch": B,
                       "stages": K, "ppv": list(ppv), "parallelism": f"pp{K}" if K > 1 else "none",
                       "precision": "fp32 storage, 3xTF32 tensor-core products (" + pst.build_info() + ")",
                       "l2": "inputs larger than L2 (saved forward state ~1 GB per mini-batch >> 126 MB)",
                       "placement": placement,
                       "lr_per_stage": lr},
            "clocks": clk, "gpu_launches": launches, "roofline": roofline, "conv_tensor_pipe": conv_pipe,
            "kernels": kernel_table,
            "e2e": e2e, "cpu_baseline": cpu, "memory": memory,
            "paper_context": {"img_s_1gpu_gtx1060": 760, "img_s_2gpu_gtx1060": 1321, "source": "PAPER.md L192"},
        }
        print(json.dumps(line), flush=True)
    pipe.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
