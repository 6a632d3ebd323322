"""Multi-process (N>1) host logic on CPU: world-size 2 and 3 over torch.distributed gloo.

One process per stage, as `bench.py --gpus N` runs libpst in distributed mode.
Each rank follows libpst's own step schedule (pst_schedule, the same plan_step
the NCCL path uses) and exchanges exactly the messages pst_api.cu's
distributed step exchanges at the end of every step:
  send activation(f) -> s+1, recv activation(prev stage's f) <- s-1,
  send delta(b)      -> s-1, recv delta(next stage's b)      <- s+1,
with the stage arithmetic done by the oracle's stage functions.  The result
must equal Oracle A (the definition) bit for bit.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import pst_workloads as W
from oracle import layers as Lx
from oracle import network as Net
from oracle import pipeline as Pl


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, ppv, n_mb, out_dir):
    import paper_1912_12675_b200 as pst
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    K = world
    net = W.tiny_resnet(width=8, hw=8, n=1)
    flat = W.init_params(net, seed=3)
    data = W.batches(net.in_shape, 4, n_mb, seed=9)
    bounds = Net.partition(net.layers, ppv)
    a, b = bounds[rank]
    stage = Net.CNNStage(net.layers[a:b], first_stage=(rank == 0))
    params = Net.unflatten(net.layers, flat)[a:b]
    mom = [{k: np.zeros_like(v) for k, v in d.items()} for d in params]
    hp = Pl.HParams(lr_pipelined=[0.05] * K, lr_nonpipelined=0.05, momentum=0.9, weight_decay=1e-3)
    # shapes of the boundary tensors (from a dry forward on a throwaway stage)
    shapes = []
    x = data[0][0]
    for s, (a2, b2) in enumerate(bounds):
        st = Net.CNNStage(net.layers[a2:b2], first_stage=(s == 0))
        x, _ = st.forward(Net.unflatten(net.layers, flat)[a2:b2], x)
        shapes.append(x.shape)
    in_shape = data[0][0].shape if rank == 0 else shapes[rank - 1]
    ring, inbox_f, inbox_b, dz = {}, {}, {}, {}
    losses = {}
    v = 0
    for t in range(n_mb + 2 * K - 1):
        bm, fm, fver = pst.schedule(K, rank, t, n_mb)
        if bm >= 0:                                   # backward + update first (AMB-1)
            g_in = dz.pop(bm) if rank == K - 1 else inbox_b.pop(bm)
            assert v == bm
            g, G = stage.backward(params, ring.pop(bm), g_in)
            new_p, new_m = [], []
            for P, M, GG in zip(params, mom, G):
                dp, dm = {}, {}
                for k in P:
                    dp[k], dm[k] = Lx.sgd_momentum(P[k], M[k], GG[k], Pl.learning_rate(hp, rank, bm), hp.momentum,
                                                   hp.weight_decay)
                new_p.append(dp)
                new_m.append(dm)
            params, mom = new_p, new_m
            v += 1
            delta = g
        if fm >= 0:
            assert fver == v, (t, rank, fver, v)      # the version the forward reads
            xin = data[fm][0] if rank == 0 else inbox_f.pop(fm)
            out, cache = stage.forward(params, xin)
            ring[fm] = cache
            if rank == K - 1:
                losses[fm], dz[fm] = Lx.softmax_ce(out, data[fm][1])
        # end-of-step exchange, exactly the NCCL group of pst_api.cu enqueue_pipe
        reqs, recvs = [], []
        if fm >= 0 and rank < K - 1:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(out)), rank + 1))
        if rank > 0:
            pf = pst.schedule(K, rank - 1, t, n_mb)[1]
            if pf >= 0:
                buf = torch.empty(in_shape, dtype=torch.float64)
                reqs.append(dist.irecv(buf, rank - 1))
                recvs.append(("f", pf, buf))
        if bm >= 0 and rank > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(delta)), rank - 1))
        if rank < K - 1:
            nb = pst.schedule(K, rank + 1, t, n_mb)[0]
            if nb >= 0:
                buf = torch.empty(shapes[rank], dtype=torch.float64)
                reqs.append(dist.irecv(buf, rank + 1))
                recvs.append(("b", nb, buf))
        for r in reqs:
            r.wait()
        for kind, mb, buf in recvs:
            (inbox_f if kind == "f" else inbox_b)[mb] = buf.numpy().copy()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), flat=Net.flatten(net.layers[a:b], params),
             losses=np.array([losses[i] for i in range(n_mb)]) if losses else np.zeros(0), v=v)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,ppv", [(2, (3,)), (3, (1, 3))])
def test_distributed_schedule_matches_definition(world, ppv):
    n_mb = 7
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_main, args=(world, _free_port(), ppv, n_mb, d), nprocs=world, join=True)
        got = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    net = W.tiny_resnet(width=8, hw=8, n=1)
    flat = W.init_params(net, seed=3)
    data = W.batches(net.in_shape, 4, n_mb, seed=9)
    bounds = Net.partition(net.layers, ppv)
    stages = [Net.CNNStage(net.layers[a:b], first_stage=(s == 0)) for s, (a, b) in enumerate(bounds)]
    per_layer = Net.unflatten(net.layers, flat)
    hp = Pl.HParams(lr_pipelined=[0.05] * world, lr_nonpipelined=0.05, momentum=0.9, weight_decay=1e-3)
    ref = Pl.run_versioned(stages, [per_layer[a:b] for a, b in bounds], data, hp)
    for r, (a, b) in enumerate(bounds):
        assert np.array_equal(got[r]["flat"], Net.flatten(net.layers[a:b], ref.params[r]))
        assert int(got[r]["v"]) == n_mb
    assert np.array_equal(got[-1]["losses"], np.array(ref.losses))
