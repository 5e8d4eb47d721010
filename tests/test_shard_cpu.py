"""Multi-rank protocol on CPU (gloo, world_size 2): the product's shard
partition (qbxg_plan_shard) + multipole exchange + straddle recompute + result
sum, executed by the oracle in two processes, must reproduce the single-process
oracle bitwise ("G-GPU output must be bitwise identical")."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle as O
    from paper_1805_06106_b200 import api
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = api.config_geometry(1, nu=24, nv=12)
    cfg = api.config_fmm(1)
    plan = api.Plan(cfg, g)
    cuts, mask = api.plan_shard(plan, world, rank)
    kp = (cfg.p_fmm + 1) ** 2
    Mbuf = np.zeros(plan.view.n_boxes * kp * 2)
    w, mu = g.weights(), g.dipoles()
    O.execute_phase(plan, g, w, mu, mask, 1, Mbuf)
    t = torch.from_numpy(Mbuf)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)  # each owned row has exactly one non-zero contributor
    Mbuf = t.numpy()
    pot, coef = O.execute_phase(plan, g, w, mu, mask, 2, Mbuf, want_centers=True)
    tp = torch.from_numpy(pot)
    tc = torch.from_numpy(np.ascontiguousarray(np.stack([coef.real, coef.imag], -1)).reshape(-1))
    dist.all_reduce(tp, op=dist.ReduceOp.SUM)
    dist.all_reduce(tc, op=dist.ReduceOp.SUM)
    if rank == 0:
        np.save(os.path.join(out_dir, "pot.npy"), tp.numpy())
        np.save(os.path.join(out_dir, "coef.npy"), tc.numpy())
        np.save(os.path.join(out_dir, "cuts.npy"), cuts)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_protocol_matches_single(tmp_path):
    import torch.multiprocessing as mp
    import oracle as O
    from paper_1805_06106_b200 import api
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    pot = np.load(tmp_path / "pot.npy")
    coef = np.load(tmp_path / "coef.npy").reshape(-1, 2)
    cuts = np.load(tmp_path / "cuts.npy")
    g = api.config_geometry(1, nu=24, nv=12)
    cfg = api.config_fmm(1)
    plan = api.Plan(cfg, g)
    ref, cref, _ = O.execute(plan, g, g.weights(), g.dipoles(), want_centers=True)
    assert 0 < cuts[1] < plan.view.n_boxes
    assert np.array_equal(pot, ref)
    c = coef[:, 0] + 1j * coef[:, 1]
    assert np.array_equal(c, cref.reshape(-1))
