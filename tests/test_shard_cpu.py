"""Multi-rank protocol on CPU (gloo, world_size 2): the product's shard partition
(qbxg_plan_shard), the multipole exchange as one broadcast per rank of its box range,
the straddle recompute, and the result all-gather as one broadcast per rank of its
packed owned targets / centres (the layout csrc/cuda/handle.cu builds for the NCCL
path: rank-major; associated targets in target order, then conventional targets in
box order; centres in box order), executed by the oracle in two processes, must
reproduce the single-process oracle bitwise ("G-GPU output must be
bitwise identical")."""
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
    rows = Mbuf.reshape(plan.view.n_boxes, -1)
    for r in range(world):  # multipole exchange: rank r's box range from rank r
        seg = torch.from_numpy(np.ascontiguousarray(rows[cuts[r]:cuts[r + 1]]))
        dist.broadcast(seg, src=r)
        rows[cuts[r]:cuts[r + 1]] = seg.numpy()
    pot, coef = O.execute_phase(plan, g, w, mu, mask, 2, rows.reshape(-1), want_centers=True)
    # result all-gather: packed owned segments, one broadcast per rank, then scatter
    A = plan.arrays()
    owner = lambda b: int(np.searchsorted(cuts, b, side="right") - 1)  # noqa: E731
    ctr_box = np.empty(g.n_centers, dtype=np.int64)
    for b in range(A["n_boxes"]):
        s0, n = A["ctr_own_start"][b], A["ctr_own_count"][b]
        ctr_box[A["ctr_perm"][s0:s0 + n]] = b
    tseg = [[] for _ in range(world)]
    cseg = [[] for _ in range(world)]
    for t in np.nonzero(g.association >= 0)[0]:
        tseg[owner(ctr_box[g.association[t]])].append(t)
    for b in range(A["n_boxes"]):
        s0, n = A["tgt_own_start"][b], A["tgt_own_count"][b]
        tseg[owner(b)].extend(A["tgt_perm"][s0:s0 + n])
        s0, n = A["ctr_own_start"][b], A["ctr_own_count"][b]
        cseg[owner(b)].extend(A["ctr_perm"][s0:s0 + n])
    full_pot = np.zeros(g.n_targets)
    full_coef = np.zeros(coef.shape, dtype=complex)
    for r in range(world):
        ti, ci = np.array(tseg[r], dtype=np.int64), np.array(cseg[r], dtype=np.int64)
        tp = torch.from_numpy(np.ascontiguousarray(pot[ti]) if r == rank else np.zeros(ti.size))
        tc = torch.from_numpy(np.ascontiguousarray(np.stack([coef[ci].real, coef[ci].imag], -1)) if r == rank
                              else np.zeros((ci.size,) + coef.shape[1:] + (2,)))
        dist.broadcast(tp, src=r)
        dist.broadcast(tc, src=r)
        full_pot[ti] = tp.numpy()
        full_coef[ci] = tc.numpy()[..., 0] + 1j * tc.numpy()[..., 1]
    assert sum(len(x) for x in tseg) == g.n_targets and sum(len(x) for x in cseg) == g.n_centers
    tp = torch.from_numpy(full_pot)
    tc = torch.from_numpy(np.ascontiguousarray(np.stack([full_coef.real, full_coef.imag], -1)).reshape(-1))
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
