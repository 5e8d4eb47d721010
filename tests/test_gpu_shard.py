"""Sharded (multi-GPU) apply, emulated on one GPU: ranks are separate handles
driven phase by phase in one process (no kernel ever waits on another rank),
the multipole exchange is a device copy (qbxg_exchange_local) standing in for
the NCCL broadcasts.  The sum of the ranks' outputs must equal the unsharded
apply bitwise (SURVEY.md §8e parity requirement)."""
import numpy as np
import pytest

from paper_1805_06106_b200 import api

pytestmark = pytest.mark.gpu


def _sharded(cfg, g, plan, nranks, w, mu, want_centres=True):
    import torch
    dev = torch.device("cuda", 0)
    dw = torch.from_numpy(w).to(dev)
    dm = torch.from_numpy(mu.reshape(-1)).to(dev) if mu is not None else None
    engines = [api.FmmEngine(cfg, g, plan, shard=(nranks, r)) for r in range(nranks)]
    pots = [torch.empty(g.n_targets, dtype=torch.float64, device=dev) for _ in range(nranks)]
    coefs = [torch.empty(g.n_centers * 2 * cfg.kq, dtype=torch.float64, device=dev) for _ in range(nranks)]
    for e in engines:
        e.apply_phase(1, dw.data_ptr(), dm.data_ptr() if dm is not None else None, None)
    api.exchange_local(engines)
    for e, p, c in zip(engines, pots, coefs):
        e.apply_phase(2, dw.data_ptr(), dm.data_ptr() if dm is not None else None, p.data_ptr(),
                      c.data_ptr() if want_centres else None)
    torch.cuda.synchronize()
    pot = sum(p for p in pots).cpu().numpy()
    c = sum(x for x in coefs).cpu().numpy().reshape(g.n_centers, cfg.kq, 2)
    for e in engines:
        e.close()
    return pot, c[..., 0] + 1j * c[..., 1]


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("case", ["torus", "urchin_vol"])
def test_sharded_equals_single_bitwise(nranks, case):
    if case == "torus":
        g = api.config_geometry(1, nu=48, nv=24)
        cfg = api.config_fmm(1)
        mu = g.dipoles()
    else:
        g = api.config_geometry(2, level=2, n_volume_targets=3000)
        cfg = api.config_fmm(2)
        mu = None
    plan = api.Plan(cfg, g)
    w = g.weights()
    ref = api.FmmEngine(cfg, g, plan)
    pot1, c1 = ref.apply(w, mu, want_centers=True)
    ref.close()
    pot, c = _sharded(cfg, g, plan, nranks, w, mu)
    assert np.array_equal(pot, pot1), np.abs(pot - pot1).max()
    assert np.array_equal(c, c1)


def test_shard_roles_partition():
    g = api.config_geometry(1, nu=48, nv=24)
    plan = api.Plan(api.config_fmm(1), g)
    a = plan.arrays()
    n = 4
    owners = np.zeros(plan.view.n_boxes, dtype=np.int32)
    for r in range(n):
        cuts, mask = api.plan_shard(plan, n, r)
        own = (mask & 1) > 0
        assert np.all(np.nonzero(own)[0] == np.arange(cuts[r], cuts[r + 1]))
        owners[own] += 1
        # every owned box is also in the downward set; straddle bits agree across ranks
        assert np.all((mask[own] & 8) > 0)
        if r == 0:
            straddle0 = (mask & 4) > 0
        else:
            assert np.array_equal((mask & 4) > 0, straddle0)
    assert np.all(owners == 1)
    assert straddle0[0]  # the root straddles every cut
    # cost balance: every rank holds at least some target boxes
    assert len(np.unique(cuts)) == n + 1


@pytest.mark.parametrize("nranks", [2, 3])
def test_sharded_result_allgather_equals_single_bitwise(nranks):
    """The result all-gather of a sharded apply (packed owned segments broadcast to every
    rank and scattered; qbxg_result_exchange_local standing in for the grouped NCCL
    broadcasts) leaves the whole single-GPU result on every rank, bitwise."""
    import torch
    g = api.config_geometry(2, level=2, n_volume_targets=3000)
    cfg = api.config_fmm(2)
    plan = api.Plan(cfg, g)
    w = g.weights()
    ref = api.FmmEngine(cfg, g, plan)
    pot1, c1 = ref.apply(w, None, want_centers=True)
    ref.close()
    dev = torch.device("cuda", 0)
    dw = torch.from_numpy(w).to(dev)
    engines = [api.FmmEngine(cfg, g, plan, shard=(nranks, r)) for r in range(nranks)]
    pots = [torch.empty(g.n_targets, dtype=torch.float64, device=dev) for _ in range(nranks)]
    coefs = [torch.empty(g.n_centers * 2 * cfg.kq, dtype=torch.float64, device=dev) for _ in range(nranks)]
    for e in engines:
        e.apply_phase(1, dw.data_ptr(), None, None)
    api.exchange_local(engines)
    for e, p, c in zip(engines, pots, coefs):
        e.apply_phase(2, dw.data_ptr(), None, p.data_ptr(), c.data_ptr())
    api.exchange_results_local(engines, [p.data_ptr() for p in pots], [c.data_ptr() for c in coefs])
    torch.cuda.synchronize()
    for p, c in zip(pots, coefs):
        assert np.array_equal(p.cpu().numpy(), pot1)
        cc = c.cpu().numpy().reshape(g.n_centers, cfg.kq, 2)
        assert np.array_equal(cc[..., 0] + 1j * cc[..., 1], c1)
    for e in engines:
        e.close()


@pytest.mark.parametrize("nranks,kernel,p,q,geo", [
    (2, 2, 8, 4, "urchin_vol"), (3, 2, 8, 4, "urchin_vol"), (2, 3, 8, 4, "urchin_vol"), (3, 3, 8, 4, "urchin_vol"),
    (2, 3, 20, 5, "sphere3")])  # the last: BASELINE config 3's orders on a level-3 sphere
def test_helmholtz_sharded_equals_single_bitwise(nranks, kernel, p, q, geo):
    """Helmholtz SL and SL+DL (complex128) over Morton shards: phases driven per rank with
    complex device arrays, full complex multipole rows exchanged, the packed owned results
    all-gathered -- every rank ends with the single-GPU result, bitwise."""
    import torch
    K = 3.0
    g = (api.config_geometry(2, level=2, n_volume_targets=2000) if geo == "urchin_vol"
         else api.config_geometry(3, level=3))
    cfg = api.FmmConfig(p_fmm=p, p_qbx=q, n_max=64, kernel=kernel, helmholtz_k=K)
    plan = api.Plan(cfg, g)
    rng = np.random.default_rng(11)
    w = g.quad_weight * (rng.uniform(-1, 1, g.n_sources) + 1j * rng.uniform(-1, 1, g.n_sources))
    mu = None
    if kernel == 3:
        mu = np.ascontiguousarray((w[:, None] * rng.standard_normal((g.n_sources, 3))).astype(np.complex128))
    ref = api.FmmEngine(cfg, g, plan)
    pot1, c1 = ref.apply_complex(w, mu, want_centers=True)
    ref.close()
    kq = (cfg.p_qbx + 1) ** 2
    dev = torch.device("cuda", 0)
    dw = torch.from_numpy(w.view(np.float64).copy()).to(dev)
    dm = torch.from_numpy(mu.reshape(-1).view(np.float64).copy()).to(dev) if mu is not None else None
    engines = [api.FmmEngine(cfg, g, plan, shard=(nranks, r)) for r in range(nranks)]
    _, row, cuts = engines[0].multipole_buffer()
    assert row == 2 * (cfg.p_fmm + 1) ** 2 and len(cuts) == nranks + 1
    pots = [torch.empty(2 * g.n_targets, dtype=torch.float64, device=dev) for _ in range(nranks)]
    coefs = [torch.empty(2 * g.n_centers * kq, dtype=torch.float64, device=dev) for _ in range(nranks)]
    mp = dm.data_ptr() if dm is not None else None
    for e in engines:
        e.apply_phase(1, dw.data_ptr(), mp, None)
    api.exchange_local(engines)
    for e, p, c in zip(engines, pots, coefs):
        e.apply_phase(2, dw.data_ptr(), mp, p.data_ptr(), c.data_ptr())
    torch.cuda.synchronize()
    # before the result exchange: the ranks' outputs partition the result (zeros elsewhere)
    psum = sum(p for p in pots).cpu().numpy().view(np.complex128)
    nz = sum((p.view(-1, 2) != 0).any(dim=1).to(torch.int32) for p in pots).cpu().numpy()
    assert nz.max() <= 1
    assert np.array_equal(psum, pot1)
    api.exchange_results_local(engines, [p.data_ptr() for p in pots], [c.data_ptr() for c in coefs])
    torch.cuda.synchronize()
    for p, c in zip(pots, coefs):
        assert np.array_equal(p.cpu().numpy().view(np.complex128), pot1)
        assert np.array_equal(c.cpu().numpy().view(np.complex128).reshape(g.n_centers, kq), c1)
    for e in engines:
        e.close()


@pytest.mark.parametrize("kernel", ["laplace_sl_dl", "helmholtz_sl_dl"])
def test_nccl_protocol_on_a_communicator_of_one(kernel):
    """The production multi-GPU path end to end through NCCL itself (libnccl loaded at run
    time, ncclCommInitRank, the grouped in-place multipole broadcast, the grouped result
    broadcasts and the scatter) on a communicator of one rank: a handle from
    qbxg_create_sharded(n_ranks = 1) runs phase 1 -> exchange -> phase 2 -> result gather
    inside qbxg_apply / qbxg_apply_complex.  Bitwise equal to the unsharded handle."""
    if kernel == "laplace_sl_dl":
        g = api.config_geometry(1, nu=48, nv=24)
        cfg = api.config_fmm(1)
        w, mu = g.weights(), g.dipoles()
        run = lambda e: e.apply(w, mu, want_centers=True)
    else:
        g = api.config_geometry(3, level=2)
        cfg = api.FmmConfig(p_fmm=8, p_qbx=4, n_max=64, kernel=3, helmholtz_k=3.0)
        rng = np.random.default_rng(5)
        w = g.quad_weight * (rng.uniform(-1, 1, g.n_sources) + 1j * rng.uniform(-1, 1, g.n_sources))
        mu = np.ascontiguousarray(w[:, None] * rng.standard_normal((g.n_sources, 3)))
        run = lambda e: e.apply_complex(w, mu, want_centers=True)
    plan = api.Plan(cfg, g)
    ref = api.FmmEngine(cfg, g, plan)
    pot1, c1 = run(ref)
    ref.close()
    eng = api.FmmEngine(cfg, g, plan, shard=(1, 0))
    with pytest.raises(ValueError, match="attach NCCL"):
        run(eng)
    eng.attach_nccl(api.FmmEngine.nccl_unique_id())
    pot, c = run(eng)
    pot2, _ = run(eng)
    eng.close()
    assert np.array_equal(pot, pot1) and np.array_equal(c, c1)
    assert np.array_equal(pot2, pot1)


def test_sharded_full_config1_equals_single_bitwise():
    """The bench workload (BASELINE config 1 at full size: 1,048,576 sources, 180,081 boxes)
    over 4 emulated ranks: every rank ends with the single-GPU potentials, bitwise.  (At this
    size the ~400 MB of exchanged multipole rows once exposed a race in the emulated exchange,
    which copied device to device without waiting: qbxg_exchange_local now synchronises.)"""
    import torch
    g = api.config_geometry(1)
    cfg = api.config_fmm(1)
    plan = api.Plan(cfg, g)
    w, mu = g.weights(), g.dipoles()
    dev = torch.device("cuda", 0)
    dw = torch.from_numpy(w).to(dev)
    dm = torch.from_numpy(mu.reshape(-1)).to(dev)
    p1 = torch.empty(g.n_targets, dtype=torch.float64, device=dev)
    ref = api.FmmEngine(cfg, g, plan)
    ref.apply_device(dw.data_ptr(), dm.data_ptr(), p1.data_ptr(), None, None)
    torch.cuda.synchronize()
    ref.close()
    n = 4
    engines = [api.FmmEngine(cfg, g, plan, shard=(n, r)) for r in range(n)]
    pots = [torch.empty(g.n_targets, dtype=torch.float64, device=dev) for _ in range(n)]
    for e in engines:
        e.apply_phase(1, dw.data_ptr(), dm.data_ptr(), None)
    api.exchange_local(engines)
    for e, p in zip(engines, pots):
        e.apply_phase(2, dw.data_ptr(), dm.data_ptr(), p.data_ptr(), None)
    api.exchange_results_local(engines, [p.data_ptr() for p in pots], None)
    torch.cuda.synchronize()
    for p in pots:
        assert torch.equal(p, p1)
    for e in engines:
        e.close()
