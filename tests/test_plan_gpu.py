"""Stage 1 on the GPU: qbxg_plan_create_gpu must give the
host plan bit for bit -- boxes, DFS numbering, particle permutations, per-role
ranges, flags, and every interaction list (CSR arrays and their hashes)."""
import numpy as np
import pytest

from paper_1805_06106_b200 import api

KEYS = ("n_boxes", "n_levels", "root_center", "root_radius", "box_center", "box_radius", "box_level", "box_parent",
        "child_starts", "children", "level_starts", "level_boxes", "box_flags", "src_perm", "ctr_perm", "tgt_perm")


def _same(host, gpu, lists=True):
    a, b = host.arrays(), gpu.arrays()
    for k in a:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
    if lists:
        assert host.list_hashes() == gpu.list_hashes()
        for k in range(6):
            for x, y in zip(host.list_csr(k), gpu.list_csr(k)):
                assert np.array_equal(x, y), k


def _cloud(seed, ns=4000, nc=3000, nt=1500, clustered=False):
    rng = np.random.default_rng(seed)
    src = rng.uniform(-1, 1, (ns, 3))
    if clustered:
        src[: ns // 2] = 0.3 + 0.01 * rng.normal(size=(ns // 2, 3))
    ctr = rng.uniform(-1, 1, (nc, 3))
    cr = 10 ** rng.uniform(-3, -0.7, nc)  # some large balls stay suspended high up
    tgt = rng.uniform(-1.2, 1.2, (nt, 3))
    assoc = np.where(rng.uniform(size=nt) < 0.5, rng.integers(0, nc, nt), -1).astype(np.int32)
    return api.Geometry(source_pos=src, center_pos=ctr, center_radius=cr, target_pos=tgt, association=assoc)


CASES = [("config0", lambda: api.config_geometry(0), api.config_fmm(0)),
         ("config2_small", lambda: api.config_geometry(2, level=2, n_volume_targets=3000), api.config_fmm(2)),
         ("cloud", lambda: _cloud(0), api.FmmConfig(p_fmm=8, p_qbx=3, n_max=32)),
         ("clustered", lambda: _cloud(1, clustered=True), api.FmmConfig(p_fmm=8, p_qbx=3, n_max=16)),
         ("one_box", lambda: _cloud(2, 20, 10, 5), api.FmmConfig(p_fmm=4, p_qbx=2, n_max=64)),
         ("no_demotion_tf0", lambda: api.config_geometry(0, level=3), api.config_fmm(0, w_far_demote=0, t_f=0.0)),
         ("torus_small", lambda: api.config_geometry(1, nu=64, nv=32), api.config_fmm(1))]


def test_gpu_plan_refuses_without_device():
    if api.device_count() > 0:
        pytest.skip("device present")
    with pytest.raises(api.CudaError):
        api.Plan(api.config_fmm(0), api.config_geometry(0), device="gpu")


@pytest.mark.gpu
@pytest.mark.parametrize("name,geo,cfg", CASES, ids=[c[0] for c in CASES])
def test_gpu_tree_matches_host(name, geo, cfg):
    g = geo()
    _same(api.Plan(cfg, g), api.Plan(cfg, g, device="gpu", gpu_lists=False))


@pytest.mark.gpu
@pytest.mark.parametrize("name,geo,cfg", CASES, ids=[c[0] for c in CASES])
def test_gpu_plan_with_lists_matches_host(name, geo, cfg):
    g = geo()
    _same(api.Plan(cfg, g), api.Plan(cfg, g, device="gpu"))


@pytest.mark.gpu
def test_gpu_plan_config1_full_size():
    g = api.config_geometry(1)
    cfg = api.config_fmm(1)
    host = api.Plan(cfg, g)
    _same(host, api.Plan(cfg, g, device="gpu", gpu_lists=False), lists=False)
    _same(host, api.Plan(cfg, g, device="gpu"))
