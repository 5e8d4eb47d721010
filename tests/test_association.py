"""Target association (Algorithm 3) and area queries (Algorithm 5) on the GPU
 against the brute-force oracle (oracle/assoc_brute.cpp):
bit-exact association arrays and leaf lists, the spec's examples
(SPEC.md:299-304), ties, empty inputs, and full-size properties
on BASELINE config 2."""
import numpy as np
import pytest

import oracle as O
from paper_1805_06106_b200 import api


def _cloud(seed=0, ns=3000, nc=2000, nt=20000):
    rng = np.random.default_rng(seed)
    src = rng.uniform(-1, 1, (ns, 3))
    dr = rng.uniform(0.01, 0.05, ns)
    ctr = rng.uniform(-1, 1, (nc, 3))
    cr = rng.uniform(0.02, 0.06, nc)
    tgt = rng.uniform(-1.05, 1.05, (nt, 3))
    return src, dr, ctr, cr, tgt


def _sc_geometry(src, ctr, cr):
    """Sources + centres only: the tree Algorithm 3 queries."""
    return api.Geometry(source_pos=src, center_pos=ctr, center_radius=cr, target_pos=np.zeros((0, 3)),
                        association=np.zeros(0, dtype=np.int32))


def _locator(src, dr, ctr, cr, side=None, n_max=32):
    g = _sc_geometry(src, ctr, cr)
    plan = api.Plan(api.FmmConfig(p_fmm=4, p_qbx=2, n_max=n_max), g)
    return api.Locator(plan, g, dr, side), plan


def _surface(cfg=0, **kw):
    g = api.config_geometry(cfg, **kw)
    side = np.where(np.arange(g.n_centers) % 2 == 0, 1, -1).astype(np.int8)  # centre 2s: x + r n
    nsurf = 2 * g.n_sources
    pref = np.where(np.arange(nsurf) % 2 == 0, 1, -1).astype(np.int8)
    return g, side, pref


# ---------------------------------------------------------------- oracle (CPU)
def test_oracle_spec_examples():
    src = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    dr = np.array([0.5, 0.5])
    ctr = np.array([[0.0, 0.2, 0], [1.0, 0.2, 0], [0.0, -0.2, 0]])
    cr = np.array([0.2, 0.2, 0.2])
    tgt = np.array([[0.0, 0.2, 0],     # coincident with centre 0 -> associated, distance 0
                    [5.0, 5.0, 5.0],   # farther than r_danger from every source -> not endangered
                    [0.0, 0.0, 0.0],   # equidistant from centres 0 and 2 -> lowest id
                    [0.3, -0.35, 0.0]])  # endangered, no centre within r_c (1 + eps) -> flagged
    a, nf = O.associate_targets(src, dr, ctr, cr, tgt, eps_ta=0.05)
    assert a.tolist() == [0, -1, 0, -2] and nf == 1
    b, _ = O.associate_targets(src, dr, ctr, cr, tgt[2:3], eps_ta=0.05, center_side=[1, 1, -1], side_pref=[-1])
    assert b.tolist() == [2]


def test_oracle_area_query_trivial_trees():
    g = _sc_geometry(np.array([[0.1, 0.2, 0.3], [-0.2, 0.1, 0.0]]), np.zeros((0, 3)), np.zeros(0))
    plan = api.Plan(api.FmmConfig(p_fmm=2, p_qbx=1, n_max=8), g)
    assert plan.view.n_boxes == 1
    st, lv = O.area_query(plan, [[0.0, 0.0, 0.0], [9.0, 9.0, 9.0]], [0.01, 0.01])
    assert st.tolist() == [0, 1, 1] and lv.tolist() == [0]  # single-box tree -> {root}
    src, dr, ctr, cr, _ = _cloud(1, 500, 300, 0)
    loc_plan = api.Plan(api.FmmConfig(p_fmm=4, p_qbx=2, n_max=16), _sc_geometry(src, ctr, cr))
    a = loc_plan.arrays()
    leaves = np.flatnonzero(np.diff(a["child_starts"]) == 0)
    st, lv = O.area_query(loc_plan, [a["root_center"]], [a["root_radius"]])
    assert lv.tolist() == leaves.tolist()  # query radius = root radius -> all leaves


def test_host_validation_before_device_work():
    src, dr, ctr, cr, _ = _cloud(2, 50, 20, 0)
    g = _sc_geometry(src, ctr, cr)
    plan = api.Plan(api.FmmConfig(p_fmm=4, p_qbx=2, n_max=16), g)
    with pytest.raises(ValueError):
        api.Locator(plan, g, dr[:-1])
    bad = dr.copy()
    bad[3] = -1.0
    with pytest.raises(ValueError, match="danger radius"):
        api.Locator(plan, g, bad)
    with pytest.raises(ValueError):
        api.Locator(plan, g, dr, center_side=np.ones(5, dtype=np.int8))


# ---------------------------------------------------------------- GPU parity
@pytest.mark.gpu
@pytest.mark.parametrize("seed,eps", [(0, 0.0), (1, 0.1), (2, 0.5)])
def test_gpu_associate_random_cloud(seed, eps):
    src, dr, ctr, cr, tgt = _cloud(seed)
    loc, _ = _locator(src, dr, ctr, cr)
    a, nf = loc.associate(tgt, eps)
    ref, nref = O.associate_targets(src, dr, ctr, cr, tgt, eps)
    assert np.array_equal(a, ref) and nf == nref
    assert (a >= 0).any() and (a == -1).any()
    loc.close()


@pytest.mark.gpu
def test_gpu_associate_ties_and_sides():
    """Targets equidistant from two centres (mirror pairs) go to the lower id; with
    side preferences only same-side centres count."""
    rng = np.random.default_rng(5)
    grid = rng.choice(32 ** 3, 400, replace=False)  # distinct points of a 1/16 grid
    base = np.c_[grid % 32, (grid // 32) % 32, grid // 1024] / 16.0 - 1.0
    h = 1.0 / 64  # exactly representable: node i is exactly h from centres i and 400 + i
    ctr = np.concatenate([base + [0, 0, h], base - [0, 0, h]])
    cr = np.full(len(ctr), h)
    src = base.copy()
    dr = np.full(len(src), 0.3)
    side = np.r_[np.ones(400), -np.ones(400)].astype(np.int8)
    tgt = np.concatenate([base, base + rng.normal(scale=0.03, size=base.shape)])
    loc, _ = _locator(src, dr, ctr, cr, side, n_max=8)
    a, nf = loc.associate(tgt, 0.05)
    ref, nref = O.associate_targets(src, dr, ctr, cr, tgt, 0.05)
    assert np.array_equal(a, ref) and nf == nref
    assert np.array_equal(a[:400], np.arange(400))  # exact ties at the nodes -> the lower id
    pref = np.where(rng.uniform(size=len(tgt)) < 0.5, 1, -1).astype(np.int8)
    b, nb = loc.associate(tgt, 0.05, side_pref=pref)
    ref2, nref2 = O.associate_targets(src, dr, ctr, cr, tgt, 0.05, center_side=side, side_pref=pref)
    assert np.array_equal(b, ref2) and nb == nref2
    ok = b >= 0
    assert np.all(side[b[ok]] == pref[ok])
    loc.close()


@pytest.mark.gpu
def test_gpu_associate_empty_and_far():
    src, dr, ctr, cr, _ = _cloud(3, 200, 100, 0)
    loc, _ = _locator(src, dr, ctr, cr)
    a, nf = loc.associate(np.zeros((0, 3)))
    assert a.shape == (0,) and nf == 0
    far = np.array([[50.0, 0, 0], [0, -80.0, 3.0]])  # outside the root cube
    a, nf = loc.associate(far, 0.1)
    assert a.tolist() == [-1, -1] and nf == 0
    loc.close()


@pytest.mark.gpu
def test_gpu_surface_nodes_associate_without_flags():
    """on-surface nodes of a refined sphere with eps = 0.05 -> no flagged
    targets; equal to the oracle with and without side preferences."""
    g, side, pref = _surface(0)
    dr = api.danger_radius_of(g)
    loc, _ = _locator(g.source_pos, dr, g.center_pos, g.center_radius, side, n_max=64)
    t = g.target_pos[:2 * g.n_sources]
    for sp, cs in ((pref, side), (None, None)):
        a, nf = loc.associate(t, 0.05, side_pref=sp)
        ref, nref = O.associate_targets(g.source_pos, dr, g.center_pos, g.center_radius, t, 0.05,
                                        center_side=cs, side_pref=sp)
        assert np.array_equal(a, ref) and nf == nref == 0
        assert np.all(a >= 0)
    loc.close()


@pytest.mark.gpu
def test_gpu_area_query_matches_leaf_scan():
    """500 random queries on a random tree equal the brute-force leaf scan."""
    src, dr, ctr, cr, _ = _cloud(4, 4000, 2000, 0)
    loc, plan = _locator(src, dr, ctr, cr, n_max=16)
    a = plan.arrays()
    rng = np.random.default_rng(9)
    qc = rng.uniform(-1.1, 1.1, (500, 3))
    qr = 10 ** rng.uniform(-3, 0, 500)
    # plus exact-contact cases: balls touching a leaf face / corner, zero radius at a box centre
    lv_ids = np.flatnonzero(np.diff(a["child_starts"]) == 0)[:20]
    bc, br = a["box_center"][lv_ids], a["box_radius"][lv_ids]
    qc = np.concatenate([qc, bc + np.c_[br + 0.01, np.zeros((20, 2))], bc + br[:, None] + 0.02, bc])
    qr = np.concatenate([qr, np.full(20, 0.01), np.full(20, 0.02), np.zeros(20)])
    st, lv = loc.area_query(qc, qr)
    rst, rlv = O.area_query(plan, qc, qr)
    assert np.array_equal(st, rst) and np.array_equal(lv, rlv)
    st, lv = loc.area_query([a["root_center"]], [a["root_radius"]])
    assert lv.tolist() == np.flatnonzero(np.diff(a["child_starts"]) == 0).tolist()
    loc.close()


@pytest.mark.gpu
def test_gpu_config2_full_size():
    """BASELINE config 2 at full size: the 1M-candidate volume targets kept by the
    generator (none within r of a node) are all conventional; every on-surface node
    finds its side's centre; a 3,000-target sample of each is bit-exact vs the oracle."""
    g, side, pref = _surface(2)
    dr = api.danger_radius_of(g)
    loc, _ = _locator(g.source_pos, dr, g.center_pos, g.center_radius, side, n_max=64)
    nsurf = 2 * g.n_sources
    t = g.target_pos
    sp = np.r_[pref, np.zeros(len(t) - nsurf, dtype=np.int8)]
    a, nf = loc.associate(t, 0.05, side_pref=sp)
    assert nf == 0
    assert np.all(a[nsurf:] == -1)
    assert np.all(a[:nsurf] >= 0)
    assert np.all(side[a[:nsurf]] == pref)
    rng = np.random.default_rng(0)
    pick = np.r_[rng.choice(nsurf, 3000, replace=False), nsurf + rng.choice(len(t) - nsurf, 3000, replace=False)]
    ref, _ = O.associate_targets(g.source_pos, dr, g.center_pos, g.center_radius, t[pick], 0.05,
                                 center_side=side, side_pref=sp[pick])
    assert np.array_equal(a[pick], ref)
    loc.close()
