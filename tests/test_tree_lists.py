"""Host tree (Stage 1) and interaction lists vs the definitions.

- lists == brute-force definitional construction on small trees
- list-size bounds |V| <= 875, |X_close| <= 250, |X_far| <= 375
- source-coverage partition for every target box
- TCR ownership / suspension invariants and the build examples
"""
import numpy as np
import pytest

import oracle as O
from paper_1805_06106_b200 import api

NAMES = ("U", "V", "W_close", "W_far", "X_close", "X_far")


def _cases():
    return [
        ("sphere-L1-nmax16", api.config_geometry(0, level=1), api.FmmConfig(p_fmm=6, p_qbx=3, n_max=16)),
        ("sphere-L1-nmax8-tf0.5", api.config_geometry(0, level=1), api.FmmConfig(p_fmm=6, p_qbx=3, n_max=8, t_f=0.5)),
        ("urchin-L1-vol", api.config_geometry(2, level=1, n_volume_targets=300),
         api.FmmConfig(p_fmm=6, p_qbx=3, n_max=24)),
        ("torus-12x6-demote", api.config_geometry(1, nu=12, nv=6),
         api.FmmConfig(p_fmm=6, p_qbx=3, n_max=24, kernel=1, w_far_demote=20)),
        ("urchin-array-small", api.config_geometry(4, variant=8, level=0),
         api.FmmConfig(p_fmm=6, p_qbx=3, n_max=12)),
        ("urchin-vol-level-restricted", api.config_geometry(2, level=1, n_volume_targets=300),
         api.FmmConfig(p_fmm=6, p_qbx=3, n_max=16, level_restrict=1)),
    ]


@pytest.mark.parametrize("name,g,cfg", _cases(), ids=[c[0] for c in _cases()])
def test_lists_equal_bruteforce(name, g, cfg):
    plan = api.Plan(cfg, g)
    brute = O.lists_brute(plan)
    for k, nm in enumerate(NAMES):
        s, b = plan.list_csr(k)
        bs, bb = brute[nm]
        assert np.array_equal(s, bs), f"{nm}: row starts differ"
        assert np.array_equal(b, bb), f"{nm}: contents differ"
    assert plan.view.n_levels >= 3


def _sub_sources(a, d):
    return a["src_sub_start"][d], a["src_sub_count"][d]


@pytest.mark.parametrize("name,g,cfg", _cases()[:4], ids=[c[0] for c in _cases()[:4]])
def test_source_coverage_partition(name, g, cfg):
    """Every source reaches every centre/target of a target box exactly once through
    U, W_close, W_far, X_close of the box and V, X_far of the box or its ancestors."""
    plan = api.Plan(cfg, g)
    a = plan.arrays()
    lists = {nm: plan.list_csr(k) for k, nm in enumerate(NAMES)}
    ns = plan.view.n_sources
    parent = a["box_parent"]
    for b in range(a["n_boxes"]):
        if not a["box_flags"][b] & 1:
            continue
        cnt = np.zeros(ns, dtype=np.int32)

        def add(nm, box, own_only):
            s, e = lists[nm][0][box], lists[nm][0][box + 1]
            for d in lists[nm][1][s:e]:
                if own_only:
                    st, c = a["src_own_start"][d], a["src_own_count"][d]
                else:
                    st, c = _sub_sources(a, d)
                cnt[st:st + c] += 1
        add("U", b, True)
        add("W_close", b, True)
        add("W_far", b, False)
        add("X_close", b, True)
        x = b
        while x >= 0:
            add("V", x, False)
            add("X_far", x, True)
            x = parent[x]
        assert cnt.min() == 1 and cnt.max() == 1, f"box {b}: coverage {cnt.min()}..{cnt.max()}"


def test_list_size_bounds_and_hash_determinism():
    g = api.config_geometry(1, nu=48, nv=24)
    cfg = api.FmmConfig(p_fmm=15, p_qbx=5, n_max=64, kernel=1)
    p1 = api.Plan(cfg, g)
    p2 = api.Plan(cfg, g)
    assert p1.list_hashes() == p2.list_hashes()
    for k, bound in ((1, 875), (4, 250), (5, 375)):
        s, _ = p1.list_csr(k)
        assert np.diff(s).max() <= bound


def test_tree_invariants():
    g = api.config_geometry(2, level=2, n_volume_targets=500)
    cfg = api.FmmConfig(p_fmm=10, p_qbx=3, n_max=32)
    plan = api.Plan(cfg, g)
    a = plan.arrays()
    nb = a["n_boxes"]
    leaf = (a["box_flags"] & 8) > 0
    # sources and conventional targets only in leaves
    assert np.all(a["src_own_count"][~leaf] == 0)
    assert np.all(a["tgt_own_count"][~leaf] == 0)
    # every owned centre fits its box's TCR; suspended ones fit no child's TCR
    cperm = a["ctr_perm"]
    tf = cfg.t_f
    for b in range(nb):
        c0, n = a["ctr_own_start"][b], a["ctr_own_count"][b]
        if n == 0 or b == 0:
            continue
        cb, hb = a["box_center"][b], a["box_radius"][b]
        for i in range(c0, c0 + n):
            c = g.center_pos[cperm[i]]
            r = g.center_radius[cperm[i]]
            assert np.linalg.norm(c - cb) + r <= np.sqrt(3) * hb * (1 + tf) * (1 + 1e-12)
            if not leaf[b]:  # suspension bound, Appendix C.2
                assert r > np.sqrt(3) * (hb / 2) * tf / 2
    # root contains all particles and balls
    rc, rh = a["root_center"], a["root_radius"]
    for pts, rad in ((g.source_pos, 0), (g.center_pos, g.center_radius[:, None])):
        assert np.all(np.abs(pts - rc) + rad <= rh)
    # permutations are permutations
    assert np.array_equal(np.sort(a["src_perm"]), np.arange(g.n_sources))
    assert np.array_equal(np.sort(a["ctr_perm"]), np.arange(g.n_centers))


def test_tree_spec_examples():
    rng = np.random.default_rng(0)
    # 10 particles, n_max 512 -> single root leaf
    g = api.Geometry(rng.uniform(-1, 1, (10, 3)), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)), np.zeros(0, np.int32))
    p = api.Plan(api.FmmConfig(p_fmm=4, p_qbx=2, n_max=512), g)
    assert p.view.n_boxes == 1
    # big centre at the root centre + 1000 sources: the centre stays suspended at the root
    src = rng.uniform(-1, 1, (1000, 3))
    g = api.Geometry(src, np.zeros((1, 3)), np.array([0.9]), np.zeros((0, 3)), np.zeros(0, np.int32))
    p = api.Plan(api.FmmConfig(p_fmm=4, p_qbx=2, n_max=64), g)
    a = p.arrays()
    assert a["ctr_own_count"][0] == 1 and p.view.n_boxes > 1
    # uniform cloud, no centres: depth >= 1 and every leaf <= n_max
    g = api.Geometry(rng.uniform(-1, 1, (4096, 3)), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)), np.zeros(0, np.int32))
    p = api.Plan(api.FmmConfig(p_fmm=4, p_qbx=2, n_max=512), g)
    a = p.arrays()
    leaf = (a["box_flags"] & 8) > 0
    assert p.view.n_levels >= 2 and a["src_own_count"][leaf].max() <= 512


def test_plan_input_errors():
    g = api.config_geometry(0, level=0)
    with pytest.raises(ValueError):
        api.Plan(api.FmmConfig(p_fmm=3, p_qbx=5), g)            # p_qbx > p_fmm
    with pytest.raises(ValueError):
        api.Plan(api.FmmConfig(p_fmm=5, p_qbx=3, t_f=1.5), g)   # t_f >= 2 sqrt 3 - 2
    bad = api.Geometry(g.source_pos, g.center_pos, g.center_radius, g.target_pos, g.association.copy())
    bad.association[0] = 10 ** 6
    with pytest.raises(ValueError):
        api.Plan(api.FmmConfig(p_fmm=5, p_qbx=3), bad)
    nanpos = g.source_pos.copy()
    nanpos[3, 1] = np.nan
    with pytest.raises(ValueError):
        api.Plan(api.FmmConfig(p_fmm=5, p_qbx=3),
                 api.Geometry(nanpos, g.center_pos, g.center_radius, g.target_pos, g.association))


def _leaf_level_violations(a):
    """Pairs of adjacent leaves (closed boxes that touch) more than one level apart."""
    leaf = np.nonzero((a["box_flags"] & 8) > 0)[0]
    c, h, lev = a["box_center"][leaf], a["box_radius"][leaf], a["box_level"][leaf]
    d = np.abs(c[:, None, :] - c[None, :, :]).max(-1)
    adj = d <= (h[:, None] + h[None, :]) * (1 + 1e-12)
    return int((adj & (np.abs(lev[:, None] - lev[None, :]) > 1)).sum() // 2)


@pytest.mark.parametrize("case", ["urchin-vol", "torus"])
def test_level_restriction(case):
    """SPEC.md:397 / Remark C.1: with level_restrict, adjacent leaves
    differ by at most one level; particles and the list invariants are untouched."""
    if case == "urchin-vol":
        g = api.config_geometry(2, level=2, n_volume_targets=2000)
        base = dict(p_fmm=8, p_qbx=4, n_max=16)
    else:
        g = api.config_geometry(1, nu=24, nv=12)
        base = dict(p_fmm=8, p_qbx=4, n_max=24, kernel=1)
    a0 = api.Plan(api.FmmConfig(**base), g).arrays()
    plan = api.Plan(api.FmmConfig(**base, level_restrict=1), g)
    a1 = plan.arrays()
    assert _leaf_level_violations(a0) > 0           # the unrestricted tree does violate it
    assert _leaf_level_violations(a1) == 0
    assert a1["n_boxes"] > a0["n_boxes"]
    for k in ("src_perm", "ctr_perm", "tgt_perm"):
        assert np.array_equal(np.sort(a1[k]), np.sort(a0[k]))
    for k, bound in ((1, 875), (4, 250), (5, 375)):
        s, _ = plan.list_csr(k)
        assert np.diff(s).max() <= bound
    with pytest.raises(ValueError, match="host plan"):
        api.Plan(api.FmmConfig(**base, level_restrict=1), g, device="gpu")
