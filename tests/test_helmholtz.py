"""Helmholtz single and double layer (BASELINE config 3; north_star
"Helmholtz single- and double-layer"; the Brakhage-Werner representation of
PAPER.md:3074-3075 is S(-i eta mu) + D(mu)): the complex128 CPU
oracle (oracle/helm_oracle.cpp) pinned against analytic anchors, since no reference
implementation exists (parity unpinned):
special functions and Gaunt coefficients against scipy, the Gegenbauer expansion and
the three translation theorems against direct sums, and the FMM converging to direct
QBX on the same tree and lists."""
from math import factorial

import numpy as np
import pytest
from scipy.special import lpmv, spherical_jn, spherical_yn

import oracle as O
from paper_1805_06106_b200 import api

K = 3.0  # config 3 wavenumber


def _pbar(n, a, x):
    return np.sqrt((2 * n + 1) / (4 * np.pi) * factorial(n - a) / factorial(n + a)) * lpmv(a, n, x) * (-1) ** a


@pytest.mark.parametrize("x", [1e-3, 0.3, 0.999, 1.0, 2.5, 7.0, 25.0])
def test_spherical_bessel_hankel(x):
    j, h = O.helm_bessel(20, x)
    n = np.arange(21)
    jr, yr = spherical_jn(n, x), spherical_yn(n, x)
    assert np.max(np.abs(j - jr) / np.abs(jr)) < 1e-12
    assert np.max(np.abs(h.imag - yr) / np.abs(yr)) < 1e-12
    assert np.array_equal(h.real, j)


def test_harmonics_and_gaunt():
    v = np.array([0.3, -0.5, 0.8])
    r = np.linalg.norm(v)
    th, ph = np.arccos(v[2] / r), np.arctan2(v[1], v[0])
    for n, m in [(0, 0), (3, 2), (7, -5), (20, 13)]:
        ref = _pbar(n, abs(m), np.cos(th)) * np.exp(1j * m * ph)
        assert abs(O.helm_ylm(n, m, v) - ref) <= 1e-14 * abs(ref) + 1e-300
    xg, wg = np.polynomial.legendre.leggauss(90)
    for n, m, n2, m2, l in [(3, 2, 5, -1, 4), (10, 3, 12, 7, 6), (20, -5, 20, 8, 38), (4, 1, 2, 1, 3)]:
        ref = 2 * np.pi * np.sum(wg * _pbar(n, abs(m), xg) * _pbar(n2, abs(m2), xg) * _pbar(l, abs(m - m2), xg))
        assert abs(O.helm_gaunt(n, m, n2, m2, l) - ref) <= 1e-13


def test_expansions_and_translations():
    rng = np.random.default_rng(1)
    src = rng.normal(size=(20, 3)) * 0.1
    w = rng.normal(size=20) + 1j * rng.normal(size=20)
    c, P = np.zeros(3), 16
    t_far = np.array([1.3, -0.7, 0.9])
    direct = O.helm_direct_sum(K, src, w, t_far[None])[0]
    M = O.helm_form(0, K, src, w, c, P)
    assert abs(O.helm_eval(0, K, M, P, c, t_far) - direct) < 1e-12 * abs(direct)
    far = src + np.array([2.0, 0.0, 0.0])
    tn = np.array([0.05, -0.08, 0.03])
    L = O.helm_form(1, K, far, w, c, P)
    assert abs(O.helm_eval(1, K, L, P, c, tn) - O.helm_direct_sum(K, far, w, tn[None])[0]) < 1e-13
    C = np.array([0.1, 0.05, -0.1])  # M2M
    M2 = O.helm_translate(0, K, M, P, c, C, P)
    assert abs(O.helm_eval(0, K, M2, P, C, t_far) - direct) < 1e-9 * abs(direct)
    C2 = np.array([1.5, 0.4, 0.2])  # M2L
    tt = C2 + np.array([0.05, 0.02, -0.04])
    L2 = O.helm_translate(1, K, M, P, c, C2, P)
    ref = O.helm_direct_sum(K, src, w, tt[None])[0]
    assert abs(O.helm_eval(1, K, L2, P, C2, tt) - ref) < 1e-11 * abs(ref)
    C3 = C2 + np.array([0.03, -0.02, 0.01])  # L2L (exact up to the truncated tail)
    L3 = O.helm_translate(2, K, L2, P, C2, C3, P)
    assert abs(O.helm_eval(1, K, L3, P, C3, tt) - O.helm_eval(1, K, L2, P, C2, tt)) < 1e-12 * abs(ref)


def _config3_small(level=1, seed=3):
    g = api.config_geometry(3, level=level)
    rng = np.random.default_rng(seed)
    mu = rng.uniform(-1, 1, g.n_sources) + 1j * rng.uniform(-1, 1, g.n_sources)  # Re, Im ~ U[-1,1]
    return g, g.quad_weight * mu


def test_direct_sum_reciprocity():
    rng = np.random.default_rng(2)
    a, b = rng.normal(size=(30, 3)), rng.normal(size=(40, 3)) + 3.0
    wa, wb = rng.normal(size=30) + 1j * rng.normal(size=30), rng.normal(size=40) + 1j * rng.normal(size=40)
    # sum_b wb phi_a(b) == sum_a wa phi_b(a): G_k is symmetric
    lhs = np.sum(wb * O.helm_direct_sum(K, a, wa, b))
    rhs = np.sum(wa * O.helm_direct_sum(K, b, wb, a))
    assert abs(lhs - rhs) < 1e-12 * abs(lhs)


def test_fmm_converges_to_direct_qbx():
    """Theorem 1 analogue: the Helmholtz FMM error against direct QBX falls with p."""
    g, w = _config3_small(level=1)
    d = O.helm_direct_qbx(K, g, w, 3)
    errs = []
    for p in (3, 5, 8):
        plan = api.Plan(api.FmmConfig(p_fmm=p, p_qbx=3, n_max=64, kernel=0), g)  # kernel-independent tree
        f = O.helm_execute(plan, g, K, p, 3, w)
        errs.append(float(np.linalg.norm(f - d) / np.linalg.norm(d)))
    assert errs[0] > errs[1] > errs[2], errs
    assert errs[2] < 1e-5, errs


def _dl_inputs(n, seed, scale=0.1):
    rng = np.random.default_rng(seed)
    src = rng.normal(size=(n, 3)) * scale
    w = rng.normal(size=n) + 1j * rng.normal(size=n)
    mu = rng.normal(size=(n, 3)) + 1j * rng.normal(size=(n, 3))
    return src, w, mu


def test_dipole_ladder_identities_vs_finite_differences():
    """The oracle's dipole expansion terms (mu . grad_s of the source's multipole / local
    coefficients, via the ladder identities of helm_oracle.cpp grad_dot) against
    4th-order central differences of the monopole coefficients."""
    rng = np.random.default_rng(7)
    for kind, c in ((0, np.array([0.02, -0.01, 0.03])), (1, np.array([1.1, 0.6, -0.4]))):
        for _ in range(3):
            s = rng.normal(size=(1, 3)) * 0.2
            mu = rng.normal(size=(1, 3)) + 1j * rng.normal(size=(1, 3))
            P = 12
            dl = O.helm_form(kind, K, s, np.zeros(1), c, P, mu=mu)
            h = 1e-3
            fd = np.zeros_like(dl)
            for d in range(3):
                e = np.zeros((1, 3))
                e[0, d] = h
                f = [O.helm_form(kind, K, s + j * e, np.ones(1), c, P) for j in (-2, -1, 1, 2)]
                fd = fd + mu[0, d] * (f[0] - 8 * f[1] + 8 * f[2] - f[3]) / (12 * h)
            assert np.linalg.norm(dl - fd) <= 1e-9 * np.linalg.norm(fd), (kind, np.linalg.norm(dl - fd))


def test_double_layer_expansions_vs_direct_sum():
    """Multipole (P2M) and local (P2L) expansions of monopoles + dipoles reproduce the
    closed-form kernel w G_k + mu . grad_y G_k = [w + mu.(x-y)(1 - ikr)/r^2] e^{ikr}/(4 pi r)."""
    src, w, mu = _dl_inputs(25, 5)
    c, P = np.zeros(3), 18
    t_far = np.array([1.4, -0.6, 1.0])
    direct = O.helm_direct_sum(K, src, w, t_far[None], mu=mu)[0]
    M = O.helm_form(0, K, src, w, c, P, mu=mu)
    assert abs(O.helm_eval(0, K, M, P, c, t_far) - direct) < 1e-11 * abs(direct)
    far = src + np.array([2.0, 0.0, 0.0])
    tn = np.array([0.05, -0.08, 0.03])
    L = O.helm_form(1, K, far, w, c, P, mu=mu)
    ref = O.helm_direct_sum(K, far, w, tn[None], mu=mu)[0]
    assert abs(O.helm_eval(1, K, L, P, c, tn) - ref) < 1e-12 * abs(ref)
    # the dipole kernel is the source gradient of the monopole kernel (finite differences)
    h = 1e-4
    dd = 0
    for d in range(3):
        e = np.zeros(3)
        e[d] = h
        dd += mu[0, d] * (O.helm_direct_sum(K, src[:1] + e, [1.0], tn[None])[0] -
                          O.helm_direct_sum(K, src[:1] - e, [1.0], tn[None])[0]) / (2 * h)
    one = O.helm_direct_sum(K, src[:1], [0.0], tn[None], mu=mu[:1])[0]
    assert abs(one - dd) < 1e-6 * abs(dd)


def test_double_layer_fmm_converges_to_direct_qbx():
    """Brakhage-Werner-type combination S(w) + D(mu) through the oracle FMM, converging to
    direct QBX with p on the same tree and lists."""
    g, w = _config3_small(level=1)
    mu = g.source_normal * (g.quad_weight * np.conj(w))[:, None]
    d = O.helm_direct_qbx(K, g, w, 3, mu=mu)
    errs = []
    for p in (3, 5, 8):
        plan = api.Plan(api.FmmConfig(p_fmm=p, p_qbx=3, n_max=64, kernel=0), g)
        f = O.helm_execute(plan, g, K, p, 3, w, mu=mu)
        errs.append(float(np.linalg.norm(f - d) / np.linalg.norm(d)))
    assert errs[0] > errs[1] > errs[2], errs
    assert errs[2] < 1e-5, errs


def test_gpu_entry_points_validate_on_host():
    """Argument checks of the GPU Helmholtz entry points run before any device work."""
    g, w = _config3_small(level=1)
    with pytest.raises(ValueError):
        api.helm_direct_sum(-1.0, g.source_pos, w, g.target_pos[:5])
    with pytest.raises(ValueError):
        api.helm_direct_qbx(K, g, w, 9)
    with pytest.raises(ValueError):
        api.helm_direct_qbx(K, g, w[:-1], 3)


@pytest.mark.gpu
def test_gpu_helm_direct_sum_matches_oracle():
    g, w = _config3_small(level=1)
    t = g.target_pos[:700] + 0.01
    pot = api.helm_direct_sum(K, g.source_pos, w, t)
    ref = O.helm_direct_sum(K, g.source_pos, w, t)
    assert np.linalg.norm(pot - ref) / np.linalg.norm(ref) <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("q", [0, 3, 5])
def test_gpu_helm_direct_qbx_matches_oracle(q):
    g, w = _config3_small(level=1)
    pot = api.helm_direct_qbx(K, g, w, q)
    ref = O.helm_direct_qbx(K, g, w, q)
    assert np.linalg.norm(pot - ref) / np.linalg.norm(ref) <= 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("cfgid,kw,p,q", [(3, dict(level=1), 6, 3), (3, dict(level=1), 10, 5),
                                          (2, dict(level=1, n_volume_targets=300), 8, 4)])
def test_gpu_helmholtz_fmm_matches_oracle(cfgid, kw, p, q):
    """Stages 2-9 for G_k on the GPU (qbxg_apply_complex) against the oracle on the same plan."""
    g = api.config_geometry(cfgid, **kw)
    rng = np.random.default_rng(3)
    w = g.quad_weight * (rng.uniform(-1, 1, g.n_sources) + 1j * rng.uniform(-1, 1, g.n_sources))
    cfg = api.FmmConfig(p_fmm=p, p_qbx=q, n_max=64, kernel=2, helmholtz_k=K)
    plan = api.Plan(cfg, g)
    eng = api.FmmEngine(cfg, g, plan)
    pot, cc = eng.apply_complex(w, want_centers=True)
    again = eng.apply_complex(w)
    eng.close()
    ref, cref = O.helm_execute(plan, g, K, p, q, w, want_centers=True)
    assert np.linalg.norm(pot - ref) / np.linalg.norm(ref) <= 1e-11
    assert np.linalg.norm(cc - cref) / np.linalg.norm(cref) <= 1e-11
    assert np.array_equal(pot, again), "Helmholtz apply is not bitwise deterministic"


def test_helmholtz_handle_rejects_real_apply():
    """A Helmholtz plan needs a wavenumber; a Laplace call on it is refused (host-side checks)."""
    g = api.config_geometry(0)
    with pytest.raises(ValueError, match="wavenumber"):
        api.Plan(api.FmmConfig(p_fmm=6, p_qbx=3, kernel=2, helmholtz_k=0.0), g)


@pytest.mark.gpu
def test_gpu_helmholtz_p20_matches_oracle_fixture():
    """BASELINE config 3's orders (p = 20, q = 5, k = 3: the point-and-shoot M2L at its largest
    blocks) against the oracle, via tests/golden/oracle_helm_p20.npz (the oracle needs minutes at
    p = 20; tests/golden/make_helm_p20.py regenerates it).  Same procedural inputs and plan,
    checked by the list hashes."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    import make_helm_p20 as M
    fx = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_helm_p20.npz"))
    g, w, cfg = M.inputs()
    assert np.array_equal(w, fx["weights"])
    plan = api.Plan(cfg, g)
    hashes = np.array([plan.list_hashes()[k] for k in sorted(plan.list_hashes())], dtype=np.uint64)
    assert np.array_equal(hashes, fx["list_hashes"])
    eng = api.FmmEngine(cfg, g, plan)
    pot, cc = eng.apply_complex(w, want_centers=True)
    eng.close()
    assert np.linalg.norm(pot - fx["pot"]) / np.linalg.norm(fx["pot"]) <= 1e-11
    assert np.linalg.norm(cc[:64] - fx["centres"]) / np.linalg.norm(fx["centres"]) <= 1e-11


# ---------------------------------------------------------------- double layer on the GPU
def _bw_dipoles(g, w):
    """Brakhage-Werner-style dipole moments m = q mu n for the density of w = q mu."""
    return g.source_normal * w[:, None]


@pytest.mark.gpu
def test_gpu_helm_direct_sum_double_layer_matches_oracle():
    g, w = _config3_small(level=1)
    mu = _bw_dipoles(g, w)
    t = g.target_pos[:700] * 1.01
    pot = api.helm_direct_sum(K, g.source_pos, -1j * 3.0 * w, t, dipoles=mu)
    ref = O.helm_direct_sum(K, g.source_pos, -1j * 3.0 * w, t, mu=mu)
    assert np.linalg.norm(pot - ref) / np.linalg.norm(ref) <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("q", [0, 3, 5])
def test_gpu_helm_direct_qbx_double_layer_matches_oracle(q):
    g, w = _config3_small(level=1)
    mu = _bw_dipoles(g, w)
    pot = api.helm_direct_qbx(K, g, w, q, dipoles=mu)
    ref = O.helm_direct_qbx(K, g, w, q, mu=mu)
    assert np.linalg.norm(pot - ref) / np.linalg.norm(ref) <= 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("cfgid,kw,p,q", [(3, dict(level=1), 6, 3), (3, dict(level=1), 12, 5),
                                          (2, dict(level=1, n_volume_targets=300), 8, 4)])
def test_gpu_helmholtz_double_layer_fmm_matches_oracle(cfgid, kw, p, q):
    """Helmholtz SL+DL (kernel 3) through qbxg_apply_complex against the oracle on the same
    plan: the Brakhage-Werner combination S(-i eta q mu) + D(q mu n), eta = k."""
    g = api.config_geometry(cfgid, **kw)
    rng = np.random.default_rng(4)
    w = g.quad_weight * (rng.uniform(-1, 1, g.n_sources) + 1j * rng.uniform(-1, 1, g.n_sources))
    mu = _bw_dipoles(g, w)
    ws = -1j * K * w
    cfg = api.FmmConfig(p_fmm=p, p_qbx=q, n_max=64, kernel=3, helmholtz_k=K)
    plan = api.Plan(cfg, g)
    eng = api.FmmEngine(cfg, g, plan)
    pot, cc = eng.apply_complex(ws, mu, want_centers=True)
    again = eng.apply_complex(ws, mu)
    with pytest.raises(ValueError, match="requires dipole"):
        eng.apply_complex(ws)
    eng.close()
    ref, cref = O.helm_execute(plan, g, K, p, q, ws, want_centers=True, mu=mu)
    assert np.linalg.norm(pot - ref) / np.linalg.norm(ref) <= 1e-11
    assert np.linalg.norm(cc - cref) / np.linalg.norm(cref) <= 1e-11
    assert np.array_equal(pot, again), "Helmholtz SL+DL apply is not bitwise deterministic"


@pytest.mark.gpu
def test_gpu_helmholtz_double_layer_p20_matches_oracle_fixture():
    """Helmholtz SL+DL (kernel 3, Brakhage-Werner) at BASELINE config 3's orders (p = 20,
    q = 5, k = 3) against the oracle via tests/golden/oracle_helm_p20_dl.npz
    (tests/golden/make_helm_p20_dl.py regenerates it); same procedural inputs and plan,
    checked by the list hashes."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    import make_helm_p20_dl as M
    fx = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_helm_p20_dl.npz"))
    g, ws, mu, cfg = M.inputs()
    assert np.array_equal(ws, fx["weights"]) and np.array_equal(mu, fx["dipoles"])
    plan = api.Plan(cfg, g)
    hashes = np.array([plan.list_hashes()[k] for k in sorted(plan.list_hashes())], dtype=np.uint64)
    assert np.array_equal(hashes, fx["list_hashes"])
    eng = api.FmmEngine(cfg, g, plan)
    pot, cc = eng.apply_complex(ws, mu, want_centers=True)
    eng.close()
    assert np.linalg.norm(pot - fx["pot"]) / np.linalg.norm(fx["pot"]) <= 1e-11
    assert np.linalg.norm(cc[:64] - fx["centres"]) / np.linalg.norm(fx["centres"]) <= 1e-11
