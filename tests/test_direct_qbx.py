"""Unaccelerated QBX: the GPU direct_qbx
against the oracle's, and the FMM's convergence towards it (Theorem 1,
SPEC.md:441, 565)."""
import numpy as np
import pytest

import oracle as O
from paper_1805_06106_b200 import api

TOL = 1e-11


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def test_direct_qbx_rejects_bad_input():
    """Argument checks run on the host before any device work (no GPU needed)."""
    g = api.config_geometry(0)
    w = g.weights()
    bad = api.Geometry(g.source_pos, g.center_pos, g.center_radius, g.target_pos,
                       np.full(g.n_targets, g.n_centers, dtype=np.int32))
    with pytest.raises(ValueError, match="association"):
        api.direct_qbx(bad, w, None, 3)
    with pytest.raises(ValueError, match="p_qbx"):
        api.direct_qbx(g, w, None, 9)
    r = g.center_radius.copy()
    r[5] = 0.0
    with pytest.raises(ValueError, match="centre 5"):
        api.direct_qbx(api.Geometry(g.source_pos, g.center_pos, r, g.target_pos, g.association), w, None, 3)
    with pytest.raises(ValueError):
        api.direct_qbx(g, w[:-1], None, 3)


@pytest.mark.gpu
@pytest.mark.parametrize("dipoles", [False, True])
def test_direct_qbx_matches_oracle(dipoles):
    g = api.config_geometry(2, level=1, n_volume_targets=300)  # associated + conventional targets
    assert (g.association < 0).any() and (g.association >= 0).any()
    w = g.weights()
    mu = g.dipoles() if dipoles else None
    for q in (0, 3, 5):
        pot = api.direct_qbx(g, w, mu, q)
        ref = O.direct_qbx(g, w, mu, q)
        assert rel(pot, ref) <= TOL, (q, rel(pot, ref))


@pytest.mark.gpu
def test_fmm_converges_to_direct_qbx():
    """|FMM - direct QBX| falls with p_fmm at fixed p_qbx (Theorem 1)."""
    g = api.config_geometry(1, nu=32, nv=16)
    w, mu = g.weights(), g.dipoles()
    d = api.direct_qbx(g, w, mu, 5)
    errs = []
    for p in (6, 9, 12, 16):
        pot, _ = api.execute(g, w, mu, api.FmmConfig(p_fmm=p, p_qbx=5, n_max=64, kernel=1))
        errs.append(rel(pot, d))
    assert all(b < a for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-7, errs
