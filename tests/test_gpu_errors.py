"""Reference error semantics through the FMM apply (SURVEY.md §8b "Errors"):
coincident points raise DomainError the way qbx::direct_sum throws std::domain_error
(/root/reference/proj/src/kernels.cpp:58-71; "domain violations -> error
with box/center diagnostics"); size mismatches raise ValueError before any copy
(SourceEnsemble::validate, kernels.cpp:27-38); Laplace entry points refuse a
Helmholtz handle."""
import dataclasses

import numpy as np
import pytest

from paper_1805_06106_b200 import api

pytestmark = pytest.mark.gpu


def _urchin():
    return api.config_geometry(2, level=1, n_volume_targets=300)


def test_conventional_target_on_source_is_domain_error():
    g = _urchin()
    conv = np.nonzero(g.association < 0)[0]
    assert conv.size > 0
    t = g.target_pos.copy()
    t[conv[7]] = g.source_pos[123]
    g2 = dataclasses.replace(g, target_pos=t)
    cfg = api.config_fmm(2)
    eng = api.FmmEngine(cfg, g2)
    with pytest.raises(api.DomainError, match=f"target {conv[7]} coincides with source 123"):
        eng.apply(g2.weights())
    # the handle stays usable: the same engine on a clean density still raises (geometry
    # is the problem), a fresh engine on the clean geometry does not
    eng.close()
    eng = api.FmmEngine(cfg, g)
    pot = eng.apply(g.weights())
    assert np.all(np.isfinite(pot))
    eng.close()


def test_source_on_qbx_center_is_domain_error():
    g = _urchin()
    s = g.source_pos.copy()
    s[40] = g.center_pos[17]
    g2 = dataclasses.replace(g, source_pos=s)
    eng = api.FmmEngine(api.config_fmm(2), g2)
    with pytest.raises(api.DomainError, match="QBX center 17 coincides with source 40"):
        eng.apply(g2.weights())
    eng.close()


def test_sl_dl_zero_weight_coincidence_still_raises():
    """A coincident pair with zero weight contributes 0 * inf = NaN: still a domain error."""
    g = api.config_geometry(4, variant=8, level=1)
    s = g.source_pos.copy()
    s[5] = g.center_pos[2]
    g2 = dataclasses.replace(g, source_pos=s)
    d = g2.density.copy()
    d[5] = 0.0
    eng = api.FmmEngine(api.config_fmm(4), g2)
    with pytest.raises(api.DomainError, match="QBX center 2 coincides with source 5"):
        eng.apply(g2.weights(d), g2.dipoles(d))
    eng.close()


def test_apply_size_validation():
    g = _urchin()
    eng = api.FmmEngine(api.config_fmm(2), g)
    with pytest.raises(ValueError, match="weights for"):
        eng.apply(g.weights()[:-1])
    eng.close()
    g4 = api.config_geometry(4, variant=8, level=1)
    eng = api.FmmEngine(api.config_fmm(4), g4)
    with pytest.raises(ValueError, match="requires dipole"):
        eng.apply(g4.weights())
    with pytest.raises(ValueError, match="dipole moments for"):
        eng.apply(g4.weights(), g4.dipoles()[:-2])
    eng.close()


def test_helmholtz_handle_rejects_laplace_entry_points():
    g = api.config_geometry(3, level=1)
    cfg = api.config_fmm(3, p_fmm=6, p_qbx=3)
    eng = api.FmmEngine(cfg, g)
    w = np.ones(g.n_sources)
    with pytest.raises(ValueError, match="Helmholtz"):
        eng.apply_batch(np.stack([w, w]))
    with pytest.raises(ValueError, match="Helmholtz"):
        eng.apply(w)
    eng.close()
