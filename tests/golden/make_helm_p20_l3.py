"""Regenerates tests/golden/oracle_helm_p20_l3.npz: the complex128 Helmholtz oracle
(oracle/helm_oracle.cpp, Stages 2-9 on the host plan) at BASELINE config 3's settings
(p_fmm = 20, p_qbx = 5, k = 3, n_max = 64) on the config-3 surface one level coarser
than BASELINE's level 6 twice over: the unit-sphere icosphere at level 3 (1,280
triangles, 20,480 sources, 40,960 centres and targets).  The oracle needs minutes
here, too slow for the test suite, so tests/test_gpu_fullsize.py compares the GPU
against this fixture; geometry, density and host plan are deterministic, so the GPU
box rebuilds identical inputs (checked by the weights and the list hashes).
Stored: all target potentials, and the centre coefficients of every 32nd centre.
    python tests/golden/make_helm_p20_l3.py"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402
from paper_1805_06106_b200 import api  # noqa: E402

K, P, Q, NMAX, LEVEL, STRIDE = 3.0, 20, 5, 64, 3, 32


def inputs():
    g = api.config_geometry(3, level=LEVEL)
    rng = np.random.default_rng(33)
    w = g.quad_weight * (rng.uniform(-1, 1, g.n_sources) + 1j * rng.uniform(-1, 1, g.n_sources))
    cfg = api.config_fmm(3, n_max=NMAX)
    assert (cfg.p_fmm, cfg.p_qbx, cfg.helmholtz_k) == (P, Q, K)
    return g, w, cfg


def hashes(plan):
    h = plan.list_hashes()
    return np.array([h[k] for k in sorted(h)], dtype=np.uint64)


def main():
    g, w, cfg = inputs()
    plan = api.Plan(cfg, g)
    t = time.time()
    pot, cc = O.helm_execute(plan, g, K, P, Q, w, want_centers=True)
    print(f"oracle: {time.time() - t:.1f} s for {g.n_sources} sources")
    np.savez_compressed(os.path.join(HERE, "oracle_helm_p20_l3.npz"), weights=w, pot=pot, centres=cc[::STRIDE],
                        list_hashes=hashes(plan))


if __name__ == "__main__":
    main()
