"""Regenerates tests/golden/oracle_helm_p20_dl.npz: the complex128 Helmholtz oracle
(oracle/helm_oracle.cpp, Stages 2-9 on the host plan) for the double-layer kernel
(kernel 3: the Brakhage-Werner combination S(-i k q mu) + D(q mu n))
at BASELINE config 3's orders (p_fmm = 20, p_qbx = 5, k = 3) on a small procedural sphere
(icosphere level 0, 320 sources, n_max = 16).  The oracle needs minutes at p = 20, so the
GPU test compares against this fixture; geometry, density and plan are deterministic.
    python tests/golden/make_helm_p20_dl.py"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402
from paper_1805_06106_b200 import api  # noqa: E402

K, P, Q, NMAX = 3.0, 20, 5, 16


def inputs():
    g = api.config_geometry(3, level=0)
    rng = np.random.default_rng(5)
    w = g.quad_weight * (rng.uniform(-1, 1, g.n_sources) + 1j * rng.uniform(-1, 1, g.n_sources))
    mu = g.source_normal * w[:, None]  # dipole moments q mu n
    ws = -1j * K * w                    # single-layer weights -i eta q mu, eta = k
    cfg = api.FmmConfig(p_fmm=P, p_qbx=Q, n_max=NMAX, kernel=3, helmholtz_k=K)
    return g, ws, mu, cfg


def main():
    g, ws, mu, cfg = inputs()
    plan = api.Plan(cfg, g)
    pot, cc = O.helm_execute(plan, g, K, P, Q, ws, want_centers=True, mu=mu)
    np.savez_compressed(os.path.join(HERE, "oracle_helm_p20_dl.npz"), weights=ws, dipoles=mu, pot=pot,
                        centres=cc[:64],
                        list_hashes=np.array([plan.list_hashes()[k] for k in sorted(plan.list_hashes())],
                                             dtype=np.uint64))


if __name__ == "__main__":
    main()
