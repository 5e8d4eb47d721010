"""Regenerates the golden fixtures in this directory from the REFERENCE's own
qbx::direct_sum (/root/reference/proj/src/kernels.cpp:46-73, compiled unmodified
into oracle/_ref/libqbxref.so by oracle/Makefile).  Run in the build container,
where /root/reference exists:  python tests/golden/make_golden.py
The fixtures travel with the repo; the tests never need the reference itself."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402
from paper_1805_06106_b200 import api  # noqa: E402


def main():
    if O.ref_lib() is None:
        raise SystemExit("oracle/_ref not built: the reference sources are needed to regenerate")
    rng = np.random.default_rng(20181805)
    # (1) random clouds, SL and SL+DL
    src = rng.uniform(-1, 1, (300, 3))
    w = rng.uniform(-1, 1, 300)
    mu = rng.normal(size=(300, 3))
    tgt = rng.uniform(-2, 2, (200, 3))
    np.savez_compressed(os.path.join(HERE, "ref_direct_sum_cloud.npz"), source_pos=src, weights=w, dipoles=mu,
                        target_pos=tgt, pot_sl=O.ref_direct_sum(src, w, None, tgt),
                        pot_sldl=O.ref_direct_sum(src, w, mu, tgt))
    # (2) BASELINE config 0 sources (sphere, 5,120 nodes, seeded uniform density) with SL+DL
    #     weights, at 400 off-surface conventional targets (|x| in [1.2, 2] and [0.3, 0.8])
    g = api.config_geometry(0)
    wt, dp = g.weights(), g.dipoles()
    d = rng.normal(size=(400, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    rad = np.r_[rng.uniform(1.2, 2.0, 200), rng.uniform(0.3, 0.8, 200)]
    t0 = d * rad[:, None]
    np.savez_compressed(os.path.join(HERE, "ref_direct_sum_config0.npz"), target_pos=t0,
                        pot_sl=O.ref_direct_sum(g.source_pos, wt, None, t0),
                        pot_sldl=O.ref_direct_sum(g.source_pos, wt, dp, t0))
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
