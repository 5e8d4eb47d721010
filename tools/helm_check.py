"""Helmholtz FMM on the GPU against the oracle (debug helper)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_1805_06106_b200 import api  # noqa: E402

K = 3.0
for cfgid, kw, p, q in [(3, dict(level=1), 6, 3), (3, dict(level=1), 10, 5), (2, dict(level=1, n_volume_targets=300), 8, 4)]:
    g = api.config_geometry(cfgid, **kw)
    rng = np.random.default_rng(3)
    w = g.quad_weight * (rng.uniform(-1, 1, g.n_sources) + 1j * rng.uniform(-1, 1, g.n_sources))
    cfg = api.FmmConfig(p_fmm=p, p_qbx=q, n_max=64, kernel=2, helmholtz_k=K)
    plan = api.Plan(cfg, g)
    eng = api.FmmEngine(cfg, g, plan)
    t = time.time()
    pot, cc = eng.apply_complex(w, want_centers=True)
    t = time.time() - t
    ref, cref = O.helm_execute(plan, g, K, p, q, w, want_centers=True)
    e1 = np.linalg.norm(pot - ref) / np.linalg.norm(ref)
    e2 = np.linalg.norm(cc - cref) / np.linalg.norm(cref)
    print(cfgid, kw, p, q, "pot %.3g centres %.3g  (%.2fs)" % (e1, e2, t), flush=True)
    eng.close()
