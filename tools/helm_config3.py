"""Helmholtz BASELINE config 3 on one GPU: create + timed applies (device events)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1805_06106_b200 import api  # noqa: E402


def main():
    level = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    g = api.config_geometry(3, level=level)
    cfg = api.config_fmm(3)
    rng = np.random.default_rng(7)
    w = g.quad_weight * (rng.uniform(-1, 1, g.n_sources) + 1j * rng.uniform(-1, 1, g.n_sources))
    t0 = time.time()
    plan = api.Plan(cfg, g)
    t1 = time.time()
    eng = api.FmmEngine(cfg, g, plan)
    t2 = time.time()
    print(f"config 3 level {level}: {g.n_sources} sources, {g.n_centers} centres; plan {t1 - t0:.1f} s, "
          f"create {t2 - t1:.1f} s", flush=True)
    for i in range(2):
        t = time.time()
        pot = eng.apply_complex(w)
        t = time.time() - t
        tm, nl, _, _ = eng.last_timings()
        print(f"apply {i}: {t * 1e3:.0f} ms wall; stages " + ", ".join(f"{k} {v:.1f}" for k, v in tm.items()),
              flush=True)
    print("checksum", complex(pot.sum()))
    eng.close()


if __name__ == "__main__":
    main()
