"""Quick GPU-vs-oracle parity check on small configs (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1805_06106_b200 import api
import oracle as O

def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))

def run(name, g, cfg, dip):
    pl = api.Plan(cfg, g)
    w = g.weights()
    mu = g.dipoles() if dip else None
    t = time.time(); ref, cref, st = O.execute(pl, g, w, mu, want_centers=True); t_o = time.time() - t
    eng = api.FmmEngine(cfg, g, pl)
    t = time.time(); pot, c = eng.apply(w, mu, want_centers=True); t_g = time.time() - t
    tm, launches, _, _ = eng.last_timings()
    pot2 = eng.apply(w, mu)
    print(f"{name}: ns={g.n_sources} nt={g.n_targets} rel_l2 pot={rel(pot, ref):.3e} centres={rel(c, cref):.3e} "
          f"bitwise_rerun={np.array_equal(pot, pot2)} oracle {t_o:.2f}s gpu {t_g*1e3:.1f}ms launches={launches}")
    print("   stage ms:", {k: round(v, 3) for k, v in tm.items()})
    return rel(pot, ref)

if __name__ == "__main__":
    g = api.config_geometry(0); cfg = api.config_fmm(0)
    run("cfg0 SL", g, cfg, False)
    g = api.config_geometry(1, nu=32, nv=16); cfg = api.config_fmm(1)
    run("torus32x16 SL+DL", g, cfg, True)
    g = api.config_geometry(2, level=2, n_volume_targets=3000); cfg = api.config_fmm(2)
    run("urchin L2 + vol", g, cfg, False)
    # direct sum vs reference
    rng = np.random.default_rng(1)
    s = rng.uniform(-1, 1, (3000, 3)); w = rng.uniform(-1, 1, 3000); m = rng.normal(size=(3000, 3))
    t = rng.uniform(-1, 1, (2000, 3)) + 3
    a = api.direct_sum(api.SourceEnsemble(s, w, m), api.TargetSet(t))
    b = O.ref_direct_sum(s, w, m, t)
    print("direct_sum vs reference rel", rel(a, b))
