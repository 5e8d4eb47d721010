cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "orders" > gpurun_out/pytest_p2.log 2>&1
timeout 300 python - > gpurun_out/p2dbg.log 2>&1 <<'PY'
import numpy as np, oracle as O
from paper_1805_06106_b200 import api
g = api.config_geometry(2, level=1, n_volume_targets=500)
for p, q in [(2, 2), (2, 1), (3, 2), (3, 3), (4, 2)]:
    cfg = api.FmmConfig(p_fmm=p, p_qbx=q, n_max=16, t_f=0.9, kernel=1)
    plan = api.Plan(cfg, g)
    w = g.weights(); mu = g.dipoles()
    eng = api.FmmEngine(cfg, g, plan)
    pot, c = eng.apply(w, mu, want_centers=True)
    eng.close()
    ref, cref, _ = O.execute(plan, g, w, mu, want_centers=True)
    led = plan.ledger()
    print(p, q, np.linalg.norm(pot-ref)/np.linalg.norm(ref), np.linalg.norm(c-cref)/np.linalg.norm(cref), led["entries"])
PY
