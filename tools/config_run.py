"""Device-resident apply time of any BASELINE config on one GPU (CUDA events, after one
warm-up apply), one JSON line per config: sizes, ms per apply, (N_S + N_T)/s, stages.

    python tools/config_run.py [config ...]      (default: 0 1 2 3)

Config 3 (Helmholtz) takes a complex density; config 4 has its own tool (config4_run.py).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_06106_b200 import api  # noqa: E402


def run(cfg_id, reps=3):
    t0 = time.time()
    g = api.config_geometry(cfg_id)
    cfg = api.config_fmm(cfg_id)
    plan = api.Plan(cfg, g, device="gpu")
    eng = api.FmmEngine(cfg, g, plan)
    t_setup = time.time() - t0
    stage = {}
    if cfg_id == 3:
        rng = np.random.default_rng(7)
        w = g.quad_weight * (rng.uniform(-1, 1, g.n_sources) + 1j * rng.uniform(-1, 1, g.n_sources))
        eng.apply_complex(w)
        torch.cuda.synchronize()
        t = time.time()
        for _ in range(reps):
            eng.apply_complex(w)
            for k, v in eng.last_timings()[0].items():
                stage[k] = stage.get(k, 0.0) + v / reps
        ms = (time.time() - t) * 1e3 / reps  # host buffers (H2D + D2H inside)
        timing = "wall clock per apply_complex, host buffers"
    else:
        w = torch.from_numpy(g.weights()).cuda()
        mu = torch.from_numpy(np.ascontiguousarray(g.dipoles())).cuda() if cfg.kernel == 1 else None
        pot = torch.empty(g.n_targets, dtype=torch.float64, device="cuda")
        args = (w.data_ptr(), mu.data_ptr() if mu is not None else None, pot.data_ptr())
        eng.apply_device(*args)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            eng.apply_device(*args)
            for k, v in eng.last_timings()[0].items():
                stage[k] = stage.get(k, 0.0) + v / reps
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        timing = "CUDA events, inputs in HBM"
    led = plan.ledger()
    out = {"config": cfg_id, "n_sources": g.n_sources, "n_targets": g.n_targets, "n_centers": g.n_centers,
           "n_conventional_targets": int((g.association < 0).sum()), "n_boxes": plan.view.n_boxes,
           "list2_entries": int(led["entries"]["V"]), "p_fmm": cfg.p_fmm, "p_qbx": cfg.p_qbx,
           "ms_per_apply": round(ms, 2), "points_per_s": (g.n_sources + g.n_targets) / (ms * 1e-3), "timing": timing,
           "stages_ms": {k: round(v, 3) for k, v in stage.items() if v > 0}, "setup_s": round(t_setup, 2)}
    print(json.dumps(out), flush=True)
    eng.close()


if __name__ == "__main__":
    for c in [int(a) for a in sys.argv[1:]] or [0, 1, 2, 3]:
        run(c)
