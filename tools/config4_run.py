"""BASELINE config 4 (4x4x4 array of level-5 urchins, Laplace SL+DL, p = 15, q = 5) on
one GPU: the strong-scaling base point (64 urchins, ~21M sources) and the weak-scaling
sizes (8 / 16 / 32 urchins).  Stage 1 on the GPU (qbxg_plan_create_gpu), then K
device-resident applies timed with CUDA events; prints one JSON line per size.

    python tools/config4_run.py [n_urchins ...]      (default: 8 64)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_06106_b200 import api  # noqa: E402


def run(n_urchins, reps=3):
    t0 = time.time()
    g = api.config_geometry(4, variant=n_urchins)
    t_geom = time.time() - t0
    cfg = api.config_fmm(4)
    t0 = time.time()
    plan = api.Plan(cfg, g, device="gpu")
    t_plan = time.time() - t0
    t0 = time.time()
    eng = api.FmmEngine(cfg, g, plan)
    t_create = time.time() - t0
    w = torch.from_numpy(g.weights()).cuda()
    mu = torch.from_numpy(np.ascontiguousarray(g.dipoles())).cuda()
    pot = torch.empty(g.n_targets, dtype=torch.float64, device="cuda")
    eng.apply_device(w.data_ptr(), mu.data_ptr(), pot.data_ptr())  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stage = {}
    e0.record()
    for _ in range(reps):
        eng.apply_device(w.data_ptr(), mu.data_ptr(), pot.data_ptr())
        for k, v in eng.last_timings()[0].items():
            stage[k] = stage.get(k, 0.0) + v / reps
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    led = plan.ledger()
    out = {"config": 4, "n_urchins": n_urchins, "n_sources": g.n_sources, "n_targets": g.n_targets,
           "n_boxes": plan.view.n_boxes, "list2_entries": int(led["entries"]["V"]),
           "ms_per_apply": round(ms, 2), "points_per_s": (g.n_sources + g.n_targets) / (ms * 1e-3),
           "stages_ms": {k: round(v, 2) for k, v in stage.items() if v > 0},
           "setup_s": {"geometry": round(t_geom, 2), "plan_gpu": round(t_plan, 2), "create": round(t_create, 2)},
           "checksum": float(pot.sum()), "finite": bool(torch.isfinite(pot).all())}
    print(json.dumps(out), flush=True)
    eng.close()
    del plan


if __name__ == "__main__":
    sizes = [int(a) for a in sys.argv[1:]] or [8, 64]
    for n in sizes:
        run(n)
