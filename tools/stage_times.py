"""Per-stage CUDA-event times of a device-resident apply (near field on the main
stream unless QBXG_OVERLAP is set).

    python tools/stage_times.py [config] [n_applies]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_06106_b200 import api  # noqa: E402


def main():
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    g = api.config_geometry(cfg_id)
    cfg = api.config_fmm(cfg_id)
    eng = api.FmmEngine(cfg, g)
    eng.set_overlap(os.environ.get("QBXG_OVERLAP", "0") != "0")
    w = torch.from_numpy(g.weights()).cuda()
    mu = torch.from_numpy(np.ascontiguousarray(g.dipoles())).cuda() if cfg.kernel == 1 else None
    pot = torch.empty(g.n_targets, dtype=torch.float64, device="cuda")
    acc = {}
    for i in range(reps + 1):
        eng.apply_device(w.data_ptr(), mu.data_ptr() if mu is not None else None, pot.data_ptr())
        torch.cuda.synchronize()
        if i == 0:
            continue
        for k, v in eng.last_timings()[0].items():
            acc[k] = acc.get(k, 0.0) + v / reps
    env = {k: v for k, v in os.environ.items() if k.startswith("QBXG_")}
    print(json.dumps({"config": cfg_id, "env": env, "checksum": float(pot.sum()),
                      "ms": {k: round(v, 3) for k, v in acc.items() if v > 0}}))
    eng.close()


if __name__ == "__main__":
    main()
