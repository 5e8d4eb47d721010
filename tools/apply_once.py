"""One device-resident apply of a BASELINE config (default 1) -- the command the
ncu captures in profiles/ were taken on.

    python tools/apply_once.py [config] [n_applies]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_06106_b200 import api  # noqa: E402


def main():
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    g = api.config_geometry(cfg_id)
    cfg = api.config_fmm(cfg_id)
    eng = api.FmmEngine(cfg, g)
    w = torch.from_numpy(g.weights()).cuda()
    mu = torch.from_numpy(np.ascontiguousarray(g.dipoles())).cuda() if cfg.kernel == 1 else None
    pot = torch.empty(g.n_targets, dtype=torch.float64, device="cuda")
    for _ in range(reps):
        eng.apply_device(w.data_ptr(), mu.data_ptr() if mu is not None else None, pot.data_ptr())
    torch.cuda.synchronize()
    print("applied", reps, "x config", cfg_id, "targets", g.n_targets, "checksum", float(pot.sum()))
    eng.close()


if __name__ == "__main__":
    main()
