"""Stage 1 timing at BASELINE config 1: host plan vs GPU plan (per-phase times on
stderr via QBXG_PLAN_TIMING)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06106_b200 import api  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = api.config_geometry(cid)
cfg = api.config_fmm(cid)
t = time.time()
h = api.Plan(cfg, g)
print(f"host: {time.time() - t:.3f} s (tree {h.view.build_seconds_tree:.3f}, lists {h.view.build_seconds_lists:.3f})",
      flush=True)
api.Plan(cfg, g, device="gpu")
os.environ["QBXG_PLAN_TIMING"] = "1"
t = time.time()
p = api.Plan(cfg, g, device="gpu")
print(f"gpu: {time.time() - t:.3f} s (tree {p.view.build_seconds_tree:.3f}, lists {p.view.build_seconds_lists:.3f}); "
      f"equal hashes {p.list_hashes() == h.list_hashes()}", flush=True)
