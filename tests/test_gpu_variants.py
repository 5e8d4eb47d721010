"""Helmholtz work-split switches (not what is computed) stay parity-green against the
oracle.  Each runs in its own process because the switches are read at
engine creation."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

HELM_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %r)
import oracle as O
from paper_1805_06106_b200 import api
g = api.config_geometry(3, level=1)
rng = np.random.default_rng(3)
w = g.quad_weight * (rng.uniform(-1, 1, g.n_sources) + 1j * rng.uniform(-1, 1, g.n_sources))
cfg = api.FmmConfig(p_fmm=8, p_qbx=4, n_max=64, kernel=2, helmholtz_k=3.0)
plan = api.Plan(cfg, g)
eng = api.FmmEngine(cfg, g, plan)
pot = eng.apply_complex(w)
eng.close()
ref = O.helm_execute(plan, g, 3.0, 8, 4, w)
print(json.dumps({"helm": float(np.linalg.norm(pot - ref) / np.linalg.norm(ref))}))
""" % ROOT


@pytest.mark.parametrize("mode", ["full", "split", "p2l-cta", "shift-box"])
def test_helmholtz_m2l_variant(mode):
    """QBXG_HELM_M2L=full (dense per-offset operators) and =split (even / odd dense
    blocks) against the oracle; the default point-and-shoot M2L is covered by
    tests/test_helmholtz.py."""
    full = dict(os.environ)
    if mode == "p2l-cta":
        full["QBXG_HELM_P2L"] = "cta"  # one CTA-wide wave table per source in P2L
    elif mode == "shift-box":
        full["QBXG_HELM_SHIFT"] = "box"  # M2M / L2L one box per CTA
    else:
        full["QBXG_HELM_M2L"] = mode
    r = subprocess.run([sys.executable, "-c", HELM_SCRIPT], env=full, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert json.loads(r.stdout.strip().splitlines()[-1])["helm"] <= 1e-11
