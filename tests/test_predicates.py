"""The adequate-separation relation on its own:
the product's predicate (qbxg_adequately_separated, the one csrc/host/plan.cpp builds
lists with) and the oracle's independent restatement (oracle/lists_brute.cpp) against
SPEC's worked examples, against each other, and for the monotonicity the list
construction relies on ("Parent(a) < b implies a < b", §5.2.2)."""
import numpy as np
import pytest

import oracle as O
from paper_1805_06106_b200 import api

KINDS = ("box_vs_tcr", "tcr_vs_box")


def both(kind, ca, ha, cb, hb, tf):
    a = api.adequately_separated(kind, ca, ha, cb, hb, tf)
    b = O.adequately_separated(KINDS.index(kind), ca, ha, cb, hb, tf)
    assert a == b, (kind, ca, ha, cb, hb, tf)
    return a


@pytest.mark.parametrize("kind", KINDS)
def test_spec_examples(kind):
    # a = b -> false for both kinds  [SPEC.md:375]
    for h in (1.0, 0.25, 3.0):
        assert not both(kind, [0.3, -0.2, 0.1], h, [0.3, -0.2, 0.1], h, 0.9)
    # unit boxes, t_f = 0.9, centres 20 apart on an axis -> true  [SPEC.md:377]
    for axis in range(3):
        c = np.zeros(3)
        c[axis] = 20.0
        assert both(kind, np.zeros(3), 1.0, c, 1.0, 0.9)
        assert both(kind, c, 1.0, np.zeros(3), 1.0, 0.9)


def test_spec_example_arithmetic_edges():
    # box_vs_tcr: d - sqrt(3)|b|(1+t_f) >= 3|a|; tcr_vs_box: d_inf - |b| >= 3|a|(1+t_f)
    tf = 0.9
    d_tcr = 3.0 + np.sqrt(3.0) * 1.9
    assert both("box_vs_tcr", [0, 0, 0], 1.0, [d_tcr + 1e-9, 0, 0], 1.0, tf)
    assert not both("box_vs_tcr", [0, 0, 0], 1.0, [d_tcr - 1e-9, 0, 0], 1.0, tf)
    assert both("tcr_vs_box", [0, 0, 0], 1.0, [6.7 + 1e-9, 0.5, -0.5], 1.0, tf)
    assert not both("tcr_vs_box", [0, 0, 0], 1.0, [6.7 - 1e-9, 0.5, -0.5], 1.0, tf)
    # l2 vs l-inf: a diagonal offset separated in l-inf is not necessarily separated in l2
    assert both("tcr_vs_box", [0, 0, 0], 1.0, [6.8, 6.8, 6.8], 1.0, tf)


def test_product_equals_oracle_random():
    rng = np.random.default_rng(3)
    for _ in range(4000):
        ha = 2.0 ** rng.integers(-4, 2)
        hb = ha * 2.0 ** rng.integers(-1, 2)
        ca = rng.integers(-8, 8, 3) * 2 * ha + ha
        cb = rng.integers(-8, 8, 3) * 2 * hb + hb
        tf = float(rng.choice([0.0, 0.5, 0.9]))
        for kind in KINDS:
            both(kind, ca, ha, cb, hb, tf)


def _tree(seed):
    g = api.config_geometry(2, level=1, n_volume_targets=200, seed=seed)
    return api.Plan(api.FmmConfig(p_fmm=6, p_qbx=3, n_max=16), g).arrays()


@pytest.mark.parametrize("seed", [0, 1])
def test_monotone_in_parent_and_oracle_agrees_on_tree(seed):
    A = _tree(seed)
    c, h, par = A["box_center"], A["box_radius"], A["box_parent"]
    nb = A["n_boxes"]
    rng = np.random.default_rng(seed)
    pairs = rng.integers(0, nb, (3000, 2))
    checked = 0
    for a, b in pairs:
        for kind in KINDS:
            sep = both(kind, c[a], h[a], c[b], h[b], 0.9)
            pa = par[a]
            if pa >= 0 and both(kind, c[pa], h[pa], c[b], h[b], 0.9):
                assert sep, f"monotonicity violated: {kind} parent({a}) < {b} but not {a} < {b}"
                checked += 1
    assert checked > 100
