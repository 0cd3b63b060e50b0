"""Oracle restatement of the cell-local dynamic-AMR operators
(transfer.py:99-158) pinned against the
reference's own outputs (tests/golden/amr.npz, tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

from oracle import transfer as ot

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "amr.npz"))
CASES = range(int(G["amr_ncases"]))


@pytest.mark.parametrize("ci", CASES)
def test_oracle_amr_operators_match_reference(ci):
    dim, p, m, C = (int(v) for v in G[f"amr{ci}_meta"])
    Q = G[f"amr{ci}_q"]
    t = ot.transfer_for(p)
    rt, ct, ml, mnl = G["amr_decision"]
    for c in range(C):
        assert ot.gradient_indicator(Q[c], p) == G[f"amr{ci}_ind"][c]
        v = ot.refinement_verdict(Q[c], int(G[f"amr{ci}_levels"][c]), p, rt, ct, int(ml), int(mnl))
        assert v == G[f"amr{ci}_verdict"][c]
    digits = list(np.ndindex(*(3,) * dim))
    for i, dg in enumerate(digits):
        assert np.array_equal(ot.interp_volume(t, Q[0], dg), G[f"amr{ci}_interp"][i])
    ch = {dg: G[f"amr{ci}_children"][i] for i, dg in enumerate(digits)}
    assert np.array_equal(ot.restrict_volume(t, ch), G[f"amr{ci}_restrict"])


@pytest.mark.parametrize("ci", CASES)
def test_refine_coarsen_round_trip_reproduces_parent(ci):
    """restrict_volume(interpolate_volume(q)) == q up to rounding (the
    reference docstring's reproduction property, transfer.py:105-110)."""
    dim, p, m, C = (int(v) for v in G[f"amr{ci}_meta"])
    q = G[f"amr{ci}_q"][3]
    r = G[f"amr{ci}_roundtrip"]
    assert np.max(np.abs(r - q)) <= 1e-12 * max(1.0, np.max(np.abs(q)))
