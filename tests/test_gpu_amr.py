"""GPU parity of the cell-local dynamic-AMR operators (SURVEY.md section 8(f)
f2; transfer.py:99-158) through the C ABI against the reference's own
outputs (tests/golden/amr.npz) and the oracle."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "amr.npz"))
CASES = range(int(G["amr_ncases"]))
TOL = 1e-13   # fp64 contraction order differs from numpy's tensordot (BLAS)


@pytest.fixture(scope="module")
def tr():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1806_07984_b200 import _lib, transfer
    _lib.load()
    return transfer


def _rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(1e-300, np.max(np.abs(b))))


@pytest.mark.parametrize("ci", CASES)
def test_indicator_and_verdicts_vs_reference(tr, ci):
    dim, p, m, C = (int(v) for v in G[f"amr{ci}_meta"])
    Q = G[f"amr{ci}_q"]
    rt, ct, ml, mnl = G["amr_decision"]
    dec = tr.RefinementDecision(refine_tol=rt, coarsen_tol=ct, max_level=int(ml))
    ind, ver = tr.gradient_indicator_batch(Q, p, G[f"amr{ci}_levels"], dec, int(mnl))
    ind = ind.cpu().numpy()
    ref = G[f"amr{ci}_ind"]
    assert np.all(np.abs(ind - ref) <= TOL * np.maximum(1.0, np.abs(ref)))
    assert np.array_equal(ver.cpu().numpy(), G[f"amr{ci}_verdict"])
    # single-cell API (reference signatures)
    assert abs(tr.gradient_indicator(Q[0], p) - ref[0]) <= TOL * max(1.0, abs(ref[0]))
    code = {1: tr.RefinementDecision.REFINE, 0: tr.RefinementDecision.KEEP, -1: tr.RefinementDecision.COARSEN}
    for c in range(C):
        v = tr.evaluate_refinement_criterion(Q[c], int(G[f"amr{ci}_levels"][c]), p, dec, int(mnl))
        assert v == code[int(G[f"amr{ci}_verdict"][c])]


@pytest.mark.parametrize("ci", CASES)
def test_interpolate_and_restrict_volume_vs_reference(tr, ci):
    dim, p, m, C = (int(v) for v in G[f"amr{ci}_meta"])
    ops = tr.get_transfer(p)
    digits = list(np.ndindex(*(3,) * dim))
    Q = G[f"amr{ci}_q"]
    # batched: all 3^d children of parent 0
    out = tr.interpolate_volume_batch(p, Q, digits, parent=[0] * len(digits)).cpu().numpy()
    assert _rel(out, G[f"amr{ci}_interp"]) <= TOL
    # single child through the reference signature
    assert _rel(tr.interpolate_volume(ops, Q[0], digits[-1]), G[f"amr{ci}_interp"][-1]) <= TOL
    ch = G[f"amr{ci}_children"]
    r = tr.restrict_volume_batch(p, ch[None]).cpu().numpy()[0]
    assert _rel(r, G[f"amr{ci}_restrict"]) <= TOL
    children = {dg: ch[i] for i, dg in enumerate(digits)}
    assert _rel(tr.restrict_volume(ops, children), G[f"amr{ci}_restrict"]) <= TOL
    # another dict order sums in that order (same value to rounding)
    rev = dict(reversed(list(children.items())))
    assert _rel(tr.restrict_volume(ops, rev), G[f"amr{ci}_restrict"]) <= 1e-12


@pytest.mark.parametrize("ci", CASES)
def test_refine_coarsen_round_trip_on_device(tr, ci):
    dim, p, m, C = (int(v) for v in G[f"amr{ci}_meta"])
    Q = G[f"amr{ci}_q"]
    digits = list(np.ndindex(*(3,) * dim))
    kids = tr.interpolate_volume_batch(p, Q, digits * C, parent=np.repeat(np.arange(C), len(digits)))
    back = tr.restrict_volume_batch(p, kids.reshape((C, len(digits)) + Q.shape[1:])).cpu().numpy()
    assert np.max(np.abs(back - Q)) <= 1e-12 * max(1.0, np.max(np.abs(Q)))


def test_indicator_nan_axis_dropped_and_errors(tr):
    import torch
    from paper_1806_07984_b200.errors import ConfigError
    from oracle import transfer as ot
    rng = np.random.default_rng(5)
    q = rng.standard_normal((4, 5, 5))
    q[0, 2, 3] = np.nan      # NaN in every axis through node (2, 3)
    ref = ot.gradient_indicator(q, 4)
    got = tr.gradient_indicator(q, 4)
    assert (np.isnan(ref) and np.isnan(got)) or got == ref
    with pytest.raises(ValueError):
        tr.RefinementDecision(refine_tol=0.1, coarsen_tol=0.2, max_level=3)
    with pytest.raises(ConfigError):
        tr.gradient_indicator_batch(torch.zeros((1, 1, 10, 10), dtype=torch.float64, device="cuda"), 9)
    empty = tr.gradient_indicator_batch(torch.zeros((0, 4, 4, 4), dtype=torch.float64, device="cuda"), 3)
    assert empty.numel() == 0
