"""The reference arm of bench.py: the reference package's own per-cell CPU
kernels timed on a bounded, Picard-stratified sample of the benchmarked
trajectory (oracle only: test / measurement infrastructure, never the
product path).

Where the reference comes from: the reference is a pure-Python package
(/root/reference/pkg/src/enclavedg, 6 files) that does not exist on the GPU
box.  `vendor_reference()` (called by __graft_entry__.build() in the build
container, where /root/reference exists) copies those files unmodified into
the git-ignored `oracle/_ref/enclavedg/`, which travels to the GPU box with
the repo snapshot, so the arm imports and times the reference's own
`kernels.py`.  Without it the arm falls back to the numpy restatement in
oracle/ops.py (bit-equal on the golden vectors) and says so
(`kind: "port"`).

What is timed per step (the reference's Algorithm-1 work for one cell,
PAPER.md:639-686): `admissible_dt` over the cell (kernels.py:267-281),
`stp_picard` (kernels.py:120-159), `riemann_rusanov` on its 2d sides
(kernels.py:162-173; the sample cell's own opposite trace stands in for the
neighbour's, which costs the same) and `corrector` (kernels.py:176-193).  The
inputs are real states of the benchmarked trajectory: for every step of
config 3, tests/golden/refarm_cfg3.npz holds the step's input state of up to
two cells per Picard count occurring in that step, plus the step's dt and
its full Picard-count histogram (written by tests/golden/make_full_parity.py
from the pinned oracle).  A timed step draws a sample whose Picard counts
are apportioned like that step's histogram (largest remainders), so the
sample's mean iteration count is the whole mesh's for that step.
"""
from __future__ import annotations

import os
import shutil
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
REF_SRC = "/root/reference/pkg/src/enclavedg"


def vendor_reference(src=REF_SRC, dst=REF_DIR):
    """Copy the reference package into oracle/_ref/enclavedg (git-ignored);
    returns the destination or None when the reference is absent."""
    if not os.path.isdir(src):
        return None
    out = os.path.join(dst, "enclavedg")
    os.makedirs(out, exist_ok=True)
    for f in os.listdir(src):
        if f.endswith(".py"):
            shutil.copyfile(os.path.join(src, f), os.path.join(out, f))
    return out


def load_reference():
    """(kernels, basis, pde) modules of the vendored reference, or None."""
    if not os.path.isfile(os.path.join(REF_DIR, "enclavedg", "kernels.py")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import enclavedg.basis as rb
    import enclavedg.kernels as rk
    import enclavedg.pde as rp
    return rk, rb, rp


def euler_descriptor(PdeDescriptor, dim, gamma=1.4):
    """The Euler system in the reference plugin format (pde.py:10-24); same
    formulas and operation order as oracle/ops.py `euler` and DESIGN.md."""
    gm1 = gamma - 1.0

    def parts(q):
        inv = 1.0 / q[0]
        ke = q[1] * q[1]
        for i in range(1, dim):
            ke = ke + q[1 + i] * q[1 + i]
        ke = 0.5 * ke * inv
        return inv, gm1 * (q[1 + dim] - ke)

    def flux(q, axis):
        inv, p = parts(q)
        u = q[1 + axis] * inv
        out = np.empty_like(q)
        out[0] = q[1 + axis]
        for i in range(dim):
            out[1 + i] = q[1 + i] * u
        out[1 + axis] = out[1 + axis] + p
        out[1 + dim] = (q[1 + dim] + p) * u
        return out

    def max_eig(q, axis):
        inv, p = parts(q)
        return np.abs(q[1 + axis] * inv) + np.sqrt(gamma * p * inv)

    return PdeDescriptor("euler", dim + 2, dim, flux, max_eig, is_linear=False)


class _Mesh:
    def __init__(self, dim, h):
        self.dim, self.h = dim, h

    def cell_edges(self, level):
        return (self.h,) * self.dim


_W = {}


def _init(dim, order, h, want_reference):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ref = load_reference() if want_reference else None
    if ref is not None:
        rk, rb, rp = ref
        _W.update(kind="reference", stp=rk.stp_picard, riemann=rk.riemann_rusanov, corr=rk.corrector,
                  dtf=lambda cells, pde, order, cfl: rk.admissible_dt(cells, pde, order, cfl, _Mesh(dim, h)),
                  pde=euler_descriptor(rp.PdeDescriptor, dim), basis=rb.get_basis(order))
    else:
        from . import ops
        _W.update(kind="port", stp=ops.predictor_picard, riemann=ops.rusanov, corr=ops.correct,
                  dtf=lambda cells, pde, order, cfl: ops.stable_dt(((h, q) for _, q in cells), pde, order, cfl, dim),
                  pde=ops.euler(dim), basis=ops.basis_for(order))
    _W.update(dim=dim, order=order, edges=(h,) * dim)


def _cells(args):
    """Algorithm-1 work of each (q, dt) item; returns (cells, iterations, seconds)."""
    items, cfl = args
    stp, rie, corr, dtf = _W["stp"], _W["riemann"], _W["corr"], _W["dtf"]
    pde, basis, edges, dim = _W["pde"], _W["basis"], _W["edges"], _W["dim"]
    its = 0
    t0 = time.perf_counter()
    for q, dt in items:
        dtf([((0, (0,) * dim), q)], pde, _W["order"], cfl)
        st = stp(q, pde, dt, basis, edges)
        res = {}
        for a in range(dim):
            for s in (0, 1):
                mine, theirs = st.trace_q[(a, s)], st.trace_q[(a, 1 - s)]
                lo, hi = (mine, theirs) if s == 1 else (theirs, mine)
                res[(a, s)] = rie(lo, hi, pde, a)
        corr(st, res, basis, edges)
        its += int(st.iterations)
    return len(items), its, time.perf_counter() - t0


def apportion(hist, total):
    """Largest-remainder apportionment of `total` draws to the histogram bins."""
    hist = np.asarray(hist, dtype=float)
    share = hist / hist.sum() * total
    n = np.floor(share).astype(int)
    rest = total - n.sum()
    if rest > 0:
        n[np.argsort(-(share - n), kind="stable")[:rest]] += 1
    return n


class RefArm:
    """Times the reference kernels on stratified samples of config 3's steps."""

    def __init__(self, fixture, dim=3, order=4, h=1.0 / 64, cfl=0.2, cores=None, want_reference=True):
        import multiprocessing as mp
        g = np.load(fixture)
        self.q, self.step, self.its = g["q"], g["step"], g["iterations"]
        self.dt, self.hist = g["dt"], g["hist"]
        self.nsteps = len(self.dt)
        self.cfl = cfl
        self.cores = cores or os.cpu_count() or 1
        self.pool = mp.get_context("fork").Pool(self.cores, initializer=_init,
                                                initargs=(dim, order, h, want_reference))
        self.kind = self.pool.apply(_kind)

    def close(self):
        self.pool.close()
        self.pool.join()

    def sample(self, k, total):
        """Items (q, dt) for trajectory step k (1-based) with Picard counts
        apportioned like the step's histogram."""
        kk = (k - 1) % self.nsteps
        sel = np.flatnonzero(self.step == kk + 1)
        bins = np.zeros_like(self.hist[kk])
        for v in self.its[sel]:
            bins[v] = self.hist[kk][v]
        counts = apportion(bins, total)
        items = []
        for v in np.flatnonzero(counts):
            cand = sel[self.its[sel] == v]
            for j in range(counts[v]):
                items.append((self.q[cand[j % cand.size]], float(self.dt[kk])))
        return items

    def mean_iterations(self, k):
        h = self.hist[(k - 1) % self.nsteps]
        return float((h * np.arange(h.size)).sum() / h.sum())

    def time_step(self, k, total):
        """Wall time of the sample of step k spread over all workers."""
        items = self.sample(k, total)
        # interleave so every worker gets the same Picard mix
        chunks = [(items[i::self.cores * 4], self.cfl) for i in range(self.cores * 4)]
        t0 = time.perf_counter()
        res = self.pool.map(_cells, [c for c in chunks if c[0]])
        wall = time.perf_counter() - t0
        return sum(r[0] for r in res), sum(r[1] for r in res), wall

    def per_cell_seconds(self, k=1, n=None):
        """One-worker probe: seconds per cell of step k's stratified mix."""
        items = self.sample(k, n or 2 * len(np.unique(self.its)))
        cells, _, sec = self.pool.apply(_cells, ((items, self.cfl),))
        return sec / cells


def _kind():
    return _W["kind"]
