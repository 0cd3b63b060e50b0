"""Generate the golden fixtures from the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/ops.npz (per-kernel known-answer vectors),
tests/golden/traj.npz (short Algorithm-1 trajectories of proxy configs),
tests/golden/mesh_cfg5_proxy.json (face forest of a refined mesh) and
tests/golden/amr.npz (volumetric transfer and refinement criterion, f2).  Every
number in them comes out of /root/reference/pkg/src/enclavedg; the only
additions are the Euler PdeDescriptor (the reference has none -- it is built
here in the reference's own plugin format, pde.py:10-24, from the formulas in
DESIGN.md) and the Algorithm-1 loop (the reference ships no driver), written
below against the reference kernels and the reference Mesh.
"""
from __future__ import annotations

import json
import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import enclavedg.basis as rb          # noqa: E402
import enclavedg.kernels as rk        # noqa: E402
import enclavedg.mesh as rm           # noqa: E402
import enclavedg.pde as rp            # noqa: E402
import enclavedg.transfer as rt       # noqa: E402

from paper_1806_07984_b200 import configs as cf   # noqa: E402  (input generator only)


def euler_descriptor(dim, gamma=1.4):
    """Euler system in the reference plugin format; same formulas / operation
    order as DESIGN.md 'Euler plugin' (and oracle/ops.py euler)."""
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

    def lam(q, axis):
        inv, p = parts(q)
        u = q[1 + axis] * inv
        with np.errstate(invalid="ignore"):
            c = np.sqrt(gamma * p * inv)
        return np.abs(u) + c

    return rp.PdeDescriptor("euler", dim + 2, dim, flux, lam, is_linear=False)


def ref_pde(name, dim):
    if name == "euler":
        return euler_descriptor(dim)
    if name == "advection":
        return rp.advection(velocity=(1.0, 0.5, 0.25)[:dim], dim=dim)
    return rp.burgers(dim=dim)


def smooth_states(rng, name, dim, n, C, amp=0.05):
    shape = (C,) + (n,) * dim
    if name == "euler":
        q = np.empty((C, dim + 2) + (n,) * dim)
        rho = 1.0 + amp * rng.random(shape)
        q[:, 0] = rho
        for i in range(dim):
            q[:, 1 + i] = rho * (0.3 + 0.2 * i + amp * rng.random(shape))
        q[:, 1 + dim] = 2.5 + amp * rng.random(shape) + 0.5 * sum(q[:, 1 + i] ** 2 for i in range(dim)) / rho
        return q
    return (1.0 + amp * rng.standard_normal(shape))[:, None]


TRACE_KEYS = lambda dim: [(a, s) for a in range(dim) for s in (0, 1)]  # noqa: E731


def gen_ops():
    out = {}
    for p in range(1, 8):
        b = rb.get_basis(p)
        kinv, lift = rk._time_operators(b)
        t = rt.get_transfer(p)
        out[f"basis{p}_nodes"] = b.nodes
        out[f"basis{p}_weights"] = b.weights
        out[f"basis{p}_D"] = b.diff_matrix
        out[f"basis{p}_tl"] = b.trace_left
        out[f"basis{p}_tr"] = b.trace_right
        out[f"basis{p}_kinv"] = kinv
        out[f"basis{p}_lift"] = lift
        out[f"basis{p}_interp"] = np.stack(t.interp)
        out[f"basis{p}_restrict"] = np.stack(t.restrict)
    rng = np.random.default_rng(20260101)
    stp_cases = [("advection", 2, 3, 0.9 / (27 * 7), 1 / 27),
                 ("euler", 2, 5, 0.2 / (243 * 11 * 2.2), 1 / 243),
                 ("euler", 3, 4, 0.2 / (64 * 9 * 1.5), 1 / 64),
                 ("euler", 2, 3, 0.2 / (243 * 7 * 2.2), 1 / 243),
                 ("burgers", 2, 2, 0.001, 1 / 27),
                 ("advection", 3, 2, 0.9 / (9 * 5), 1 / 9),
                 ("euler", 2, 1, 0.3 / (27 * 3 * 2), 1 / 27),
                 ("euler", 3, 2, 0.3 / (27 * 5 * 2), 1 / 27)]
    out["stp_ncases"] = np.array(len(stp_cases))
    for ci, (name, dim, p, dt, h) in enumerate(stp_cases):
        C = 6
        b = rb.get_basis(p)
        pde = ref_pde(name, dim)
        Q = smooth_states(rng, name, dim, p + 1, C)
        # exercise non-square cells in one case
        edges = (h,) * dim if ci != 5 else (h, 0.5 * h, 2.0 * h)
        res = [rk.stp_picard(Q[c], pde, dt, b, edges) for c in range(C)]
        pre = f"stp{ci}_"
        out[pre + "meta"] = np.array([dim, p, {"advection": 0, "burgers": 1, "euler": 2}[name]])
        out[pre + "q"] = Q
        out[pre + "dt"] = np.array(dt)
        out[pre + "edges"] = np.array(edges)
        out[pre + "q_int"] = np.stack([r.q_int for r in res])
        out[pre + "q_end"] = np.stack([r.q_end for r in res])
        out[pre + "trace_q"] = np.stack([np.stack([r.trace_q[k] for k in TRACE_KEYS(dim)]) for r in res])
        out[pre + "trace_f"] = np.stack([np.stack([r.trace_f[k] for k in TRACE_KEYS(dim)]) for r in res])
        out[pre + "iterations"] = np.array([r.iterations for r in res])
        out[pre + "converged"] = np.array([r.converged for r in res])
        # corrector with synthetic outcomes for these stores
        outc = rng.standard_normal((C, 2 * dim) + res[0].trace_f[(0, 0)].shape) * 1e-3
        corr = [rk.corrector(res[c], {k: outc[c, j] for j, k in enumerate(TRACE_KEYS(dim))}, b, edges)
                for c in range(C)]
        out[pre + "outcomes"] = outc
        out[pre + "corrected"] = np.stack(corr)
        # linear cross-check (Picard with tol -> 0 vs Cauchy-Kowalevski)
        if pde.is_linear:
            lin = [rk.stp_linear(Q[c], pde, dt, b, edges) for c in range(C)]
            out[pre + "ck_q_end"] = np.stack([r.q_end for r in lin])
            out[pre + "ck_q_int"] = np.stack([r.q_int for r in lin])
    # Riemann known answers on traces
    riem = []
    for ci, (name, dim) in enumerate([("advection", 2), ("euler", 2), ("euler", 3), ("burgers", 2)]):
        pde = ref_pde(name, dim)
        lo = smooth_states(rng, name, dim, 5, 7, amp=0.3)[..., 0]
        hi = smooth_states(rng, name, dim, 5, 7, amp=0.3)[..., 0]
        lo = lo.reshape(7, pde.m, -1)
        hi = hi.reshape(7, pde.m, -1)
        for axis in range(dim):
            o = np.stack([rk.riemann_rusanov(lo[c], hi[c], pde, axis) for c in range(7)])
            on = np.stack([rk.riemann_rusanov(lo[c], hi[c], pde, axis, sign=-1) for c in range(7)])
            key = f"riem{ci}_{axis}_"
            out[key + "lo"] = lo
            out[key + "hi"] = hi
            out[key + "out"] = o
            out[key + "neg"] = on
            riem.append((ci, name, dim, axis))
    out["riem_index"] = np.array([[ci, {"advection": 0, "burgers": 1, "euler": 2}[nm], d, a]
                                  for ci, nm, d, a in riem])
    # FV patch updates
    for ci, (name, dim, k) in enumerate([("euler", 3, 8), ("euler", 2, 5), ("advection", 2, 5)]):
        pde = ref_pde(name, dim)
        P = smooth_states(rng, name, dim, k, 3, amp=0.2)
        halos = [{(a, s): smooth_states(rng, name, dim, k, 1, amp=0.2)[0][(slice(None),) + tuple(
            0 if t == a else slice(None) for t in range(dim))] for a in range(dim) for s in (0, 1)}
            for _ in range(3)]
        edges = (1.0 / 16,) * dim
        dt = 0.4 * (edges[0] / k) / 3.0
        o = np.stack([rk.fv_patch_update(P[c], pde, dt, edges, halos[c]) for c in range(3)])
        key = f"fv{ci}_"
        out[key + "meta"] = np.array([dim, k, {"advection": 0, "burgers": 1, "euler": 2}[name]])
        out[key + "patch"] = P
        out[key + "halos"] = np.stack([np.stack([halos[c][kk] for kk in TRACE_KEYS(dim)]) for c in range(3)])
        out[key + "dt"] = np.array(dt)
        out[key + "out"] = o
        out[key + "layers"] = np.stack([np.stack([rk.patch_boundary_layers(P[c])[kk] for kk in TRACE_KEYS(dim)])
                                        for c in range(3)])
    # SPEC known answers
    adv1 = rp.advection(velocity=(1.0, 0.5))
    out["kat_rusanov_adv_equal"] = rk.riemann_rusanov(np.full((1, 4), 2.0), np.full((1, 4), 2.0), adv1, 0)
    out["kat_rusanov_adv_upwind"] = rk.riemann_rusanov(np.full((1, 4), 1.0), np.full((1, 4), 0.0), adv1, 0)
    out["kat_rusanov_burgers"] = rk.riemann_rusanov(np.full((1, 4), 2.0), np.full((1, 4), 0.0), rp.burgers(), 0)
    mesh9 = rm.build_uniform(2, dim=2, periodic=True)
    cells = [(k, np.ones((1, 4, 4))) for k in mesh9.real_cells]
    out["kat_dt_adv_h9"] = np.array(rk.admissible_dt(cells, rp.advection(velocity=(1.0, 0.0)), 3, 0.9, mesh9))
    # admissible_dt on Euler states incl. a NaN cell and a zero-speed cell
    pde = euler_descriptor(2)
    Q = smooth_states(rng, "euler", 2, 4, 12)
    Q[3, 0, 1, 1] = np.nan
    Q[5, 1:3] = 0.0
    Q[5, 3] = 0.0   # p = 0, u = 0 -> lambda = 0 (skipped)
    keys = list(mesh9.real_cells)[:12]
    out["dt_euler_q"] = Q
    out["dt_euler_val"] = np.array(rk.admissible_dt(list(zip(keys, Q)), pde, 3, 0.9, mesh9))
    # transfer functions
    for p in (2, 3, 4):
        t = rt.get_transfer(p)
        tr2 = rng.standard_normal((4, p + 1))
        tr3 = rng.standard_normal((5, p + 1, p + 1))
        for j in range(3):
            out[f"xfer{p}_i2_{j}"] = rt.interpolate_face_trace(t, tr2, (j,))
            out[f"xfer{p}_r2_{j}"] = rt.restrict_face_values(t, tr2, (j,))
        for j in range(3):
            for l in range(3):
                out[f"xfer{p}_i3_{j}{l}"] = rt.interpolate_face_trace(t, tr3, (j, l))
                out[f"xfer{p}_r3_{j}{l}"] = rt.restrict_face_values(t, tr3, (j, l))
        buf = types.SimpleNamespace(write_guard=__import__("threading").Lock(), accum_sweep=None,
                                    outcome=None, restricted_children=set())
        for j in range(3):
            rt.restrict_riemann(t, buf, tr2 * (j + 1), (j,), sweep=7)
        out[f"xfer{p}_acc2"] = buf.outcome
        out[f"xfer{p}_tr2"] = tr2
        out[f"xfer{p}_tr3"] = tr3
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **out)
    print("ops.npz:", len(out), "arrays")


# ------------------------------------------------------ reference drivers ---

def ref_step_mesh(mesh, Q, pde, p, cfl, sweep):
    """Algorithm 1 over a reference Mesh (uniform or adaptive), per cell."""
    b = rb.get_basis(p)
    t = rt.get_transfer(p)
    dim = mesh.dim
    keys = [n.key for n in mesh.sfc_cells]
    dt = rk.admissible_dt([(k, Q[k]) for k in keys], pde, p, cfl, mesh)
    st = {k: rk.stp_picard(Q[k], pde, dt, b, mesh.cell_edges(k[0])) for k in keys}
    outcome = {}
    bufs = {}
    for f in mesh.faces.values():
        if not f.is_leaf:
            continue
        a = f.axis
        tr = [None, None]
        for s in (0, 1):
            tag, node = f.sides[s]
            if tag == "cell":
                tr[s] = st[node.key].trace_q[(a, 1 - s)]
            elif tag == "virtual":
                tr[s] = rt.interpolate_to_virtual(t, st[f.owners[s].key].trace_q[(a, 1 - s)], f.child_pos)
        if f.sides[0][0] == "boundary":
            tr[0] = tr[1]
        if f.sides[1][0] == "boundary":
            tr[1] = tr[0]
        o = rk.riemann_rusanov(tr[0], tr[1], pde, a)
        if f.parent is not None:
            buf = bufs.setdefault(f.parent.key, types.SimpleNamespace(
                write_guard=__import__("threading").Lock(), accum_sweep=None, outcome=None,
                restricted_children=set()))
            rt.restrict_riemann(t, buf, o, f.child_pos, sweep)
        outcome[f.key] = o
    for k, buf in bufs.items():
        outcome[k] = buf.outcome
    Qn = {}
    for n in mesh.sfc_cells:
        res = {(a, s): outcome[mesh.side_face_key(n, a, s)] for a in range(dim) for s in (0, 1)}
        Qn[n.key] = rk.corrector(st[n.key], res, b, mesh.cell_edges(n.level))
    return Qn, dt, np.array([st[k].iterations for k in keys])


def ref_step_cartesian(Q, N, dim, periodic, pde, p, cfl, h=None):
    """Algorithm 1 on a non-3^k Cartesian grid (row-major cells), per cell."""
    b = rb.get_basis(p)
    h = 1.0 / N if h is None else h
    edges = (h,) * dim
    C = Q.shape[0]
    fake = types.SimpleNamespace(dim=dim, cell_edges=lambda level: edges)
    dt = rk.admissible_dt([((0, c), Q[c]) for c in range(C)], pde, p, cfl, fake)
    st = [rk.stp_picard(Q[c], pde, dt, b, edges) for c in range(C)]
    strides = [N ** (dim - 1 - t) for t in range(dim)]
    up = {}
    for c in range(C):
        idx = [(c // strides[t]) % N for t in range(dim)]
        for a in range(dim):
            j = idx[a] + 1
            lo = st[c].trace_q[(a, 1)]
            if j < N or periodic:
                hi = st[c + ((j % N) - idx[a]) * strides[a]].trace_q[(a, 0)]
            else:
                hi = lo
            up[(c, a)] = rk.riemann_rusanov(lo, hi, pde, a)
    Qn = np.empty_like(Q)
    for c in range(C):
        idx = [(c // strides[t]) % N for t in range(dim)]
        res = {}
        for a in range(dim):
            res[(a, 1)] = up[(c, a)]
            j = idx[a] - 1
            if j >= 0 or periodic:
                res[(a, 0)] = up[(c + ((j % N) - idx[a]) * strides[a], a)]
            else:
                own = st[c].trace_q[(a, 0)]
                res[(a, 0)] = rk.riemann_rusanov(own, own, pde, a)
        Qn[c] = rk.corrector(st[c], res, b, edges)
    return Qn, dt, np.array([s.iterations for s in st])


def ref_fv_step(P, npx, k, pde, cfl, h):
    dim = 3
    B = P.shape[0]
    fake = types.SimpleNamespace(dim=dim, cell_edges=lambda level: (h,) * dim)
    dt = rk.admissible_dt([((0, c), P[c]) for c in range(B)], pde, 0, cfl, fake)
    layers = [rk.patch_boundary_layers(P[c]) for c in range(B)]
    out = np.empty_like(P)
    for c in range(B):
        idx = [c // (npx * npx), (c // npx) % npx, c % npx]
        strides = [npx * npx, npx, 1]
        halos = {}
        for a in range(dim):
            for s in (0, 1):
                j = idx[a] + (1 if s else -1)
                if 0 <= j < npx:
                    halos[(a, s)] = layers[c + (j - idx[a]) * strides[a]][(a, 1 - s)]
                else:
                    halos[(a, s)] = layers[c][(a, s)]
        out[c] = rk.fv_patch_update(P[c], pde, dt, (h * k,) * dim, halos)
    return out, dt


def gen_traj():
    out = {}
    # cfg1 in full on the reference's own 3-partitioned mesh
    cfg = cf.CONFIGS["cfg1"]
    Q0 = cf.initial_dg_uniform(cfg)
    mesh = rm.build_uniform(3, dim=2, periodic=True)
    N = cfg.cells
    Q = {(3, (c // N, c % N)): Q0[c] for c in range(N * N)}
    pde = rp.advection(velocity=cfg.velocity)
    dts, its = [], []
    for k in range(cfg.steps):
        Q, dt, it = ref_step_mesh(mesh, Q, pde, cfg.order, cfg.cfl, k)
        dts.append(dt)
    out["cfg1_q0"] = Q0
    out["cfg1_q"] = np.stack([Q[(3, (c // N, c % N))] for c in range(N * N)])
    out["cfg1_dt"] = np.array(dts)
    print("cfg1 done")
    # DG proxies on Cartesian grids: (name, base cfg, overrides, steps)
    # cfg3w: a 6^3 window of the real 64^3 blast grid across the interface
    # (h = 1/64, outflow at the window faces)
    proxies = [("cfg2p", "cfg2", dict(cells=9), 3, None),
               ("cfg2s", "cfg2", dict(cells=9, cfl=0.2), 5, None),
               ("cfg3w", "cfg3", dict(), 3, (14, 6))]
    for tag, base, kw, steps, window in proxies:
        cfg = cf.CONFIGS[base].with_(**kw)
        Q0 = cf.initial_dg_uniform(cfg, window=window)
        pde = ref_pde(cfg.pde, cfg.dim)
        Q = Q0.copy()
        N = cfg.cells if window is None else window[1]
        dts, its = [], []
        for _ in range(steps):
            Q, dt, it = ref_step_cartesian(Q, N, cfg.dim, cfg.periodic and window is None, pde,
                                           cfg.order, cfg.cfl, h=1.0 / cfg.cells)
            dts.append(dt)
            its.append(it)
        out[tag + "_q0"] = Q0
        out[tag + "_q"] = Q
        out[tag + "_dt"] = np.array(dts)
        out[tag + "_its"] = np.stack(its)
        out[tag + "_meta"] = np.array([N, cfg.dim, cfg.order, int(cfg.periodic and window is None), steps,
                                       cfg.cells, -1 if window is None else window[0]])
        out[tag + "_cfl"] = np.array(cfg.cfl)
        print(tag, "done")
    # FV proxy: 16^3 cells as 2^3 patches of 8^3
    cfg = cf.CONFIGS["cfg4"].with_(cells=16)
    P0 = cf.initial_fv(cfg)
    pde = euler_descriptor(3)
    P = P0.copy()
    dts = []
    for _ in range(5):
        P, dt = ref_fv_step(P, 2, 8, pde, cfg.cfl, 1.0 / 16)
        dts.append(dt)
    out["cfg4p_q0"] = P0
    out["cfg4p_q"] = P
    out["cfg4p_dt"] = np.array(dts)
    print("cfg4p done")
    # AMR proxy: base 9x9 (level 2) + refined disc, p = 3, periodic
    cfg = cf.CONFIGS["cfg5"].with_(cells=9)
    cells = cf.amr_cells(cfg)
    mesh = rm.build_uniform(2, dim=2, periodic=True)
    refine = [mesh.real_cells[c_ix] for c_ix in {(2, tuple(i // 3 for i in ix)) for l, ix in cells if l == 3}]
    mesh.refine_many(refine)
    order = [n.key for n in mesh.sfc_cells]
    assert order == cf.sfc_sort(cells, 2)
    Q0 = cf.initial_dg_amr(cfg, order)
    Q = {k: Q0[i] for i, k in enumerate(order)}
    pde = euler_descriptor(2)
    dts, its = [], []
    for k in range(3):
        Q, dt, it = ref_step_mesh(mesh, Q, pde, cfg.order, cfg.cfl, k)
        dts.append(dt)
        its.append(it)
    out["cfg5p_q0"] = Q0
    out["cfg5p_q"] = np.stack([Q[k] for k in order])
    out["cfg5p_dt"] = np.array(dts)
    out["cfg5p_its"] = np.stack(its)
    out["cfg5p_levels"] = np.array([k[0] for k in order])
    out["cfg5p_index"] = np.array([k[1] for k in order])
    np.savez_compressed(os.path.join(HERE, "traj.npz"), **out)
    # the face forest of the proxy mesh, for the topology pins
    faces = []
    for f in mesh.faces.values():
        faces.append(dict(key=[f.axis, f.level, list(f.pos)],
                          sides=[s[0] for s in f.sides],
                          owners=[None if o is None else [o.level, list(o.index)] for o in f.owners],
                          children=len(f.children or ()),
                          child_pos=None if f.child_pos is None else list(f.child_pos),
                          parent=None if f.parent is None else [f.parent.axis, f.parent.level, list(f.parent.pos)]))
    skel = [[n.level, list(n.index)] for n in mesh.sfc_cells
            if rm.classify_cell(mesh, n) is rm.CellClass.SKELETON]
    with open(os.path.join(HERE, "mesh_cfg5_proxy.json"), "w") as fh:
        json.dump({"faces": faces, "skeleton": skel,
                   "sfc": [[l, list(ix)] for l, ix in order]}, fh)
    print("traj.npz + mesh json done")


def gen_amr():
    """SURVEY.md section 8(f) f2, the cell-local part of dynamic AMR:
    transfer.py:99-158 (interpolate_volume, restrict_volume,
    gradient_indicator, evaluate_refinement_criterion) on seeded cells."""
    out = {}
    rng = np.random.default_rng(20261020)
    cases = [(2, 3, 4), (2, 5, 4), (3, 4, 5), (2, 1, 1), (3, 2, 5), (2, 7, 4), (3, 5, 1)]
    out["amr_ncases"] = np.array(len(cases))
    dec = rt.RefinementDecision(refine_tol=0.5, coarsen_tol=0.05, max_level=3)
    for ci, (dim, p, m) in enumerate(cases):
        n = p + 1
        t = rt.get_transfer(p)
        C = 5
        Q = rng.standard_normal((C, m) + (n,) * dim)
        Q[1] *= 1e-3                      # a smooth, low-indicator cell
        Q[2] = Q[2, :, :1].repeat(n, axis=1) if dim == 2 else Q[2]
        pre = f"amr{ci}_"
        out[pre + "meta"] = np.array([dim, p, m, C])
        out[pre + "q"] = Q
        out[pre + "ind"] = np.array([rt.gradient_indicator(Q[c], p) for c in range(C)])
        levels = np.array([0, 1, 2, 3, 1], dtype=np.int32)
        out[pre + "levels"] = levels
        code = {rt.RefinementDecision.REFINE: 1, rt.RefinementDecision.KEEP: 0, rt.RefinementDecision.COARSEN: -1}
        out[pre + "verdict"] = np.array([code[rt.evaluate_refinement_criterion(Q[c], int(levels[c]), p, dec, 1)]
                                         for c in range(C)], dtype=np.int8)
        digits = list(np.ndindex(*(3,) * dim))
        out[pre + "interp"] = np.stack([rt.interpolate_volume(t, Q[0], dg) for dg in digits])
        children = {dg: rng.standard_normal((m,) + (n,) * dim) for dg in digits}
        out[pre + "children"] = np.stack([children[dg] for dg in digits])
        out[pre + "restrict"] = rt.restrict_volume(t, children)
        # refine -> coarsen round trip of a parent polynomial (reproduced exactly up to rounding)
        out[pre + "roundtrip"] = rt.restrict_volume(t, {dg: rt.interpolate_volume(t, Q[3], dg) for dg in digits})
    out["amr_decision"] = np.array([dec.refine_tol, dec.coarsen_tol, dec.max_level, 1.0])
    # plan_mesh_updates / apply_mesh_updates (transfer.py:161-219) on the
    # reference Mesh: a 9x9 periodic base with a refined 3x3 block, seeded
    # verdicts (refine, a fully agreeing coarsen cluster, a split cluster)
    for mi, (seed, p) in enumerate([(11, 3), (12, 2)]):
        mr = np.random.default_rng(seed)
        mesh = rm.build_uniform(2, dim=2, periodic=True)
        mesh.refine_many([mesh.real_cells[(2, (3, 3))], mesh.real_cells[(2, (4, 3))]])
        cells0 = sorted(mesh.real_cells)
        m, n = 4, p + 1
        sol = {k: mr.standard_normal((m, n, n)) for k in cells0}
        verdicts = {}
        fine = [k for k in cells0 if k[0] == 3]
        for k in fine:
            if k[1][0] // 3 == 3:
                verdicts[k] = rt.RefinementDecision.COARSEN                     # whole cluster agrees
            else:
                verdicts[k] = rt.RefinementDecision.COARSEN if mr.random() < 0.7 else rt.RefinementDecision.KEEP
        coarse = [k for k in cells0 if k[0] == 2]
        for k in mr.permutation(len(coarse))[:6]:
            verdicts[coarse[k]] = rt.RefinementDecision.REFINE
        for k in coarse[:3]:
            verdicts.setdefault(k, rt.RefinementDecision.KEEP)
        ref_nodes, co_parents = rt.plan_mesh_updates(mesh, verdicts)
        solutions = dict(sol)
        delta, new_data = rt.apply_mesh_updates(mesh, verdicts, solutions, p)
        code = {rt.RefinementDecision.REFINE: 1, rt.RefinementDecision.KEEP: 0, rt.RefinementDecision.COARSEN: -1}
        enc = lambda ks: np.array([[k[0], *k[1]] for k in ks], dtype=np.int64).reshape(-1, 3)   # noqa: E731
        pre = f"mesh{mi}_"
        out[pre + "order"] = np.array(p)
        out[pre + "cells0"] = enc(cells0)
        out[pre + "sol0"] = np.stack([sol[k] for k in cells0])
        vk = list(verdicts)
        out[pre + "verdict_keys"] = enc(vk)
        out[pre + "verdicts"] = np.array([code[verdicts[k]] for k in vk], dtype=np.int8)
        out[pre + "refine"] = enc([nd.key for nd in ref_nodes])
        out[pre + "coarsen"] = enc([pp.key for pp in co_parents])
        out[pre + "created"] = enc(sorted(delta.created_cells))
        out[pre + "removed"] = enc(sorted(delta.removed_cells))
        nk = sorted(new_data)
        out[pre + "new_keys"] = enc(nk)
        out[pre + "new_data"] = np.stack([new_data[k] for k in nk])
        out[pre + "cells1"] = enc(sorted(mesh.real_cells))
    out["mesh_ncases"] = np.array(2)
    np.savez_compressed(os.path.join(HERE, "amr.npz"), **out)
    print("amr.npz done")


if __name__ == "__main__":
    what = sys.argv[1:] or ["ops", "traj", "amr"]
    if "ops" in what:
        gen_ops()
    if "traj" in what:
        gen_traj()
    if "amr" in what:
        gen_amr()
