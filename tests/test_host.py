"""CPU tests of the host side: the C-ABI library loads and exports every
declared symbol, the uploaded operator tables are the reference's bits, and
the host mesh builders reproduce the oracle / reference topology."""
import ctypes
import os

import numpy as np
import pytest

from paper_1806_07984_b200 import _lib, basis, configs, errors, mesh, pde
from oracle import spacetree


def test_library_loads_and_exports_header_symbols():
    lib = _lib.load()
    syms = _lib.header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} declared in the header but not bound"
    assert b"sm_100a" in lib.edg_build_info()


def test_library_compiled_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_supported_matrix():
    lib = _lib.load()
    e3 = pde.euler(3).native()
    e2 = pde.euler(2).native()
    assert lib.edg_supported(ctypes.byref(e2), 5) and lib.edg_supported(ctypes.byref(e2), 7)
    assert lib.edg_supported(ctypes.byref(e3), 4) and lib.edg_supported(ctypes.byref(e3), 7)
    bad = _lib.make_pde_struct("euler", 2, 5)
    assert not lib.edg_supported(ctypes.byref(bad), 3)


def test_status_mapping_and_config_errors():
    lib = _lib.load()
    st = lib.edg_stp_picard(ctypes.byref(pde.euler(2).native()), 9, None, None, None, 1, None, 0, None, 1e-10, 0,
                            None, None, None, None, None, None, None, None)
    assert st == 2
    with pytest.raises(errors.ConfigError):
        _lib.check(st, "stp")
    with pytest.raises(errors.ConfigError):
        basis.get_basis(0)


def test_packed_basis_table_is_reference_bits(golden_ops):
    for p in range(1, 8):
        b = basis.get_basis(p)
        n = p + 1
        tab = b.packed_table()
        assert np.array_equal(tab[:n * n].reshape(n, n), golden_ops[f"basis{p}_D"])
        assert np.array_equal(tab[n * n:n * n + n], golden_ops[f"basis{p}_weights"])
        kinv = tab[n * n + 3 * n: 2 * n * n + 3 * n].reshape(n, n)
        assert np.array_equal(kinv, golden_ops[f"basis{p}_kinv"])
        klift = tab[2 * n * n + 3 * n: 2 * n * n + 4 * n]
        assert np.array_equal(klift, (golden_ops[f"basis{p}_kinv"] @ golden_ops[f"basis{p}_lift"][:, None]).ravel())
        assert np.array_equal(tab[2 * n * n + 4 * n: 5 * n * n + 4 * n].reshape(3, n, n), golden_ops[f"basis{p}_interp"])
        assert np.array_equal(tab[5 * n * n + 4 * n:].reshape(3, n, n), golden_ops[f"basis{p}_restrict"])


def test_cartesian_neighbours():
    m = mesh.CartesianMesh(5, 3, False)
    assert m.nbr.shape == (125, 6)
    c = 1 * 25 + 2 * 5 + 3
    assert m.nbr[c, 0] == c - 25 and m.nbr[c, 1] == c + 25
    assert m.nbr[c, 4] == c - 1 and m.nbr[c, 5] == c + 1
    assert m.nbr[0, 0] == -1 and m.nbr[124, 5] == -1
    mp = mesh.CartesianMesh(4, 2, True)
    assert mp.nbr[0, 0] == 12 and mp.nbr[3, 3] == 0


@pytest.mark.parametrize("base", [9, 27])
def test_adaptive_mesh_matches_oracle_forest(base):
    cfg = configs.CONFIGS["cfg5"].with_(cells=base)
    cells = configs.amr_cells(cfg)
    am = mesh.AdaptiveMesh(cells, 2, True)
    ff = spacetree.FaceForest(cells, 2, True)
    assert am.cells == ff.sfc
    leaves = ff.leaf_faces()
    assert am.nleaf == len(leaves)
    assert am.nparent == sum(1 for f in ff.faces.values() if f.children)
    # every cell side resolves to the same neighbour relation
    kind_of = {"cell": 0, "virtual": 1, "boundary": 2}
    mine = set()
    for i in range(am.nleaf):
        cl = tuple(am.cells[c] for c in am.face_cell[i])
        mine.add((int(am.face_axis[i]), cl, tuple(int(k) for k in am.face_kind[i]),
                  int(am.face_child_pos[i, 0]) if 1 in am.face_kind[i] else -1))
    theirs = set()
    for f in leaves:
        cl = tuple(o if o is not None else None for o in f.owners)
        theirs.add((f.axis, cl, tuple(kind_of[s] for s in f.sides), f.child_pos[0] if f.child_pos else -1))
    assert mine == theirs
    # skeleton: reference classify_cell marks the coarse side; ours adds the fine side and the cut
    ref_coarse = {c for c in ff.sfc if ff.is_skeleton_amr(c)}
    ours = {am.cells[i] for i in am.skeleton}
    assert ref_coarse <= ours
    # corrector lookup: side_face of a coarse hanging side points at a parent
    for c_i, c in enumerate(am.cells):
        for fs in range(4):
            key = ff.side_face_key(c, fs >> 1, fs & 1)
            f = ff.faces[key]
            assert (am.side_face[c_i, fs] >= am.nleaf) == bool(f.children)


def test_configs_sizes_and_pins():
    c2 = configs.CONFIGS["cfg2"]
    assert configs.dof_count(c2) == 8503056
    assert configs.dof_count(configs.CONFIGS["cfg3"]) == 163840000
    assert configs.dof_count(configs.CONFIGS["cfg4"]) == 10485760
    assert configs.dof_count(configs.CONFIGS["cfg1"]) == 11664
    cells5 = configs.amr_cells(configs.CONFIGS["cfg5"])
    assert 12000 < len(cells5) < 15000
    P = configs.initial_fv(configs.CONFIGS["cfg4"].with_(cells=16))
    g = configs.patches_to_grid(P, 8)
    assert np.array_equal(configs.grid_to_patches(g, 8), P)


@pytest.mark.parametrize("name", ["deep2d", "deep3d"])
def test_adaptive_mesh_deep_chains_match_forest(name):
    """Multi-level chains: the device tables of AdaptiveMesh (leaf faces with
    their interpolation paths, parents deepest level first, each outcome row's
    child position) describe the reference face forest (mesh_deep.json,
    pinned to the reference Mesh by tests/test_oracle_golden.py)."""
    import json
    import os
    from oracle import drivers
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "mesh_deep.json")))[name]
    cells = [(l, tuple(ix)) for l, ix in ref["sfc"]]
    am = mesh.AdaptiveMesh(cells, ref["dim"], ref["periodic"])
    ff = spacetree.FaceForest(cells, ref["dim"], ref["periodic"])
    assert am.cells == ff.sfc
    assert am.nleaf == len(ff.leaf_faces())
    assert am.nparent == sum(1 for f in ff.faces.values() if f.children)
    assert am.max_chain == 2
    kind_of = {"cell": 0, "virtual": 1, "boundary": 2}
    mine = set()
    for i in range(am.nleaf):
        cl = tuple(None if am.face_kind[i, s] == 2 else am.cells[am.face_cell[i, s]] for s in (0, 1))
        depth = int(am.face_vdepth[i])
        path = tuple(tuple(int(v) for v in am.face_vpath[i, l, :ref["dim"] - 1]) for l in range(depth))
        mine.add((int(am.face_axis[i]), cl, tuple(int(k) for k in am.face_kind[i]), path))
    theirs = set()
    for f in ff.leaf_faces():
        path = tuple(drivers.virtual_path(f)) if "virtual" in f.sides else ()
        theirs.add((f.axis, tuple(f.owners), tuple(kind_of[s] for s in f.sides), path))
    assert mine == theirs
    # parents: deepest first, every parent's children complete before it is restricted
    F = am.nleaf
    done = set(range(F))
    for g0, gn in am.parent_groups:
        for p in range(g0, g0 + gn):
            assert all(int(c) in done for c in am.parent_children[p])
        done.update(range(F + g0, F + g0 + gn))
    # the coarse side of every chain reads a root parent
    for c_i, c in enumerate(am.cells):
        for fs in range(2 * ref["dim"]):
            f = ff.faces[ff.side_face_key(c, fs >> 1, fs & 1)]
            assert (am.side_face[c_i, fs] >= am.nleaf) == bool(f.children)
