"""Host side of dynamic AMR: plan_mesh_updates and
the topology update of AdaptiveMesh against the reference's own
plan_mesh_updates / apply_mesh_updates on the same mesh and verdicts
(tests/golden/amr.npz, generated from the reference by make_golden.py)."""
import os

import numpy as np
import pytest

from paper_1806_07984_b200 import amr
from paper_1806_07984_b200.errors import ConfigError
from paper_1806_07984_b200.mesh import AdaptiveMesh

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "amr.npz"))
CODE = {1: amr.REFINE, 0: amr.KEEP, -1: amr.COARSEN}


def keys(a):
    return [(int(r[0]), (int(r[1]), int(r[2]))) for r in a]


def case(mi):
    pre = f"mesh{mi}_"
    mesh = AdaptiveMesh(keys(G[pre + "cells0"]), 2, True)
    verdicts = {k: CODE[int(v)] for k, v in zip(keys(G[pre + "verdict_keys"]), G[pre + "verdicts"])}
    return pre, mesh, verdicts


@pytest.mark.parametrize("mi", range(int(G["mesh_ncases"])))
def test_plan_and_topology_match_reference(mi):
    pre, mesh, verdicts = case(mi)
    refine, coarsen = amr.plan_mesh_updates(mesh, verdicts)
    assert refine == keys(G[pre + "refine"])
    assert coarsen == keys(G[pre + "coarsen"])
    delta = mesh.update_topology(refine, coarsen)
    assert sorted(delta.created_cells) == keys(G[pre + "created"])
    assert sorted(delta.removed_cells) == keys(G[pre + "removed"])
    assert sorted(mesh.cells) == keys(G[pre + "cells1"])
    assert mesh.version == 1 and not delta.empty
    # the coarse owners of the new hanging faces are in the skeleton
    assert mesh.nparent > 0 and mesh.skeleton.size > 0


def test_topology_errors_leave_mesh_untouched():
    mesh = AdaptiveMesh([(1, (i, j)) for i in range(3) for j in range(3)], 2, True)
    mesh.update_topology([(1, (1, 1))], [])
    cells = list(mesh.cells)
    with pytest.raises(ConfigError):
        mesh.update_topology([(1, (1, 1))], [])           # no longer a real cell
    with pytest.raises(ConfigError):
        mesh.update_topology([], [(0, (0, 0))])           # one child is refined
    assert mesh.cells == cells and mesh.version == 1


def test_multi_level_jumps_up_to_max_chain():
    """Hanging-face chains of several levels are supported (mesh.py:67-100);
    a chain longer than MAX_CHAIN is a ConfigError and leaves the mesh as is."""
    from paper_1806_07984_b200.mesh import MAX_CHAIN
    mesh = AdaptiveMesh([(1, (i, j)) for i in range(3) for j in range(3)], 2, True)
    mesh.update_topology([(1, (1, 1))], [])
    mesh.update_topology([(2, (3, 3))], [])          # level 3 next to a level-1 cell: a 2-level chain
    assert mesh.max_chain == 2 and mesh.nparent > 0
    lvl, idx = 3, (9, 9)
    for _ in range(MAX_CHAIN - 2):                  # deepen the corner chain to MAX_CHAIN levels
        mesh.update_topology([(lvl, idx)], [])
        lvl, idx = lvl + 1, (3 * idx[0], 3 * idx[1])
    assert mesh.max_chain == MAX_CHAIN
    before = list(mesh.cells)
    with pytest.raises(ConfigError):
        mesh.update_topology([(lvl, idx)], [])      # one level more
    assert mesh.cells == before


def test_coarsen_merges_a_real_cluster():
    mesh = AdaptiveMesh([(1, (i, j)) for i in range(3) for j in range(3)], 2, True)
    d = mesh.update_topology([], [(0, (0, 0))])
    assert mesh.cells == [(0, (0, 0))] and d.created_cells == {(0, (0, 0))} and len(d.removed_cells) == 9
