"""Face forest of a mesh with multi-level hanging-face chains, from the
REFERENCE mesh (mesh.py:67-100 FaceRecord chains, mesh.py:355-424 build).

    python tests/golden/make_golden_deep.py      (build container only)

Base 9x9 periodic (level 2); the cell (2,(4,4)) is refined to level 3 and its
corner child (3,(12,12)) once more to level 4, so level-4 cells face level-2
cells across two-level chains (and level-3 cells across one-level ones).  A
3-D variant (base 3^3, outflow) refines (1,(1,1,1)) and then its corner child
(2,(3,3,3)).  Writes tests/golden/mesh_deep.json: per mesh the SFC cell order,
the faces (key, side tags, owners, child count, child_pos, parent) and the
skeleton cells of classify_cell.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import enclavedg.mesh as rm  # noqa: E402


def record(mesh):
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
    return {"faces": faces, "skeleton": skel, "sfc": [[n.level, list(n.index)] for n in mesh.sfc_cells],
            "dim": mesh.dim, "periodic": mesh.periodic}


def main():
    out = {}
    m2 = rm.build_uniform(2, dim=2, periodic=True)
    m2.refine_many([m2.real_cells[(2, (4, 4))]])
    m2.refine_many([m2.real_cells[(3, (12, 12))]])
    out["deep2d"] = record(m2)
    m3 = rm.build_uniform(1, dim=3, periodic=False)
    m3.refine_many([m3.real_cells[(1, (1, 1, 1))]])
    m3.refine_many([m3.real_cells[(2, (3, 3, 3))]])
    out["deep3d"] = record(m3)
    with open(os.path.join(HERE, "mesh_deep.json"), "w") as fh:
        json.dump(out, fh)
    print({k: (len(v["sfc"]), len(v["faces"])) for k, v in out.items()})


if __name__ == "__main__":
    main()
