"""Generate tests/golden/decomp.json from the REFERENCE mesh (row f3).

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_decomp.py

For uniform 3x3 (R in {2, 3, 4, 5}) and 9x9 periodic meshes and the 9x9 mesh
with a refined block (R in {2, 3, 4}), the decomposition is the contiguous SFC split of the
reference's own `mesh.sfc_cells` (SPEC.md rank-sim `decompose`); recorded are
the reference's `boundary_face_order(mesh, decomp, pair)` (mesh.py:613-628)
as (lo key, hi key, face key) triples in order, and the skeleton set of
`classify_cell(mesh, node, decomp)` (mesh.py:585-596).
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import enclavedg.mesh as rm  # noqa: E402


class _Decomp:
    def __init__(self, mesh, nranks):
        n = len(mesh.sfc_cells)
        base, extra = divmod(n, nranks)
        # secondary_order caches on (mesh.version, decomp.version): a distinct
        # version per decomposition keeps the cache from serving another R
        self.nranks, self.version, self._rank = nranks, nranks, {}
        i = 0
        for r in range(nranks):
            for _ in range(base + (1 if r < extra else 0)):
                self._rank[mesh.sfc_cells[i].key] = r
                i += 1

    def rank_of(self, key):
        return self._rank[key]


def _record(mesh, R):
    d = _Decomp(mesh, R)
    pairs = {}
    for r1 in range(R):
        for r2 in range(r1 + 1, R):
            fs = rm.boundary_face_order(mesh, d, (r1, r2))
            back = rm.boundary_face_order(mesh, d, (r2, r1))
            assert [f.key for f in fs] == [f.key for f in back]
            pairs[f"{r1},{r2}"] = [[list(f.owners[0].key), list(f.owners[1].key), list(f.key)] for f in fs]
    skel = [list(n.key) for n in mesh.sfc_cells if rm.classify_cell(mesh, n, d) is rm.CellClass.SKELETON]
    return dict(R=R, pairs=pairs, skeleton=skel)


def main():
    out = {}
    m3 = rm.build_uniform(1, dim=2, periodic=True)
    out["uniform3"] = dict(cells=[list(n.key) for n in m3.sfc_cells],
                           cases=[_record(m3, R) for R in (2, 3, 4, 5)])
    mesh = rm.build_uniform(2, dim=2, periodic=True)
    out["uniform9"] = dict(cells=[list(n.key) for n in mesh.sfc_cells],
                           cases=[_record(mesh, R) for R in (2, 3, 4)])
    ref = rm.build_uniform(2, dim=2, periodic=True)
    ref.refine_many([ref.real_cells[(2, (i, j))] for i in (3, 4) for j in (4, 5)])
    out["refined"] = dict(cells=[list(n.key) for n in ref.sfc_cells],
                          cases=[_record(ref, R) for R in (2, 3, 4)])
    with open(os.path.join(HERE, "decomp.json"), "w") as f:
        json.dump(out, f)
    print({k: len(v["cells"]) for k, v in out.items()})


if __name__ == "__main__":
    main()
