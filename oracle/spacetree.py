"""Face-forest restatement of the reference spacetree (oracle only).

Restates the parts of /root/reference/pkg/src/enclavedg/mesh.py that the
Algorithm-1 driver needs on a static adaptive mesh:
  * SFC (depth-first, lexicographic child digits) cell order  mesh.py:322-338
  * root-face selection                                      mesh.py:346-353
  * face records with hanging-face children and child_pos    mesh.py:355-424
  * 'coarse' sides re-tagged as 'virtual'                    mesh.py:470-483
  * side_face_key                                            mesh.py:221-227
  * classify_cell (no decomposition)                         mesh.py:585-596

The mesh is given directly by its set of real cells {(level, index)} instead
of by refine operations; tests/test_oracle_golden.py pins the result against
the reference Mesh (face keys, side tags, owners, child_pos, classes).
"""
from __future__ import annotations


class Face:
    __slots__ = ("key", "axis", "level", "pos", "sides", "owners", "children", "parent", "child_pos")

    def __init__(self, key):
        self.key = key
        self.axis, self.level, self.pos = key
        self.sides = [None, None]     # tag in {'cell', 'virtual', 'boundary', 'refined'}
        self.owners = [None, None]    # (level, index) of the real cell covering the side
        self.children = None
        self.parent = None
        self.child_pos = None

    @property
    def is_leaf(self):
        return not self.children


class FaceForest:
    def __init__(self, cells, dim, periodic, extent=1.0):
        self.dim = dim
        self.periodic = periodic
        self.extent = extent
        self.cells = set((int(l), tuple(int(i) for i in ix)) for l, ix in cells)
        self.max_level = max(l for l, _ in self.cells)
        self.sfc = sorted(self.cells, key=self._sfc_key)
        self.faces = {}
        self._build()

    # geometry ------------------------------------------------------------
    def cell_edges(self, level):
        return tuple(self.extent / 3 ** level for _ in range(self.dim))

    def _sfc_key(self, cell):
        level, idx = cell
        return tuple(tuple((idx[t] // 3 ** (level - l)) % 3 for t in range(self.dim))
                     for l in range(1, level + 1))

    def region(self, level, idx):
        """mesh.py:198-209: the real cell at level <= `level` covering idx, else refined."""
        for lev in range(level + 1):
            key = (lev, tuple(i // 3 ** (level - lev) for i in idx))
            if key in self.cells:
                return "cell", key
        return "refined", (level, tuple(idx))

    def neighbour_index(self, idx, level, axis, side):
        """mesh.py:211-219."""
        n = 3 ** level
        j = idx[axis] + (1 if side == 1 else -1)
        if 0 <= j < n:
            return idx[:axis] + (j,) + idx[axis + 1:]
        if self.periodic:
            return idx[:axis] + (j % n,) + idx[axis + 1:]
        return None

    def side_face_key(self, cell, axis, side):
        """mesh.py:221-227."""
        level, idx = cell
        n = 3 ** level
        p = idx[axis] + side
        if self.periodic and p == n:
            p = 0
        return (axis, level, idx[:axis] + (p,) + idx[axis + 1:])

    def _face_cells(self, key):
        """mesh.py:229-243."""
        axis, level, pos = key
        n = 3 ** level
        upper = pos if pos[axis] < n else None
        la = pos[axis] - 1
        if la < 0:
            la = n - 1 if self.periodic else None
        lower = pos[:axis] + (la,) + pos[axis + 1:] if la is not None else None
        if not self.periodic:
            if pos[axis] == 0:
                lower = None
            if pos[axis] == n:
                upper = None
        return lower, upper

    # construction ----------------------------------------------------------
    def _root_key(self, cell, axis, side):
        """mesh.py:346-353."""
        level, idx = cell
        nb = self.neighbour_index(idx, level, axis, side)
        if nb is None:
            return self.side_face_key(cell, axis, side)
        tag, other = self.region(level, nb)
        if tag == "cell" and other[0] < level:
            return self.side_face_key(other, axis, 1 - side)
        return self.side_face_key(cell, axis, side)

    def _build(self):
        roots = set()
        for cell in self.sfc:
            for a in range(self.dim):
                for s in (0, 1):
                    roots.add(self._root_key(cell, a, s))
        for key in sorted(roots):
            if key not in self.faces:
                self._make(key)

    def _make(self, key):
        """mesh.py:378-420 with the finalize step of mesh.py:470-483 folded in."""
        axis, level, pos = key
        f = Face(key)
        self.faces[key] = f
        hanging = False
        for s, idx in enumerate(self._face_cells(key)):
            if idx is None:
                f.sides[s] = "boundary"
                continue
            tag, node = self.region(level, idx)
            if tag == "refined":
                hanging = True
                f.sides[s] = "refined"
            elif node[0] == level:
                f.sides[s] = "cell"
                f.owners[s] = node
            else:
                f.sides[s] = "virtual"
                f.owners[s] = node
        if hanging:
            f.children = []
            trans = [t for t in range(self.dim) if t != axis]
            n_next = 3 ** (level + 1)
            pa = 3 * pos[axis]
            if self.periodic and pa == n_next:
                pa = 0
            for digits in _digit_tuples(self.dim - 1):
                cpos = [3 * p for p in pos]
                cpos[axis] = pa
                for t, dg in zip(trans, digits):
                    cpos[t] = 3 * pos[t] + dg
                ck = (axis, level + 1, tuple(cpos))
                child = self._make(ck)
                child.parent = f
                child.child_pos = digits
                f.children.append(child)
        return f

    # queries ---------------------------------------------------------------
    def leaf_faces(self):
        """Leaves in face-forest insertion order (children in child_pos order)."""
        return [f for f in self.faces.values() if f.is_leaf]

    def is_skeleton_amr(self, cell):
        """classify_cell without a decomposition (mesh.py:585-596)."""
        for a in range(self.dim):
            for s in (0, 1):
                f = self.faces.get(self.side_face_key(cell, a, s))
                if f is not None and f.children:
                    return True
        return False


def _digit_tuples(k):
    out = [()]
    for _ in range(k):
        out = [p + (j,) for p in out for j in (0, 1, 2)]
    return out

