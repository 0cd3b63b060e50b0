"""Host-side static mesh topology, exported once as index arrays for the GPU.

Two mesh kinds cover the BASELINE configurations:

* CartesianMesh -- uniform N^d cells, periodic or outflow, row-major cell
  order (configs 1-4; the reference's 3-partitioned tree only offers 3^k,
  SURVEY.md section 0).  Exports nbr[c][2a+s] (-1 = outflow).
* AdaptiveMesh -- a mesh of real cells (level, index) in the reference's SFC
  order (config 5), with up to MAX_CHAIN levels between face neighbours.
  Builds the same face forest as the reference Mesh (mesh.py:67-100,
  346-483): a coarse face whose other side is refined becomes a parent with
  3^(d-1) child faces in child_pos order, recursively while the fine side is
  refined further, and each leaf of such a chain has the fine cell on one
  side and a virtual side on the other (the coarse owner's trace
  interpolated level by level along the chain, transfer.py:75-79).  Exports
  the leaf-face list (with each leaf's interpolation path), the parent list
  (deepest level first, with per-level launch groups) and
  side_face[c][2a+s] (an index into the outcome array: leaves first, then
  parents), plus the skeleton / enclave split of the schedule.

Skeleton rule (BASELINE.json config 5, pinned in DESIGN.md): a cell is
skeleton iff one of its faces is hanging (coarse side of a parent face -- the
reference classify_cell, mesh.py:585-596 -- or fine side of a child face) or
its closure meets the synthetic partition cut x = 0.5.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError

MAX_CHAIN = 4      # levels a hanging-face chain may span (virtual-side interpolation path length)


def _row_major_strides(N, dim):
    return [N ** (dim - 1 - t) for t in range(dim)]


class CartesianMesh:
    def __init__(self, N: int, dim: int, periodic: bool, extent: float = 1.0):
        if dim not in (2, 3):
            raise ConfigError(f"dim must be 2 or 3, got {dim}")
        self.N, self.dim, self.periodic = N, dim, periodic
        self.h = extent / N
        self.ncells = N ** dim
        idx = np.stack(np.meshgrid(*[np.arange(N)] * dim, indexing="ij"), axis=-1).reshape(-1, dim)
        strides = np.array(_row_major_strides(N, dim))
        nbr = np.empty((self.ncells, 2 * dim), dtype=np.int32)
        for a in range(dim):
            for s in (0, 1):
                j = idx[:, a] + (1 if s else -1)
                ok = (j >= 0) & (j < N)
                jw = j % N
                nb = (idx.copy())
                nb[:, a] = jw
                lin = (nb * strides).sum(axis=1)
                if not periodic:
                    lin = np.where(ok, lin, -1)
                nbr[:, 2 * a + s] = lin
        self.index = idx
        self.nbr = nbr

    def cell_edges(self, level=None):
        return (self.h,) * self.dim


@dataclass
class MeshDelta:
    """Topology change between two mesh states (the reference's MeshDelta,
    mesh.py:104-115).  Face keys are this package's (axis, level, position)
    leaf-face keys."""
    created_cells: set = field(default_factory=set)
    removed_cells: set = field(default_factory=set)
    created_faces: set = field(default_factory=set)
    removed_faces: set = field(default_factory=set)

    @property
    def empty(self):
        return not (self.created_cells or self.removed_cells or self.created_faces or self.removed_faces)


class AdaptiveMesh:
    def __init__(self, cells, dim: int, periodic: bool, extent: float = 1.0, cut_x=0.5, max_depth: int = 10):
        if dim not in (2, 3):
            raise ConfigError(f"dim must be 2 or 3, got {dim}")
        self.dim, self.periodic, self.extent = dim, periodic, extent
        self.max_depth = max_depth
        self.version = 0
        self._init_cells(cells, cut_x)

    def _init_cells(self, cells, cut_x):
        dim, extent = self.dim, self.extent
        cells = [(int(l), tuple(int(i) for i in ix)) for l, ix in cells]
        self.cells = sorted(cells, key=self._sfc_key)
        self.ncells = len(self.cells)
        self.pos = {c: i for i, c in enumerate(self.cells)}
        self.levels = np.array([l for l, _ in self.cells], dtype=np.int32)
        h = extent / 3.0 ** self.levels
        self.edges = np.repeat(h[:, None], dim, axis=1)
        self.hmin = h.copy()
        self.cut_x = cut_x
        self._build()

    def cell_edges(self, level):
        return tuple(self.extent / 3 ** level for _ in range(self.dim))

    # ------------------------------------------------- topology updates --
    def child_keys(self, key):
        """The 3^d children of a cell key in the reference's child-digit order
        (mesh.py:170-181, digits row-major)."""
        level, idx = key
        return [(level + 1, tuple(3 * idx[t] + dg[t] for t in range(self.dim)))
                for dg in itertools.product(range(3), repeat=self.dim)]

    def parent_key(self, key):
        level, idx = key
        return None if level == 0 else (level - 1, tuple(i // 3 for i in idx))

    def _face_keys(self):
        return set(k[1:] for k in self._leaf_keys)

    def update_topology(self, refine_cells=(), coarsen_parents=(), cut_x="keep"):
        """Refine real cells into their 3^d children and merge fully real
        3^d clusters into their parents, then rebuild the face forest once
        (mesh.py:309-317).  Raises ConfigError for an invalid target (the
        reference's InvalidTargetError / NotCoarsenableError / CapacityError)
        and for hanging-face chains longer than MAX_CHAIN levels.  Returns a
        MeshDelta."""
        before_cells, before_faces = set(self.cells), self._face_keys()
        cells = set(self.cells)
        for key in refine_cells:
            if key not in cells:
                raise ConfigError(f"cannot refine {key}: not a real cell")
            if key[0] + 1 > self.max_depth:
                raise ConfigError(f"refinement beyond max depth {self.max_depth}")
            cells.remove(key)
            cells.update(self.child_keys(key))
        for parent in coarsen_parents:
            kids = self.child_keys(parent)
            if parent in cells or not all(k in cells for k in kids):
                raise ConfigError(f"cannot coarsen {parent}: children are not all real cells")
            cells.difference_update(kids)
            cells.add(parent)
        # build the new state first: an invalid result leaves the mesh untouched
        new = AdaptiveMesh(cells, self.dim, self.periodic, self.extent,
                           self.cut_x if cut_x == "keep" else cut_x, self.max_depth)
        version = self.version + 1
        self.__dict__.update(new.__dict__)
        self.version = version
        after_faces = self._face_keys()
        return MeshDelta(set(self.cells) - before_cells, before_cells - set(self.cells),
                         after_faces - before_faces, before_faces - after_faces)

    def _sfc_key(self, cell):
        level, idx = cell
        return tuple(tuple((idx[t] // 3 ** (level - l)) % 3 for t in range(self.dim)) for l in range(1, level + 1))

    def _covering(self, level, idx):
        """Real cell at level <= `level` covering idx, or None if refined."""
        for lev in range(level, -1, -1):
            key = (lev, tuple(i // 3 ** (level - lev) for i in idx))
            if key in self.pos:
                return key
        return None

    def _build(self):
        d = self.dim
        leaf = {}          # key -> dict(axis, cells[2], kinds[2], child_pos, vpath)
        parents = {}       # key -> {digits: child key (leaf or parent)}
        par_cp = {}        # parent key -> its digits within its own parent (None for a root)
        side_key = {}      # (cell, fs) -> face key (leaf or parent)
        for c in self.cells:
            level, idx = c
            n = 3 ** level
            for a in range(d):
                for s in (0, 1):
                    j = idx[a] + (1 if s else -1)
                    if not (0 <= j < n) and not self.periodic:
                        key = ("L", a, level, idx[:a] + (idx[a] + s,) + idx[a + 1:])
                        leaf[key] = dict(axis=a, cells=[self.pos[c], self.pos[c]],
                                         kinds=[2, 0] if s == 0 else [0, 2], child_pos=(0, 0), vpath=[])
                        side_key[(c, 2 * a + s)] = key
                        continue
                    nb = idx[:a] + (j % n,) + idx[a + 1:]
                    cov = self._covering(level, nb)
                    up = idx[a] + s
                    if self.periodic and up == n:
                        up = 0
                    fpos = idx[:a] + (up,) + idx[a + 1:]
                    if cov is not None and cov[0] == level:
                        key = ("L", a, level, fpos)
                        lo, hi = (c, cov) if s == 1 else (cov, c)
                        leaf[key] = dict(axis=a, cells=[self.pos[lo], self.pos[hi]], kinds=[0, 0], child_pos=(0, 0),
                                         vpath=[])
                        side_key[(c, 2 * a + s)] = key
                    elif cov is not None:
                        # this fine cell sits at the bottom of a chain of hanging faces
                        # below the coarse neighbour's side face (mesh.py:67-100,
                        # 378-420): parents at levels cov_level .. level-1, the leaf
                        # at `level` with the coarse owner on its virtual side
                        lc = cov[0]

                        def digits_at(l):
                            return tuple((idx[t] // 3 ** (level - l)) % 3 for t in range(d) if t != a)

                        def key_at(l, kind):
                            sh = 3 ** (level - l)
                            return (kind, a, l, tuple(fpos[t] // sh for t in range(d)))

                        vpath = [digits_at(l) for l in range(lc + 1, level + 1)]
                        key = key_at(level, "L")
                        lo, hi = (c, cov) if s == 1 else (cov, c)
                        kinds = [0, 1] if s == 1 else [1, 0]
                        leaf[key] = dict(axis=a, cells=[self.pos[lo], self.pos[hi]], kinds=kinds,
                                         child_pos=vpath[-1] + (0,) * (2 - len(vpath[-1])), vpath=vpath)
                        side_key[(c, 2 * a + s)] = key
                        child = key
                        for l in range(level - 1, lc - 1, -1):
                            pk = key_at(l, "P")
                            parents.setdefault(pk, {})[digits_at(l + 1)] = child
                            par_cp.setdefault(pk, digits_at(l) if l > lc else None)
                            child = pk
                    else:
                        key = ("P", a, level, fpos)
                        parents.setdefault(key, {})
                        par_cp.setdefault(key, None)
                        side_key[(c, 2 * a + s)] = key
        # coarse cells' sides on parents
        nch = 3 ** (d - 1)
        for pkey, ch in parents.items():
            if len(ch) != nch:
                raise ConfigError(f"parent face {pkey} has {len(ch)} children, expected {nch}")
        # classification (needs the face kinds), then the face order:
        # skeleton-only leaves first so each schedule phase is a contiguous range
        self.hanging = np.zeros(self.ncells, dtype=bool)
        for rec in leaf.values():
            if 1 in rec["kinds"]:
                self.hanging[rec["cells"]] = True
        x0 = np.array([ix[0] for _, ix in self.cells]) * self.hmin
        x1 = x0 + self.hmin
        cut = np.zeros(self.ncells, dtype=bool) if self.cut_x is None else (x0 <= self.cut_x) & (self.cut_x <= x1)
        self.skeleton_mask = self.hanging | cut
        self.skeleton = np.nonzero(self.skeleton_mask)[0].astype(np.int32)
        self.enclave = np.nonzero(~self.skeleton_mask)[0].astype(np.int32)
        on_skel = {k: bool(self.skeleton_mask[rec["cells"]].all()) for k, rec in leaf.items()}
        leaf_keys = sorted(leaf, key=lambda k: (not on_skel[k], k[1], k[2], k[3]))
        self._leaf_keys = leaf_keys
        self.nleaf_skeleton = sum(on_skel.values())
        # parents deepest level first (a parent is restricted after all of its
        # children, which may be parents one level below), grouped by level
        par_keys = sorted(parents, key=lambda k: (-k[2], k[1], k[3]))
        index = {k: i for i, k in enumerate(leaf_keys)}
        F = len(leaf_keys)
        for i, k in enumerate(par_keys):
            index[k] = F + i
        self.nleaf, self.nparent = F, len(par_keys)
        self.face_axis = np.array([leaf[k]["axis"] for k in leaf_keys], dtype=np.int32)
        self.face_cell = np.array([leaf[k]["cells"] for k in leaf_keys], dtype=np.int32).reshape(F, 2)
        self.face_kind = np.array([leaf[k]["kinds"] for k in leaf_keys], dtype=np.int8).reshape(F, 2)
        self.face_child_pos = np.array([leaf[k]["child_pos"] for k in leaf_keys], dtype=np.int8).reshape(F, 2)
        # virtual-side interpolation path of every leaf (coarsest level first)
        depth = max([len(leaf[k]["vpath"]) for k in leaf_keys] + [1])
        if depth > MAX_CHAIN:
            raise ConfigError(f"hanging-face chains deeper than {MAX_CHAIN} levels are not supported")
        self.max_chain = depth
        self.face_vdepth = np.array([len(leaf[k]["vpath"]) for k in leaf_keys], dtype=np.int8)
        self.face_vpath = np.zeros((F, MAX_CHAIN, 2), dtype=np.int8)
        for i, k in enumerate(leaf_keys):
            for l, dg in enumerate(leaf[k]["vpath"]):
                self.face_vpath[i, l, :len(dg)] = dg
        digits_all = list(itertools.product(range(3), repeat=d - 1))
        self.parent_face = np.arange(F, F + self.nparent, dtype=np.int32)
        self.parent_children = np.array([[index[parents[k][dg]] for dg in digits_all] for k in par_keys],
                                        dtype=np.int32).reshape(self.nparent, nch)
        # child position of every outcome row within its parent (leaves and parents)
        self.outcome_cp = np.zeros((F + self.nparent, 2), dtype=np.int8)
        self.outcome_cp[:F] = self.face_child_pos
        for i, k in enumerate(par_keys):
            dg = par_cp.get(k)
            if dg is not None:
                self.outcome_cp[F + i, :len(dg)] = dg
        # restriction launches: contiguous parent ranges of one level, deepest first
        self.parent_groups = []
        for i, k in enumerate(par_keys):
            if self.parent_groups and par_keys[i - 1][2] == k[2]:
                self.parent_groups[-1][1] += 1
            else:
                self.parent_groups.append([i, 1])
        leaf_children = self.parent_children[self.parent_children < F]
        if leaf_children.size and leaf_children.max() >= self.nleaf_skeleton:
            raise ConfigError("internal: a hanging child face is not on the skeleton")
        self.side_face = np.full((self.ncells, 2 * d), -1, dtype=np.int32)
        for (c, fs), k in side_key.items():
            self.side_face[self.pos[c], fs] = index[k]
        if (self.side_face < 0).any():
            raise ConfigError("internal: cell side without a face")
