"""Generate / check the 3-D p=4 STP lane->node map (csrc/edg_stp.cuh kStpPerm3d5).

Warp w of the 128-thread CTA takes a compact block of (i1, i2) pencil pairs
with all five i0 values (+ the leftover pair's nodes), so a warp-wide LDS.64
touches <= 16 distinct pencils -- one shared-memory wavefront -- per axis
(warp 3: 20 on axis 1).  Prints per-warp distinct-pencil counts."""
blocks = [
    [(i1, i2) for i1 in (0, 1) for i2 in (0, 1, 2)],
    [(i1, i2) for i1 in (2, 3) for i2 in (0, 1, 2)],
    [(i1, i2) for i1 in (0, 1, 2) for i2 in (3, 4)],
    [(3, 3), (3, 4), (4, 3), (4, 4), (4, 1), (4, 2)],
]
extra = {0: [(0, 4, 0), (1, 4, 0)], 1: [(2, 4, 0), (3, 4, 0)], 2: [(4, 4, 0)], 3: []}
perm = []
for w in range(4):
    nodes = [(i0, i1, i2) for (i1, i2) in blocks[w] for i0 in range(5)] + extra[w]
    real = list(nodes)
    nodes += [None] * (32 - len(nodes))
    perm += [-1 if n is None else n[0] * 25 + n[1] * 5 + n[2] for n in nodes]
    print(f"warp {w}: {len(real)} nodes, distinct pencils axis0 {len({(a[1], a[2]) for a in real})} "
          f"axis1 {len({(a[0], a[2]) for a in real})} axis2 {len({(a[0], a[1]) for a in real})}")
assert sorted(p for p in perm if p >= 0) == list(range(125))
print(perm)
