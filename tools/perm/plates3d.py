"""Lane -> node map of the 3-D p=4 STP kernel (one 5^3 cell per 128-thread CTA)
built from 2x2 'plates' (tools/probes: a warp-wide LDS.64 is one wavefront
when every lane quad asks for <= 2 words split 2+2 (or one word) and the
warp's distinct words fall in distinct bank pairs).  A plate in the (a1, a2)
plane gives 2 words split 2+2 on the loads along a1 and a2 and 4 words on the
third axis.  Prints the per-warp modelled wavefronts of the derivative loads
(row-major flux storage) against the row-major lane order."""
import itertools
N = 5


def rm(i, j, k):
    return (i * N + j) * N + k


def plates():
    q = []
    # warps 0, 1 and half of 2: (j,k) plates of every i-plane
    for i in range(N):
        for bj in (0, 2):
            for bk in (0, 2):
                q.append(('jk', [(i, bj, bk), (i, bj, bk + 1), (i, bj + 1, bk), (i, bj + 1, bk + 1)]))
    ik = [('ik', [(i, 4, k), (i, 4, k + 1), (i + 1, 4, k), (i + 1, 4, k + 1)]) for i in (0, 2) for k in (0, 2)]
    ij = [('ij', [(i, j, 4), (i, j + 1, 4), (i + 1, j, 4), (i + 1, j + 1, 4)]) for i in (0, 2) for j in (0, 2)]
    rest = [('line', [(4, 4, k) for k in range(4)]), ('line', [(4, j, 4) for j in range(4)]),
            ('line', [(i, 4, 4) for i in range(4)]), ('single', [(4, 4, 4), None, None, None])]
    return q[:16], q[16:] + ik, ij + rest


def lanes():
    w01, w2, w3 = plates()
    out = []
    for grp in (w01, w2, w3):
        for _, nodes in grp:
            out += nodes
    assert len(out) == 128
    return out


def wf(addr):
    best = 1
    for q in range(8):
        cnt = {}
        for t in range(4 * q, 4 * q + 4):
            if addr[t] is not None:
                cnt[addr[t]] = cnt.get(addr[t], 0) + 1
        best = max(best, (sum((c + 1) // 2 for c in cnt.values()) + 1) // 2)
    banks = {}
    for a in set(x for x in addr if x is not None):
        banks.setdefault(a % 16, set()).add(a)
    return max(best, max(len(s) for s in banks.values()))


def evaluate(lane_nodes, label):
    tot = 0
    for w in range(4):
        ln = lane_nodes[32 * w:32 * w + 32]
        per = []
        for a in range(3):
            s = 0
            for l in range(N):
                addr = []
                for n in ln:
                    if n is None:
                        addr.append(None)
                        continue
                    c = list(n)
                    c[a] = l
                    addr.append(rm(*c))
                s += wf(addr)
            per.append(s)
        st = wf([None if n is None else rm(*n) for n in ln])
        tot += sum(per)
        print(f"{label} warp {w}: loads axis0/1/2 = {per} (per l {[p / N for p in per]}), store {st}")
    print(f"{label}: total load wavefronts per time node and component {tot}")
    return tot


if __name__ == "__main__":
    rowmajor = [(n // 25, (n // 5) % 5, n % 5) if n < 125 else None for n in range(128)]
    evaluate(rowmajor, "row-major")
    p = lanes()
    assert sorted(rm(*n) for n in p if n is not None) == list(range(125))
    evaluate(p, "plates")
    print([-1 if n is None else rm(*n) for n in p])
