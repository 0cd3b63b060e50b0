"""CPU oracle for the ADER-DG cell/face hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the algorithms of the reference package
`enclavedg` (arXiv 1806.07984 companion code, /root/reference/pkg/src/enclavedg)
for the hot path named in BASELINE.json:north_star.  Every function cites the
reference file:line it follows.

Who may import it: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
CPU legs (`cpu_baseline` and `--impl reference`).  It is the checker, never the
thing measured for the GPU arm and never a fallback: the product package
`paper_1806_07984_b200` does not import anything from here.

Pinning: the restatement is checked against golden vectors produced by running
the reference package itself in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`); see
`tests/test_oracle_golden.py`.

Modules
  ops       per-cell restatement (basis, PDE plugins incl. the added Euler
            system, STP Picard / CK, Rusanov, corrector, FV patch, dt)
  batched   the same arithmetic with a leading cell axis (bitwise equal to
            `ops` on the same inputs; used at scale)
  transfer  3:1 face/volume transfer operators
  spacetree restatement of the reference spacetree face forest (hanging-face
            chains, cell classification) for the AMR configuration
  drivers   Algorithm-1 three-loop time-step drivers
"""
