"""Time edg_pack_face_traces / edg_unpack_face_traces (row f3) on cfg3's
geometry: 64^3 cells, p = 4, 5 variables, traces (C, 6, 5, 25) fp64, cut
into R SFC ranks; prints one JSON line per R with the per-launch time and
the algorithmic bytes (row read + row written, 2 * 2*m*n^2*8 per face).

    python tools/bench_pack.py            # on a GPU box
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_07984_b200.decomposition import (decompose, exchange_plan, pack_boundary_traces,  # noqa: E402
                                                 unpack_boundary_traces)
from paper_1806_07984_b200.mesh import CartesianMesh  # noqa: E402


def main():
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    mesh = CartesianMesh(64, 3, False)
    m, n = 5, 5
    tq = torch.rand((mesh.ncells, 6, m, n * n), dtype=torch.float64, device="cuda")
    tf = torch.rand_like(tq)
    for R in (2, 8):
        dec = decompose(mesh, R)
        plan = exchange_plan(mesh, dec, 0)
        peer = max(plan.peers, key=lambda p: plan.faces[p].size)
        k = plan.faces[peer].size
        out = pack_boundary_traces(plan, peer, tq, tf)
        ghost = torch.empty_like(out)
        slots = torch.arange(k, dtype=torch.int32, device="cuda")
        reps = 200
        for fn in ("pack", "unpack"):
            for _ in range(10):
                pack_boundary_traces(plan, peer, tq, tf) if fn == "pack" else unpack_boundary_traces(out, slots, ghost)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                pack_boundary_traces(plan, peer, tq, tf) if fn == "pack" else unpack_boundary_traces(out, slots, ghost)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / reps
            nbytes = 2 * out.numel() * 8
            print(json.dumps({"kernel": fn, "ranks": R, "faces": k, "us_per_call": round(us, 2),
                              "bytes": nbytes, "gbs": round(nbytes / us / 1e3, 1), "hbm_peak_gbs": peak,
                              "note": "per call: launch + kernel, indices resident"}))


if __name__ == "__main__":
    main()
