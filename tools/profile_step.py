"""Run a few eager steps of one configuration (the target of an ncu capture).

    python tools/profile_step.py --config cfg3 [--steps 4] [--cells N]

e.g. ncu --set full --import-source on --clock-control none -k regex:stp_picard
     --launch-skip 3 --launch-count 1 -o gpurun_out/stp_cfg3 python tools/profile_step.py --config cfg3
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO))

import bench  # noqa: E402
from paper_1806_07984_b200 import configs as cf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--cells", type=int, default=None)
    ap.add_argument("--lib", default=None, help="variant build of libenclavedg_b200.so")
    a = ap.parse_args()
    import torch
    if a.lib:
        from paper_1806_07984_b200 import _lib
        _lib.load(a.lib)
    cfg = cf.CONFIGS[a.config]
    if a.cells:
        cfg = cfg.with_(cells=a.cells)
    s, Q0, _ = bench.build_solver(cfg)
    s.set_state(Q0)
    for _ in range(a.steps):
        s.step()
    torch.cuda.synchronize()
    print("ok", a.config, s.steps_done)


if __name__ == "__main__":
    main()
