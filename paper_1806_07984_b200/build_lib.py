"""Build libenclavedg_b200.so in-tree with nvcc for sm_100a.

    python -m paper_1806_07984_b200.build_lib [--jobs N] [--force]

Each csrc/*.cu is compiled to an object in parallel (one per PDE x dim
instantiation unit plus the ABI unit) and linked into
paper_1806_07984_b200/_lib/libenclavedg_b200.so.  The objects and the .so are
git-ignored but travel to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libenclavedg_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", os.path.join(os.path.dirname(HERE), "include")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, obj, defines=()):
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    log = obj + ".ptxas.txt"
    with open(log, "w") as fh:
        fh.write(p.stdout + p.stderr)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{p.stderr[-4000:]}")
    return obj


def build(jobs=None, force=False, verbose=True, defines=(), variant=None):
    """Build the library; `defines` (e.g. EDG_FV_CPT=1) with a `variant` name
    go to _lib/<variant>/ for A/B experiments (bench.py --lib <path>)."""
    out_dir = OUT_DIR if variant is None else os.path.join(OUT_DIR, variant)
    lib = os.path.join(out_dir, "libenclavedg_b200.so")
    os.makedirs(out_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(os.path.dirname(HERE), "include", "*.h"))
    objs = []
    todo = []
    for s in srcs:
        o = os.path.join(out_dir, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s, *hdrs]):
            todo.append((s, o))
    if todo:
        jobs = jobs or min(len(todo), os.cpu_count() or 4)
        with cf.ThreadPoolExecutor(jobs) as ex:
            list(ex.map(lambda so: _compile(*so, defines=defines), todo))
        if verbose:
            print(f"compiled {len(todo)} unit(s)", file=sys.stderr)
    if force or todo or _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stderr[-4000:]}")
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    ap.add_argument("--variant", default=None)
    a = ap.parse_args()
    print(build(a.jobs, a.force, defines=a.defines, variant=a.variant))
