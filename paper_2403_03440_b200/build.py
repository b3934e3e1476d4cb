"""Build the sm_100a library in-tree: paper_2403_03440_b200/_lib/libcsflow_b200.so.

nvcc compiles each csrc/*.cu to an object in parallel, then links one shared
library against the CUDA runtime.  The .so travels to the GPU box with the
repo snapshot (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libcsflow_b200.so")
OBJDIR = os.path.join(ROOT, "build", "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
BUCKETS = (2, 4, 5, 6, 8, 12, 16, 20, 24, 32, 40, 48, 64)  # csb_common.cuh CSB_BUCKET_LIST
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(ROOT, "include", "csflow_b200.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False, extra_flags=(), tag=None):
    """Compile and link the library.  ``tag`` builds an experiment variant
    (``extra_flags`` such as -DCSB_RES_MINB=3) into _variants/<tag>/ with its
    own object directory; load it with CSB_LIB_PATH."""
    global OBJDIR, LIB
    saved = (OBJDIR, LIB)
    if tag:
        OBJDIR = os.path.join(ROOT, "build", f"obj_{tag}")
        LIB = os.path.join(ROOT, "_variants", tag, "libcsflow_b200.so")
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
    try:
        return _build(verbose, force, extra_flags)
    finally:
        OBJDIR, LIB = saved


def _build(verbose, force, extra_flags):
    os.makedirs(OBJDIR, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    cc = nvcc()
    hdrs = _headers()
    jobs = []
    objs = []
    units = []
    for src in _sources():
        if os.path.basename(src) == "csb_bucket.cu":
            for b in BUCKETS:
                units.append((src, f"csb_bucket_{b}.o", [f"-DCSB_BUCKET={b}"]))
        else:
            units.append((src, os.path.basename(src)[:-3] + ".o", []))
    for src, oname, defs in units:
        obj = os.path.join(OBJDIR, oname)
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs + [__file__]):
            cmd = [cc, *ARCH, *FLAGS, *defs, *extra_flags, "-c", src, "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
        return p.stderr

    if jobs:
        with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
            for out in ex.map(run, jobs):
                if verbose and out:
                    print(out, file=sys.stderr)
    if force or jobs or _stale(LIB, objs):
        cmd = [cc, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        run(cmd)
    return LIB


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("-") or a.startswith("-D")]
    tag = next((a[6:] for a in sys.argv[1:] if a.startswith("--tag=")), None)
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, extra_flags=defs, tag=tag))
