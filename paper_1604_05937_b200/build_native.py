"""Build libprismesh_cuda.so in-tree with nvcc for sm_100a.

Every ``csrc/*.cu`` / ``csrc/*.cpp`` is compiled to an object under
``build/obj`` (rebuilt when the source or any header is newer) and linked
into ``paper_1604_05937_b200/_native/libprismesh_cuda.so``.  The built
library is git-ignored but travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJDIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "_native", "libprismesh_cuda.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# diag 128 ("loop is not reachable"): the window-fill steps of the strip
# kernels return before the cell computation on purpose (compile-time)
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-O3", "--expt-relaxed-constexpr",
         "-diag-suppress", "128", "-I", INCLUDE, "-I", CSRC]


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.cuh")) +
            glob.glob(os.path.join(CSRC, "*.h")) +
            glob.glob(os.path.join(INCLUDE, "*.h")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, ptxas_verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) +
                  glob.glob(os.path.join(CSRC, "*.cpp")))
    headers = _headers()
    # objects built with other -D flags are stale
    flags = " ".join([os.environ.get("PM_EXPERIMENTAL", "0"),
                      os.environ.get("PM_NVCC_EXTRA", "")])
    stamp = os.path.join(OBJDIR, ".flags")
    old = open(stamp).read() if os.path.exists(stamp) else None
    if old != flags:
        for o in glob.glob(os.path.join(OBJDIR, "*.o")):
            os.remove(o)
        with open(stamp, "w") as fh:
            fh.write(flags)
    objs, cmds = [], []
    for src in srcs:
        obj = os.path.join(OBJDIR, os.path.basename(src) + ".o")
        objs.append(obj)
        if not _stale(obj, [src] + headers):
            continue
        # PM_NVCC_EXTRA: extra -D tuning flags (experiments, e.g. -DPM_SR_DEPTH=6)
        # PM_EXPERIMENTAL=1: also compile the experimental schedules (tile,
        # store-first patch strips), slower than the defaults
        exp = ["-DPM_EXPERIMENTAL=1"] if os.environ.get(
            "PM_EXPERIMENTAL", "0") != "0" else []
        cmd = [NVCC, *ARCH, *FLAGS, *exp,
               *os.environ.get("PM_NVCC_EXTRA", "").split(),
               "-c", src, "-o", obj]
        if ptxas_verbose and src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        if src.endswith(".cpp"):
            cmd += ["-x", "cu"]
        cmds.append(cmd)
    # translation units are independent: compile them side by side
    from concurrent.futures import ThreadPoolExecutor
    jobs = max(1, min(len(cmds), os.cpu_count() or 1))

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r
    with ThreadPoolExecutor(jobs) as pool:
        for cmd, r in pool.map(run, cmds):
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            if verbose or r.returncode:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode:
                raise subprocess.CalledProcessError(r.returncode, cmd)
    if _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, ptxas_verbose="-v" in sys.argv))
