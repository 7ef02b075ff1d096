"""In-tree build of libafgpu.so (sm_100a) with nvcc.

The parity build uses --fmad=false: the reference CPU build (x86-64, -O3, no
-mfma) never contracts a*b+c into an FMA, so disabling contraction on the GPU
is what makes the results bit-identical. Division and sqrt are IEEE
correctly rounded in both.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libafgpu.so")

SOURCES = ["af_abi.cu", "af_uniform.cu", "af_fv3d_tol.cu", "af_mr.cu", "af_mr_full_tol.cu",
           "af_mr_dist.cu", "af_io.cu", "af_mr_storage.cu", "af_amr.cu"]
# translation units compiled WITH FMA contraction (tolerance-mode kernels only)
FMAD_TRUE = {"af_fv3d_tol.cu", "af_mr_full_tol.cu"}
HEADERS = sorted(f for f in os.listdir(os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc"))
                 if f.endswith((".cuh", ".h")))
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "-Xcompiler", "-fno-fast-math",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _nccl_dirs() -> tuple[str, str]:
    """torch's bundled NCCL (the one libtorch_cuda needs; one libnccl.so.2 per
    process, so libafgpu must use the same build)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []) or []:
        inc, lib = os.path.join(base, "nccl", "include"), os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(ROOT, "include", f) for f in ("af_gpu.h", "af_cases.h")]
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def _deps(src: str, seen: set | None = None) -> set:
    """The quoted includes of a translation unit, followed recursively (csrc/ and
    include/), so that only the objects a change reaches are recompiled."""
    import re
    seen = set() if seen is None else seen
    if src in seen or not os.path.exists(src):
        return seen
    seen.add(src)
    with open(src) as f:
        for name in re.findall(r'^\s*#\s*include\s+"([^"]+)"', f.read(), re.M):
            for base in (CSRC, os.path.join(ROOT, "include")):
                _deps(os.path.join(base, name), seen)
    return seen


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    srcs = [os.path.join(CSRC, f) for f in SOURCES if os.path.exists(os.path.join(CSRC, f))]
    nccl_inc, nccl_lib = _nccl_dirs()
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", CSRC, "-I", os.path.join(ROOT, "include"), "-I", nccl_inc]
    # one nvcc per translation unit, in parallel, then one link
    procs, objs = [], []
    for src in srcs:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if (not force and os.path.exists(obj) and
                all(os.path.getmtime(d) <= os.path.getmtime(obj) for d in _deps(src))
                and os.path.getmtime(os.path.abspath(__file__)) <= os.path.getmtime(obj)):
            continue
        flags = list(NVCC_FLAGS)
        if os.path.basename(src) in FMAD_TRUE:
            flags[flags.index("--fmad=false")] = "--fmad=true"
        cmd = [_nvcc(), *flags, *(["-Xptxas=-v"] if verbose else []), *inc, "-c", src,
               "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, subprocess.Popen(cmd)))
    bad = [src for src, p in procs if p.wait() != 0]
    if bad:
        raise subprocess.CalledProcessError(1, "nvcc " + " ".join(bad))
    link = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
            "-Xcompiler", "-fPIC", "-o", LIB + ".tmp", *objs, "-L", nccl_lib, "-l:libnccl.so.2",
            "-Xlinker", "-rpath", "-Xlinker", nccl_lib]
    subprocess.run(link, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
