"""Build libdp.so (CUDA, sm_100a) in-tree with nvcc.

    python -m paper_1804_10987_b200._build [--force] [--verbose]

The shared library links NCCL from the torch-bundled `nvidia.nccl` wheel
(rpath set to its lib/ directory) and the static CUDA runtime.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libdp.so")
# one translation unit per kernel group (compiled in parallel, then linked)
SOURCES = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
DEPS = SOURCES + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "dp.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    cands = []
    try:
        import nvidia.nccl as nn  # torch-bundled NCCL 2.28

        base = list(nn.__path__)[0]
        cands.append(base)
    except Exception:
        pass
    cands += glob.glob("/opt/prime-rl/.venv/lib/python3*/site-packages/nvidia/nccl")
    for b in cands:
        inc, lib = os.path.join(b, "include"), os.path.join(b, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
            return inc, lib
    raise RuntimeError("NCCL headers/library not found (expected the nvidia-nccl wheel)")


def nvcc():
    for p in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.sep not in p or os.path.exists(p):
            return p
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile libdp.so; `out`/`defines` build experiment variants (e.g. -DDP_VARIANT=1)."""
    if out is not None:
        global LIB
        saved, LIB = LIB, out
        try:
            return build(force=True, verbose=verbose, defines=defines)
        finally:
            LIB = saved
    if not force and not stale():
        return LIB
    inc, lib = nccl_dirs()
    libname = os.path.basename(sorted(glob.glob(os.path.join(lib, "libnccl.so*")))[0])
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden", "-DDP_BUILD", *[f"-D{d}" for d in defines],
              "-I", INCLUDE, "-I", CSRC, "-I", inc]
    if verbose:
        common.insert(1, "-Xptxas=-v")
    tmp = tempfile.mkdtemp(prefix="dpbuild_")
    objs = [os.path.join(tmp, os.path.basename(src)[:-3] + ".o") for src in SOURCES]

    def compile_one(args):
        src, obj = args
        cmd = [*common, "-c", src, "-o", obj]
        print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0 or verbose:
            sys.stderr.write(r.stderr)
        return r.returncode

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        rcs = list(ex.map(compile_one, zip(SOURCES, objs)))
    if any(rcs):
        raise subprocess.CalledProcessError(max(rcs), "nvcc -c")
    link = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", LIB + ".tmp",
            "-L", lib, f"-l:{libname}", "-Xlinker", f"-rpath,{lib}"]
    print(" ".join(link), file=sys.stderr)
    subprocess.check_call(link)
    for o in objs:
        os.remove(o)
    os.rmdir(tmp)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--out=")]
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, out=outs[0] if outs else None,
          defines=defs)
