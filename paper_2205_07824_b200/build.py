"""Build libldgb200.so in-tree with nvcc for sm_100a.

    python -m paper_2205_07824_b200.build

The shared library lands in ``paper_2205_07824_b200/lib/`` (git-ignored, but
shipped to the GPU box with the repo snapshot).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib" / "libldgb200.so"
SOURCES = ["capi.cu", "ldg_tensor.cu", "ldg_fused.cu", "ldg_dense.cu", "krylov.cu",
           "bjacobi.cu", "jit.cu", "probe.cu", "comm.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (Path(c).exists() or c == "nvcc"):
            return c
    raise RuntimeError("nvcc not found")


def needs_build():
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + \
        list((ROOT / "include").glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build(force=False, verbose=False, out=None, defines=()):
    lib = Path(out) if out else LIB
    if not force and out is None and not needs_build():
        return LIB
    lib.parent.mkdir(parents=True, exist_ok=True)
    objs = []
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                    "--expt-relaxed-constexpr", "-Xcompiler", "-fopenmp", "-I", str(ROOT / "include"),
                    "-I", str(CSRC)] + [f"-D{d}" for d in defines]
    if verbose:
        flags += ["-Xptxas", "-v"]
    procs = []
    for src in SOURCES:
        obj = lib.parent / (Path(src).stem + ".o")
        objs.append(obj)
        cmd = [nvcc(), *flags, "-c", str(CSRC / src), "-o", str(obj)]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                            stderr=subprocess.STDOUT, text=True)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stdout.write(out)
        if p.returncode:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "shared", *map(str, objs), "-lnvrtc", "-lgomp", "-ldl",
           "-Xlinker", "-rpath=/usr/local/cuda/lib64", "-o", str(tmp)]
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    for o in objs:
        o.unlink(missing_ok=True)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
