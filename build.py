"""In-tree build of the three native libraries (run by __graft_entry__.build()).

* ``paper_1702_03484_b200/libmapsq.so`` — the product: sm_100a CUDA kernels + C ABI (nvcc).
* ``datagen/libdatagen.so``             — seeded input generators (gcc, OpenMP).
* ``oracle/liboracle.so``               — the CPU oracle, test infrastructure only (g++).

Each library is rebuilt only when one of its sources is newer than the .so, so importing a
package never pays for a compile once the tree has been built.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list[str]) -> None:
    print("[build]", " ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=ROOT)


def build_datagen(force: bool = False) -> str:
    src = [os.path.join(ROOT, "datagen", "datagen.c")]
    hdr = [os.path.join(ROOT, "datagen", "datagen.h")]
    out = os.path.join(ROOT, "datagen", "libdatagen.so")
    if force or _stale(out, src + hdr):
        _run(["gcc", "-O3", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-o", out, *src, "-lm"])
    return out


def build_oracle(force: bool = False) -> str:
    src = [os.path.join(ROOT, "oracle", "oracle.cpp")]
    hdr = [os.path.join(ROOT, "oracle", "oracle.h")]
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    if force or _stale(out, src + hdr):
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-o", out, *src])
    return out


def build_mapsq(force: bool = False) -> str:
    csrc = os.path.join(ROOT, "paper_1702_03484_b200", "csrc")
    cu = sorted(glob.glob(os.path.join(csrc, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(csrc, "*.cuh")) + glob.glob(os.path.join(csrc, "*.h"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))
    out = os.path.join(ROOT, "paper_1702_03484_b200", "libmapsq.so")
    if force or _stale(out, cu + hdrs):
        objdir = os.path.join(ROOT, "build", "mapsq")
        os.makedirs(objdir, exist_ok=True)
        objs = []
        for f in cu:
            o = os.path.join(objdir, os.path.basename(f) + ".o")
            # MAPSQ_NVCC_DEFS: extra -D flags for ablation builds (tools/gpu_ablate_*.sh)
            extra = os.environ.get("MAPSQ_NVCC_DEFS", "").split()
            _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr", *extra,
                  "-I", os.path.join(ROOT, "include"), "-c", f, "-o", o])
            objs.append(o)
        _run([NVCC, *ARCH, "-shared", "-o", out, *objs, "-cudart", "static", "-ldl"])
    return out


def build_all(force: bool = False) -> None:
    build_datagen(force)
    build_oracle(force)
    build_mapsq(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
