"""Build libprism.so in-tree for sm_100a (B200) with nvcc.

``python -m paper_2605_08581_b200.build`` (or ``__graft_entry__.build()``).
nvcc cross-compiles without a GPU, so this runs in the build container.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libprism.so")
SOURCES = ["dart.cu", "qas.cu", "serve.cu", "trace_io.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def flags(extra: list[str] | None = None) -> list[str]:
    return [
        "-O3",
        "-std=c++17",
        *ARCH,
        "-lineinfo",
        "-fmad=false",  # QAS float expressions round like the reference's Python
        "--expt-relaxed-constexpr",
        "-Xcompiler",
        "-fPIC",
        "-I",
        os.path.join(ROOT, "include"),
        *(extra or []),
        *os.environ.get("PRISM_NVCC_EXTRA", "").split(),  # e.g. -DPRISM_TRACE (diagnostics builds)
    ]


def commands(out: str = LIB, extra: list[str] | None = None) -> tuple[list[list[str]], list[str]]:
    """(one compile command per translation unit, the link command): the units
    compile in parallel into build/, then one nvcc -shared links them."""
    objdir = os.path.join(ROOT, "build")
    srcs = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in srcs]
    comp = [[nvcc(), *flags(extra), "-c", "-o", o, s] for s, o in zip(srcs, objs)]
    link = [nvcc(), *ARCH, "-shared", "-o", out, *objs]
    return comp, link


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    mtime = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "prism.h")]
    return any(os.path.getmtime(p) > mtime for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = True) -> str:
    if force or needs_build():
        comp, link = commands()
        os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
        procs = []
        for cmd in comp:
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((cmd, subprocess.Popen(cmd)))
        for cmd, p in procs:
            if p.wait() != 0:
                raise subprocess.CalledProcessError(p.returncode, cmd)
        if verbose:
            print(" ".join(link), flush=True)
        subprocess.run(link, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
