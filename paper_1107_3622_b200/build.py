"""Build libksort.so (the sm_100a K-sort engine) in-tree with nvcc.

    python -m paper_1107_3622_b200.build        # or __graft_entry__.build()

SASS for sm_100a only (no PTX JIT), -lineinfo for ncu source pages, static
cudart so the .so carries its own runtime (it shares the primary context and
the caller's stream with PyTorch).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libksort.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _git_rev() -> str:
    try:
        return subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True,
                              text=True, check=True).stdout.strip() or "dev"
    except Exception:
        return "dev"


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    lib = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    defs = os.environ.get("KS_DEFS", "").split()   # experiment variants: extra -D flags
    objdir = os.path.join(HERE, "build", "v_" + "_".join(d.lstrip("-D").replace("=", "") for d in defs)) if defs \
        else os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
             f'-DKS_GIT="{_git_rev()}"', *ARCH]
    if verbose:
        flags += ["-Xptxas", "-v"]
    if os.environ.get("KS_TRACE"):
        flags += ["-DKS_TRACE"]
    flags += defs
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        subprocess.run([nvcc, *flags, "-c", src, "-o", obj], check=True)
        objs.append(obj)
    tmp = lib + ".tmp"
    subprocess.run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs], check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    out = None
    if "--out" in sys.argv:
        out = sys.argv[sys.argv.index("--out") + 1]
    print(build(force="--force" in sys.argv or out is not None, verbose="-v" in sys.argv, out=out))
