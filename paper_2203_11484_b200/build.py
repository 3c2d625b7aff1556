"""Build libvplgi.so in-tree with nvcc for sm_100a (no JIT cache, so the
shared object travels with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INC = PKG.parent / "include"
LIB = PKG / "libvplgi.so"
OBJ = PKG / "build"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["api.cu", "scene.cu", "bvh.cu", "generate.cu", "render.cu", "reject.cu"]
# -fmad=false: the bit-exact steps (DESIGN.md §3 O0) must not contract a*b+c;
# kernels that want FMA call fmaf() explicitly.
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
              "-Xptxas", "-warn-spills", f"-I{INC}"]


def _headers():
    return list(CSRC.glob("*.cuh")) + list(INC.glob("*.h"))


def build(force: bool = False, verbose: bool = False, defines: tuple = (), out: Path | None = None) -> Path:
    """Build libvplgi.so; `defines`/`out` build a tuning variant (tools/ only) into its own file."""
    lib = Path(out) if out else LIB
    extra = os.environ.get("VPLGI_NVCC_EXTRA", "").split() if out else []   # tuning variants only (tools/)
    tag = [d.replace("=", "") for d in defines] + [e.strip("-").replace("=", "") for e in extra]
    obj = OBJ if not tag else OBJ / ("v_" + "_".join(tag))
    obj.mkdir(parents=True, exist_ok=True)
    flags = NVCC_FLAGS + [f"-D{d}" for d in defines] + extra
    hdr_mtime = max(p.stat().st_mtime for p in _headers())
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = obj / (s.stem + ".o")
        objs.append(o)
        if force or not o.exists() or o.stat().st_mtime < max(s.stat().st_mtime, hdr_mtime):
            cmd = [NVCC, *flags, "-c", str(s), "-o", str(o)]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd)
    if force or not lib.exists() or lib.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        tmp = lib.with_suffix(f".{os.getpid()}.tmp")
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp), *map(str, objs),
               "-Xcompiler", "-fPIC"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
