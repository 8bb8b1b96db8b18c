"""Builds libbbsi_cuda.so (sm_100a) in-tree with nvcc. No torch, no JIT cache."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libbbsi_cuda.so"
SOURCES = ["zgemm.cu", "zgemm_tma.cu", "zinv.cu", "band_ops.cu", "rgf.cu", "ddrgf.cu", "ddrgf_iface.cu", "prof.cu", "multi.cu", "capi.cu"]
HEADERS = ["zcommon.cuh", "internal.h", "dyson_gen.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2"]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "bbsi_cuda.h"]
    return any(p.exists() and p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, extra: tuple = (), out: Path | None = None) -> Path:
    """extra/out: instrumented variants (e.g. -DBBSI_ZINV_DEBUG into _lib/libbbsi_cuda_dbg.so,
    loaded with BBSI_LIB=...); the default call builds the product library."""
    srcs = [s for s in SOURCES if (CSRC / s).exists()]
    lib = Path(out) if out else LIB
    if out is None and not force and not _stale():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    objs = []
    for s in srcs:
        obj = LIB_DIR / (Path(s).stem + lib.stem + ".o")
        cmd = [NVCC, *FLAGS, *extra, "-c", str(CSRC / s), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True, cwd=CSRC)
        objs.append(str(obj))
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", str(lib), "-cudart", "static", "-ldl"]
    subprocess.run(cmd, check=True, cwd=CSRC)
    for o in objs:
        Path(o).unlink(missing_ok=True)
    return lib


if __name__ == "__main__":
    if "--debug-zinv" in sys.argv:
        print(build(verbose=True, extra=("-DBBSI_ZINV_DEBUG",), out=LIB_DIR / "libbbsi_cuda_dbg.so"))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
