"""In-tree builds: the sm_100a library (the product) and the CPU checkers.

    python -m paper_1610_07159_b200.build          # both
    python -m paper_1610_07159_b200.build cuda

The .so files are git-ignored but travel to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
# HWF_CUDA_LIB: run the test suite against an A/B variant build (lib/variants/<name>/libhwflow_cuda.so)
CUDA_LIB = Path(os.environ["HWF_CUDA_LIB"]) if os.environ.get("HWF_CUDA_LIB") else LIBDIR / "libhwflow_cuda.so"
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "_build" / "libhwflow_oracle.so"
REF_LIB = ORACLE_DIR / "_ref" / "libhwflow_ref.so"

SOURCES = ["pixel.cu", "solve.cu", "maps.cu", "capi.cu", "stages.cu", "geometry.cu", "split.cu"]
NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    f"-I{ROOT / 'include'}", f"-I{CSRC}",
]


def _nvcc() -> str:
    for cand in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand == "nvcc" or Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_cuda(force: bool = False, verbose: bool = False, defines: tuple[str, ...] = (),
               variant: str | None = None) -> Path:
    """The product library; with `defines` (e.g. ("HWF_PIX_MINB=3",)) an A/B variant built to
    lib/variants/<variant>/libhwflow_cuda.so (tools/ab.py)."""
    objdir = LIBDIR / "obj" if variant is None else LIBDIR / "variants" / variant / "obj"
    out = LIBDIR / "libhwflow_cuda.so" if variant is None else LIBDIR / "variants" / variant / "libhwflow_cuda.so"
    objdir.mkdir(parents=True, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list((ROOT / "include").glob("*.h"))
    nvcc = _nvcc()

    def compile_one(src: str) -> Path:
        obj = objdir / (Path(src).stem + ".o")
        if force or _stale(obj, [CSRC / src] + headers):
            cmd = [nvcc, *NVCC_FLAGS, *dflags, "-c", str(CSRC / src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    if force or _stale(out, objs):
        cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(out), *map(str, objs)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return out


def build_oracle() -> None:
    """The CPU checker (test infrastructure only) and, where /root/reference exists, oracle/_ref."""
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "all"], check=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["cuda", "oracle"]
    if "cuda" in what:
        print(build_cuda(verbose=True))
    if "oracle" in what:
        build_oracle()
