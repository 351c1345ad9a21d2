"""Build the sm_100a shared library (and, for tests, the CPU oracle).

The product is one C-ABI shared library, ``_lib/libqadc_b200.so``, compiled
in-tree with nvcc for ``-gencode arch=compute_100a,code=sm_100a`` (no JIT
cache, so the built file travels with the repo snapshot to the GPU box).
"""

from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libqadc_b200.so"
SOURCES = ["layout.cu", "lut.cu", "probe_tc.cu", "scan.cu", "select.cu", "simple.cu", "encode.cu",
           "peak.cu", "capi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
                     "-I" + str(ROOT / "include")] + os.environ.get("QADC_NVCC_EXTRA", "").split()


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the B200 library cannot be built")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    """Compile csrc/*.cu into _lib/libqadc_b200.so (incremental)."""
    nvcc = _nvcc()
    obj_dir = LIB_DIR / "obj"
    obj_dir.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "qadc_b200.h"]

    def compile_one(src: str) -> Path:
        s = CSRC / src
        o = obj_dir / (s.stem + ".o")
        if force or _stale(o, [s, *headers]):
            cmd = [nvcc, *NVCC_FLAGS, "-c", str(s), "-o", str(o)]
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
        return o

    with ThreadPoolExecutor(max_workers=min(6, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    if force or _stale(LIB, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB


def build_stock_reference(verbose: bool = False) -> None:
    """The UNMODIFIED reference package for the CPU baseline and the
    `--impl reference` arm: `pip install --no-index --no-build-isolation
    --no-deps --target baseline/_ref` of a scratch copy of
    /root/reference/pkg (its setup.py builds in the source tree, which is
    read-only). Only where the reference exists and the install is absent;
    baseline/_ref is git-ignored and travels to the GPU box."""
    import sys
    import tempfile
    src = Path("/root/reference/pkg")
    target = ROOT / "baseline" / "_ref"
    if not src.exists() or list(target.glob("qadc/_kernels*.so")):
        return
    with tempfile.TemporaryDirectory() as tmp:
        work = Path(tmp) / "pkg"
        shutil.copytree(src, work)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--target", str(target), "."]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, cwd=work, check=True, stdout=None if verbose else subprocess.DEVNULL)


def build_oracle(verbose: bool = False) -> None:
    """Test infrastructure: oracle/_build (restatement) and, when the
    reference sources are present, oracle/_ref (the reference's own C)."""
    oracle = ROOT / "oracle"
    subprocess.run(["make", "-s", "-C", str(oracle)], check=True)
    if Path("/root/reference/pkg/src/qadc/src/scan_kernels.c").exists():
        subprocess.run(["make", "-s", "-C", str(oracle), "ref"], check=True)


if __name__ == "__main__":
    build_library(verbose=True)
    build_oracle(verbose=True)
    build_stock_reference(verbose=True)
