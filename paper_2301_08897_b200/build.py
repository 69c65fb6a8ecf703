"""In-tree build of the sm_100a shared library (``libscadles_b200.so``).

Plain ``nvcc`` (no torch extension machinery): the library exposes only the C-ABI declared in
``include/scadles_b200.h`` and is loaded with ctypes, so the built ``.so`` travels to the GPU
box with the repo snapshot.  ``python -m paper_2301_08897_b200.build`` rebuilds it.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libscadles_b200.so"
SOURCES = ["capi.cu", "topk.cu", "topk_fused.cu", "aggregate.cu", "gather.cu"]
HEADERS = ["common.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _inputs() -> list[Path]:
    files = [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS]
    files.append(ROOT / "include" / "scadles_b200.h")
    return files


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(f.stat().st_mtime <= t for f in _inputs())


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every .cu for sm_100a and link the shared library in-tree.

    Safe to call from every rank of a torchrun job at once: the build holds an exclusive
    file lock (the first caller compiles, the others wait and then find the library up to
    date), objects go to a per-process directory, and the library is published with one
    atomic rename.
    """
    if not force and up_to_date():
        return LIB
    import fcntl

    (PKG / "build").mkdir(exist_ok=True)
    with open(PKG / "build" / ".lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        if not force and up_to_date():  # another process built it while we waited
            return LIB
        return _build_locked(verbose)


def build_variant(out: Path, extra: list[str]) -> Path:
    """A diagnostic build (e.g. ``-DSG_STAMPS``) linked to ``out``, leaving the product
    library untouched; load it by pointing ``_capi.LIB_PATH`` at ``out`` before the first call."""
    (PKG / "build").mkdir(exist_ok=True)
    return _build_locked(False, extra=extra, lib=Path(out))


def _build_locked(verbose: bool, extra: list[str] | None = None, lib: Path = LIB) -> Path:
    objdir = PKG / "build" / f"obj.{os.getpid()}"
    objdir.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        flags = os.environ.get("SG_NVCC_EXTRA", "").split() + list(extra or [])  # e.g. -DSG_PHASES (diagnostics)
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *flags, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        objs.append(str(obj))
    tmp = lib.with_suffix(f".so.tmp{os.getpid()}")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    shutil.rmtree(objdir, ignore_errors=True)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
