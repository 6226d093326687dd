"""In-tree build of libhsrnn.so (nvcc, sm_100a only).

The library is built next to the sources (``paper_2307_11339_b200/_lib``) so
that it travels with the repository snapshot to the GPU host; nothing is
installed into site-packages and no JIT cache is used.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIBNAME = "libhsrnn.so"
INCLUDE = PKG.parent / "include"

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler", "-fPIC",
    "-shared",
    "-cudart", "shared",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libhsrnn.so")


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def library_path() -> Path:
    return LIBDIR / LIBNAME


def needs_build() -> bool:
    lib = library_path()
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    return any(src.stat().st_mtime > t for src in _sources())


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines: tuple = ()) -> Path:
    """Compile ``csrc/hs_rnn.cu`` (which includes every kernel header) into
    ``_lib/libhsrnn.so`` (or ``out``, with extra ``-D`` defines: variant builds
    for experiments, loaded through ``HS_LIB_PATH``).  Returns the library path."""
    lib = Path(out) if out else library_path()
    if not force and not needs_build():
        return lib
    LIBDIR.mkdir(parents=True, exist_ok=True)
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc_path(), *ARCH_FLAGS, *NVCC_FLAGS, *(f"-D{d}" for d in defines), "-I", str(INCLUDE), "-o", str(tmp),
           str(CSRC / "hs_rnn.cu")]
    if verbose:
        cmd += ["-Xptxas", "-v"]
        print(" ".join(cmd))
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{proc.stdout}\n{proc.stderr}")
    if verbose and proc.stderr:
        print(proc.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import sys

    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
