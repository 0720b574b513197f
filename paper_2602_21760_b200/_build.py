"""Build the C-ABI extension (libhybridpar_b200.so) in-tree with nvcc.

Every ``csrc/*.cu`` file is compiled for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a``) with ``-lineinfo`` so ncu's
source page maps back to the kernels, then linked into one shared library
under ``paper_2602_21760_b200/lib/``. The build is incremental (object files
are rebuilt when their source, a header, or this script changes) and runs the
nvcc invocations in parallel. Works without a GPU (nvcc cross-compiles).
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIBDIR = PKG / "lib"
OBJDIR = ROOT / "build" / "obj"
LIBNAME = "libhybridpar_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "--expt-relaxed-constexpr", "-DNDEBUG"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA extension cannot be built")


def _header_digest() -> str:
    h = hashlib.sha256()
    for d in (CSRC, INCLUDE):
        for p in sorted(d.glob("*.h*")):
            h.update(p.name.encode())
            h.update(p.read_bytes())
    h.update(Path(__file__).read_bytes())
    return h.hexdigest()[:16]


def _compile(src: Path, digest: str) -> Path:
    obj = OBJDIR / f"{src.stem}.{digest}.o"
    if obj.exists() and obj.stat().st_mtime >= src.stat().st_mtime:
        return obj
    cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, f"-I{INCLUDE}", f"-I{CSRC}", "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
    return obj


def library_path() -> Path:
    return LIBDIR / LIBNAME


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    """Compile every csrc/*.cu for sm_100a and link the shared library."""
    OBJDIR.mkdir(parents=True, exist_ok=True)
    LIBDIR.mkdir(parents=True, exist_ok=True)
    digest = _header_digest()
    sources = sorted(CSRC.glob("*.cu"))
    if not sources:
        raise RuntimeError(f"no CUDA sources under {CSRC}")
    jobs = jobs or min(len(sources), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, digest), sources))
    lib = library_path()
    newest = max(o.stat().st_mtime for o in objs)
    if not lib.exists() or lib.stat().st_mtime < newest:
        tmp = lib.with_suffix(".so.tmp")
        cmd = [_nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcuda"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
        os.replace(tmp, lib)
    # drop stale objects from previous header digests
    for o in OBJDIR.glob("*.o"):
        if o not in objs:
            try:
                o.unlink()
            except OSError:
                pass
    if verbose:
        print(f"built {lib} from {len(sources)} sources")
    return lib


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
