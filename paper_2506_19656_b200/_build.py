"""Build the sm_100a CUDA library ``lib/libcvb200.so`` in-tree with nvcc.

Every ``csrc/*.cu`` file is compiled in parallel (``-gencode
arch=compute_100a,code=sm_100a -lineinfo``, no fast-math: the quantiser must
reproduce IEEE float64 rounding) and linked into one shared library with a
static CUDA runtime, so the ``.so`` travels with the repository snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = ROOT / "build" / "cvb200"
LIB = PKG / "lib" / "libcvb200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC,-O2",
    "--expt-relaxed-constexpr",
    "-Wno-deprecated-gpu-targets",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found (set NVCC or install the CUDA toolkit)")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _deps() -> list[Path]:
    return sources() + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _deps())


def _compile(nvcc: str, src: Path, extra: list[str], build_dir: Path = BUILD) -> Path:
    obj = build_dir / (src.stem + ".o")
    cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, f"-I{INCLUDE}", f"-I{CSRC}", "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False, extra_flags: list[str] | None = None,
          out: Path | None = None) -> Path:
    """Compile the library if any source is newer than it; return its path.

    ``extra_flags`` / ``out`` build an experimental variant next to the
    default library (e.g. a different launch-bounds setting for A/B runs).
    """
    lib = Path(out) if out else LIB
    if not force and out is None and up_to_date():
        return LIB
    nvcc = _nvcc()
    build_dir = BUILD if out is None else BUILD.parent / ("cvb200_" + lib.stem)
    build_dir.mkdir(parents=True, exist_ok=True)
    lib.parent.mkdir(parents=True, exist_ok=True)
    extra = list(extra_flags or [])
    srcs = sources()
    # compile the heaviest translation units first
    srcs.sort(key=lambda p: -p.stat().st_size)
    workers = max(1, min(len(srcs), os.cpu_count() or 4))
    with cf.ThreadPoolExecutor(workers) as ex:
        objs = list(ex.map(lambda s: _compile(nvcc, s, extra, build_dir), srcs))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, lib)
    if verbose:
        print(f"built {lib}", file=sys.stderr)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    flags = []
    for a in args:
        if a.startswith("--out="):
            out = Path(a.split("=", 1)[1])
        elif a.startswith("-D"):
            flags.append(a)
    build(force="--force" in args or out is not None, verbose=True, extra_flags=flags, out=out)
