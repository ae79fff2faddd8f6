"""Build recipe for libfsk_b200.so (in-tree, sm_100a only).

    python -m paper_2602_03067_b200.build        # or __graft_entry__.build()

Every source under csrc/ is compiled with nvcc for
-gencode arch=compute_100a,code=sm_100a (-lineinfo for Nsight source mapping)
into paper_2602_03067_b200/_build/libfsk_b200.so. The .so carries the C ABI
(include/fsk_b200.h) and the C++ drop-in API (include/fsk/*.hpp). It travels to
the GPU box inside the repo snapshot; nothing is installed into site-packages.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "_build"
OBJ = OUT / "obj"
LIB = OUT / "libfsk_b200.so"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++20", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=default",
          "--expt-relaxed-constexpr", "-I", str(ROOT / "include"), "-I", str(CSRC),
          *os.environ.get("FSK_NVCC_EXTRA", "").split()]


def sources() -> list[Path]:
    return sorted([*CSRC.glob("*.cu"), *CSRC.glob("*.cpp"), *CSRC.glob("api/*.cpp")])


def _compile(src: Path) -> Path:
    rel = src.relative_to(CSRC)
    obj = OBJ / (str(rel).replace("/", "_") + ".o")
    deps = [src, *CSRC.glob("*.h"), *CSRC.glob("api/*.h"), *(ROOT / "include").rglob("*.h*")]
    cmd = [NVCC, *ARCH, *COMMON, "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cu":
        cmd += ["-Xptxas", "-v"] if os.environ.get("FSK_PTXAS_VERBOSE") else []
    # the full command line (FSK_NVCC_EXTRA flags change numerics / add traps) is
    # part of the object's identity, not just the source mtimes
    stamp = obj.with_suffix(".cmd")
    digest = hashlib.sha256("\0".join(cmd).encode()).hexdigest()
    if (obj.exists() and stamp.exists() and stamp.read_text() == digest
            and obj.stat().st_mtime >= max(p.stat().st_mtime for p in deps)):
        return obj
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed on {src}")
    stamp.write_text(digest)
    if r.stderr.strip() and os.environ.get("FSK_PTXAS_VERBOSE"):
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(_compile, srcs))
    if not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs),
               "-lcuda"]
        subprocess.run(cmd, check=True)
    if verbose:
        print(f"[build] {LIB}")
    return LIB


if __name__ == "__main__":
    build(verbose=True)
