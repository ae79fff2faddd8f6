"""Compile the reference's own doctest suites against the B200 library.

The unmodified reference test sources (/root/reference/proj/tests/test_core.cpp
and test_stream.cpp) are compiled here, in the build container, against the
drop-in headers in include/fsk/ and linked to libfsk_b200.so. The binaries
(tests/refsuite/_bin/, git-ignored) travel to the GPU box inside the snapshot;
tests/test_refsuite_gpu.py runs them there. Nothing reads /root/reference at
run time. The doctest stand-in is oracle/doctest_shim/doctest.h.
"""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
REF_TESTS = Path(os.environ.get("FSK_REFERENCE_ROOT", "/root/reference")) / "proj" / "tests"
BIN = Path(__file__).resolve().parent / "_bin"
LIBDIR = ROOT / "paper_2602_03067_b200" / "_build"


def build() -> list[Path]:
    if not REF_TESTS.exists():
        print(f"[refsuite] {REF_TESTS} absent - keeping prebuilt binaries")
        return sorted(BIN.glob("*"))
    BIN.mkdir(exist_ok=True)
    out = []
    for t in ("test_core", "test_stream"):
        exe = BIN / f"{t}_b200"
        src = REF_TESTS / f"{t}.cpp"
        if exe.exists() and exe.stat().st_mtime >= max(src.stat().st_mtime,
                                                       (LIBDIR / "libfsk_b200.so").stat().st_mtime):
            out.append(exe)
            continue
        subprocess.run(
            ["g++", "-std=c++20", "-O2", "-w", "-DDOCTEST_CONFIG_IMPLEMENT_WITH_MAIN",
             "-I", str(ROOT / "oracle" / "doctest_shim"), "-I", str(ROOT / "include"), str(src),
             "-L", str(LIBDIR), "-lfsk_b200", f"-Wl,-rpath,$ORIGIN/../../../paper_2602_03067_b200/_build",
             "-o", str(exe)],
            check=True,
        )
        out.append(exe)
    return out


if __name__ == "__main__":
    for p in build():
        print(p)
