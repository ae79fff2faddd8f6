#!/usr/bin/env python3
"""Build recipe for oracle/_ref: the reference CPU library compiled from its own
sources where they lie under /root/reference/proj (never copied into the repo).

TEST INFRASTRUCTURE ONLY (checker + CPU baseline). Outputs go to oracle/_ref/
(git-ignored, travels to the GPU box with the snapshot).

As shipped the reference does not compile (SURVEY.md §0 finding 2). Two
documented, mechanical patches are applied to private copies written into
oracle/_ref/patched/ at build time:

  1. proj/include/fsk/mathutil.hpp:60-71 - `pairwise_sum` re-instantiates itself
     with a fresh lambda type at every recursion level (unbounded template
     recursion; cc1plus never finishes). Replaced by an offset-based recursion
     with the *same association order* (h = n/2 split, <=8 sequential leaf), so
     every sum is bit-identical to the intended one.
  2. proj/src/stream.cpp:117 and :166 - the score tile is written with row
     stride `bm` (actual tile width, stream.cpp:66 via :115/:164) but read back
     with the nominal width `bc`; ragged last tiles read garbage for rows >= 1
     (SURVEY.md §0 finding 3; 7/16 reference tests fail without it). Read stride
     changed to `bm`.

dense.cpp is not built (needs Eigen3, absent); the dense Hessian oracle is the
numpy restatement in oracle/dense.py.

Products:
  oracle/_ref/libfsk_ref_check.so   -std=c++20 -ffp-contract=off, x86-64-v3: the
      checker (strict IEEE evaluation order, so oracle/fsk_oracle.c can be
      compared with it bit for bit)
  oracle/_ref/libfsk_ref_fast_v3.so / _v4.so   the reference's own CMake
      flavour (-std=gnu++20 -O3, FMA contraction on) for x86-64-v3 / -v4
      (AVX-512): the CPU baseline that bench.py times
  oracle/_ref/test_core_ref, oracle/_ref/test_stream_ref - the reference's own
      doctest suites, unmodified, linked against the patched reference.
"""
from __future__ import annotations

import os
import re
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = Path(os.environ.get("FSK_REFERENCE_ROOT", "/root/reference")) / "proj"
OUT = HERE / "_ref"
PATCHED = OUT / "patched"

LIB_SOURCES = ["core.cpp", "schedule.cpp", "threads.cpp", "alloc_stats.cpp", "solver.cpp"]

FIXED_PAIRWISE = r"""template <typename T, typename F>
T pairwise_sum_at_(std::size_t off, std::size_t n, F& f) {
    // same association as the shipped recursion: <=8 sequential leaf, split at n/2
    if (n == 0) return T(0);
    if (n <= 8) {
        T s = f(off);
        for (std::size_t i = 1; i < n; ++i) s += f(off + i);
        return s;
    }
    std::size_t h = n / 2;
    return pairwise_sum_at_<T>(off, h, f) + pairwise_sum_at_<T>(off + h, n - h, f);
}

template <typename T, typename F>
T pairwise_sum(std::size_t n, F&& f) {
    return pairwise_sum_at_<T>(0, n, f);
}
"""


def patch_sources() -> None:
    (PATCHED / "fsk").mkdir(parents=True, exist_ok=True)
    src = (REF / "include/fsk/mathutil.hpp").read_text()
    # the (T, F&&) overload of pairwise_sum: from its template line to the
    # closing brace that follows `return pairwise_sum<T>(h, f) + ...;`
    pat = re.compile(
        r"template <typename T, typename F>\nT pairwise_sum\(std::size_t n, F&& f\) \{.*?"
        r"return pairwise_sum<T>\(h, f\) \+ pairwise_sum<T>\(n - h, g\);\n\}\n",
        re.S,
    )
    new, k = pat.subn(FIXED_PAIRWISE, src)
    if k != 1:
        raise RuntimeError("mathutil.hpp: pairwise_sum pattern not found (reference changed?)")
    (PATCHED / "fsk/mathutil.hpp").write_text(new)

    s = (REF / "src/stream.cpp").read_text()
    needle_a = "const T* srow = s.tile.data() + i * bc;"
    needle_b = "const double* srow = s.tile.data() + i * bc;"
    if s.count(needle_a) != 1 or s.count(needle_b) != 1:
        raise RuntimeError("stream.cpp: ragged-tile stride lines not found (reference changed?)")
    s = s.replace(needle_a, "const T* srow = s.tile.data() + i * bm;")
    s = s.replace(needle_b, "const double* srow = s.tile.data() + i * bm;")
    (PATCHED / "stream.cpp").write_text(s)


def run(cmd: list[str]) -> None:
    print("+", " ".join(str(c) for c in cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(jobs: int = 8) -> None:
    if not REF.exists():
        print(f"[build_ref] {REF} absent - keeping prebuilt oracle/_ref", flush=True)
        return
    cxx = shutil.which("g++")
    if cxx is None:
        raise RuntimeError("g++ not found")
    OUT.mkdir(parents=True, exist_ok=True)
    patch_sources()
    inc = ["-I", str(PATCHED), "-I", str(REF / "include")]
    srcs = [str(REF / "src" / f) for f in LIB_SOURCES] + [str(PATCHED / "stream.cpp")]
    strict = [cxx, "-std=c++20", "-ffp-contract=off", "-O3", "-fPIC", "-pthread", "-w"]
    fast = [cxx, "-std=gnu++20", "-O3", "-fPIC", "-pthread", "-w"]
    variants = (("check", strict, "x86-64-v3"), ("fast_v3", fast, "x86-64-v3"),
                ("fast_v4", fast, "x86-64-v4"))
    for tag, base, march in variants:
        objdir = OUT / f"obj_{tag}"
        objdir.mkdir(exist_ok=True)
        procs = []
        objs = []
        for s in srcs + [str(HERE / "ref_capi.cpp")]:
            o = objdir / (Path(s).stem + ".o")
            objs.append(str(o))
            procs.append(subprocess.Popen(base + [f"-march={march}", *inc, "-c", s, "-o", str(o)]))
        for p in procs:
            if p.wait() != 0:
                raise RuntimeError(f"compile failed ({tag})")
        run([cxx, "-shared", "-pthread", "-o", str(OUT / f"libfsk_ref_{tag}.so"), *objs])
    # the reference's own test suites, unmodified, against the patched reference
    objs_v3 = [str(OUT / "obj_check" / (Path(s).stem + ".o")) for s in srcs]
    for t in ("test_core", "test_stream"):
        run(strict + ["-march=x86-64-v3", "-DDOCTEST_CONFIG_IMPLEMENT_WITH_MAIN", "-include",
                    str(HERE / "doctest_shim/doctest.h"), "-I", str(HERE / "doctest_shim"), *inc,
                    str(REF / "tests" / f"{t}.cpp"), *objs_v3, "-o", str(OUT / f"{t}_ref")])
    # keep only binaries: no reference-derived source or object travels further
    shutil.rmtree(PATCHED, ignore_errors=True)
    for tag, _, _ in variants:
        shutil.rmtree(OUT / f"obj_{tag}", ignore_errors=True)


if __name__ == "__main__":
    build()
    sys.exit(0)
