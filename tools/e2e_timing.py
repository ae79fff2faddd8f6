"""Repeated end-to-end calls through the C ABI (host buffers) with per-call wall time
and free device memory after each call. FSK_TIMING=1 adds the library's phase marks.
    python tools/e2e_timing.py [cfg3] ; env REPS (default 2), PIN (default 1)"""
import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import bench, paper_2602_03067_b200 as fsk
n, m, d, eps, iters = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
X, Y = bench.make_inputs(n, m, d)
a, b = bench.uniform_weights(n), bench.uniform_weights(m)
if os.environ.get("PIN", "1") == "1":   # as bench.py's e2e arm: page-locked inputs
    X, Y, a, b = (fsk.pinned_copy(v) for v in (X, Y, a, b))
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None


def free_gb():
    if rt is None:
        return float("nan")
    f, t = ctypes.c_size_t(), ctypes.c_size_t()
    rt.cudaMemGetInfo(ctypes.byref(f), ctypes.byref(t))
    return f.value / 1e9


for rep in range(int(os.environ.get("REPS", "2"))):
    t0 = time.perf_counter()
    out = fsk.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=iters, precision="single", grad=True)
    print(f"rep {rep}: {time.perf_counter() - t0:.3f} s  free {free_gb():.1f} GB", file=sys.stderr,
          flush=True)
