#!/usr/bin/env python3
"""Phase times of one single-precision HVP at a bench config (FSK_TIMING=1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2602_03067_b200 as fsk  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
n, m, d, eps, iters = bench.CONFIGS[cfg]
X, Y = bench.make_inputs(n, m, d)
a, b = bench.uniform_weights(n), bench.uniform_weights(m)
out = fsk.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=iters, precision="single")
A = np.random.default_rng(7).standard_normal((n, d))
for rep in range(2):
    t0 = time.perf_counter()
    fsk.hvp_apply(X, a, Y, b, out["f_hat"], out["g_hat"], eps, A, tau=1e-5, cg_tol=1e-30,
                  cg_max_iters=50, precision="single")
    print(f"rep {rep}: {time.perf_counter() - t0:.3f} s", file=sys.stderr, flush=True)
