#!/usr/bin/env python3
"""Bisect the opt-in HVP plan cache (FSK_PLAN_CACHE=1) against the streaming default
over shapes: relative Frobenius difference of the single-precision HVP."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_03067_b200 as fsk  # noqa: E402

for n, m, d, eps, K in [(700, 650, 100, 0.5, 30), (2048, 1900, 1024, 0.1, 50),
                        (2048, 2048, 1024, 0.1, 50), (2048, 1900, 128, 0.1, 50),
                        (2048, 1900, 1024, 0.1, 1), (2048, 1900, 1024, 0.5, 50)]:
    z = fsk.rng_normal(1000, (n + m) * d)
    X, Y = z[: n * d].reshape(n, d), z[n * d:].reshape(m, d)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    s = fsk.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=10, precision="single")
    A = np.random.default_rng(7).standard_normal((n, d))
    out = {}
    for flag in ("0", "1"):
        os.environ["FSK_PLAN_CACHE"] = flag
        out[flag], info = fsk.hvp_apply(X, a, Y, b, s["f_hat"], s["g_hat"], eps, A, tau=1e-5,
                                        cg_tol=1e-30, cg_max_iters=K, precision="single")
    os.environ.pop("FSK_PLAN_CACHE", None)
    rel = np.linalg.norm(out["1"] - out["0"]) / np.linalg.norm(out["0"])
    print(f"n={n} m={m} d={d} eps={eps} K={K}: plan cache vs streaming rel {rel:.2e}", flush=True)
