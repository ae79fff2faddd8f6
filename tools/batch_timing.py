#!/usr/bin/env python3
"""Wall time of fsk_sinkhorn_divergence_batch on cfg5-sized clouds (diagnostics).

    FSK_TIMING=1 python tools/batch_timing.py [pairs]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2602_03067_b200 as fsk  # noqa: E402

npairs = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rng = np.random.default_rng(5)
clouds = [rng.normal(size=(10000, 784)) for _ in range(4)]
w = np.full(10000, 1e-4)
pairs = [(clouds[i % 4], w, clouds[(i + 1) % 4], w) for i in range(npairs)]
for rep in range(3):
    t0 = time.perf_counter()
    fsk.sinkhorn_divergence_batch(pairs, eps=0.1, max_iters=10, precision="single")
    dt = time.perf_counter() - t0
    print(f"rep {rep}: {dt * 1e3:.1f} ms for {npairs} pairs = {dt * 1e3 / (3 * npairs):.2f} ms/solve",
          file=sys.stderr, flush=True)
