#!/usr/bin/env python3
"""FMA (CUDA-core fp32) vs tcgen05 (split-fp16) half-step A/B over d (N2: the north
star's "ncu counters must back this choice").

    python tools/dsweep.py [--n 65536] [--ds 3,8,16,32,64] [--passes 6]
    ncu --metrics <list> -k regex:"lse" python tools/dsweep.py --passes 1 --warm 0

Each (d, mode) runs dense LSE passes (FSK_WARM=0 FSK_SCREEN=0: every block scored,
the fair comparison with the FMA kernel, which never skips) on fsk::Rng Gaussian
clouds, eps = 0.1, timed with CUDA events on the launching stream. One JSON line
per case: ms per half-step, the score FLOP rate (2 n m d) and the exp rate (n m).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("FSK_WARM", "0")
os.environ.setdefault("FSK_SCREEN", "0")


def main():
    import numpy as np
    import torch

    import paper_2602_03067_b200 as fsk

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--ds", default="3,8,16,32,64")
    ap.add_argument("--passes", type=int, default=6)
    ap.add_argument("--warm", type=int, default=2)
    ap.add_argument("--modes", default="fma,tensor")
    args = ap.parse_args()
    n = m = args.n
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    for d in [int(x) for x in args.ds.split(",")]:
        z = fsk.rng_normal(1000, (n + m) * d)
        X, Y = z[: n * d].reshape(n, d), z[n * d:].reshape(m, d)
        a = np.full(n, 1.0 / n)
        for mode in args.modes.split(","):
            eng = fsk.Engine(0, X, a, Y, a, mode=mode)
            eng.set_eps(0.1)
            f = torch.empty(n, dtype=torch.float32, device="cuda")
            g = torch.empty(m, dtype=torch.float32, device="cuda")
            eng.bind(f.data_ptr(), g.data_ptr())
            eng.init_potentials(s.cuda_stream)
            for k in range(args.warm):
                eng.half_step(k % 2, 0, n, 0, s.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            for k in range(args.passes):
                eng.half_step(k % 2, 0, n, 0, s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.passes
            print(json.dumps({"d": d, "mode": mode, "path": eng.path, "n": n, "m": m,
                              "ms_per_half_step": ms,
                              "score_tflops": 2.0 * n * m * d / ms / 1e9,
                              "gexp_per_s": n * m / ms / 1e6}), flush=True)
            eng.close()


if __name__ == "__main__":
    main()
