#!/usr/bin/env python3
"""Per-half-step device times of one solve (init + K iterations) on a bench config,
with the tracked live fraction after each pass (diagnostics for the warm bounds).

    python tools/pass_profile.py [--config cfg3] [--iters 10] [--reps 2]
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> int:
    import torch

    import bench
    import paper_2602_03067_b200 as fsk

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    n, m, d, eps, _ = bench.CONFIGS[a.config]
    X, Y = bench.make_inputs(n, m, d)
    wa, wb = bench.uniform_weights(n), bench.uniform_weights(m)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    eng = fsk.Engine(0, X, wa, Y, wb, mode="tensor")
    eng.set_eps(eps)
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    g = torch.empty(m, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())
    for rep in range(a.reps):
        eng.init_potentials(sp)
        rows = []
        for it in range(a.iters):
            for side, rows_ in ((0, n), (1, m)):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                l0, b0 = eng.live_tiles(), eng.screened_blocks()
                c0 = eng.pass_counts()
                e0.record(stream)
                eng.half_step(side, 0, rows_, 0, sp)
                e1.record(stream)
                torch.cuda.synchronize()
                l1, b1 = eng.live_tiles(), eng.screened_blocks()
                c1 = eng.pass_counts()
                kind = [k for k in c1 if c1[k] != c0[k]]
                rows.append((it, side, e0.elapsed_time(e1), (l1 - l0) / max(1, b1 - b0),
                             eng.live_set_fraction(side), kind[0] if kind else "?"))
        G = torch.empty((n, d), dtype=torch.float32, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.grad(0, n, G.data_ptr(), sp)
        e1.record(stream)
        torch.cuda.synchronize()
        tot = sum(r[2] for r in rows)
        print(f"rep {rep}: half-steps {tot:.1f} ms, grad {e0.elapsed_time(e1):.1f} ms")
        for it, side, ms, lf, lset, kind in rows:
            print(f"  it {it:2d} side {side} {kind:8s} {ms:8.2f} ms  probe-live {lf:.3f}  "
                  f"live-set {lset:.3f}")
    eng.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
