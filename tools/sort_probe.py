#!/usr/bin/env python3
"""Probe: does a locality order of the points (rows sorted by squared norm, or by a
random-projection tree) change the warm-bound live fractions and the cfg3 solve time?
    python tools/sort_probe.py [--config cfg3] [--orders none,norm,rptree]"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def rptree_order(P, leaf=128, seed=0):
    """Recursive median split along the top principal direction of each cell
    (power iteration), leaves of `leaf` rows: a locality order in any d."""
    rng = np.random.default_rng(seed)
    idx = np.arange(len(P))
    out = []
    stack = [idx]
    while stack:
        cur = stack.pop()
        if len(cur) <= leaf:
            out.append(cur)
            continue
        Q = P[cur] - P[cur].mean(0)
        v = rng.standard_normal(P.shape[1])
        for _ in range(3):
            v = Q.T @ (Q @ v)
            v /= np.linalg.norm(v)
        proj = Q @ v
        half = (len(cur) // 2 + leaf - 1) // leaf * leaf if len(cur) > 2 * leaf else len(cur) // 2
        part = np.argpartition(proj, half)
        stack.append(cur[part[half:]])
        stack.append(cur[part[:half]])
    return np.concatenate(out)


def main():
    import torch

    import bench
    import paper_2602_03067_b200 as fsk

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--orders", default="none,norm,rptree")
    a = ap.parse_args()
    n, m, d, eps, iters = bench.CONFIGS[a.config]
    X0, Y0 = bench.make_inputs(n, m, d)
    wa, wb = bench.uniform_weights(n), bench.uniform_weights(m)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    for order in a.orders.split(","):
        if order == "norm":
            px, py = np.argsort((X0 ** 2).sum(1)), np.argsort((Y0 ** 2).sum(1))
        elif order == "rptree":
            px, py = rptree_order(X0), rptree_order(Y0, seed=1)
        else:
            px, py = np.arange(n), np.arange(m)
        X, Y = np.ascontiguousarray(X0[px]), np.ascontiguousarray(Y0[py])
        eng = fsk.Engine(0, X, wa, Y, wb)
        eng.set_eps(eps)
        f = torch.empty(n, dtype=torch.float32, device="cuda")
        g = torch.empty(m, dtype=torch.float32, device="cuda")
        G = torch.empty((n, d), dtype=torch.float32, device="cuda")
        eng.bind(f.data_ptr(), g.data_ptr())
        for rep in range(2):
            eng.init_potentials(sp)
            l0, b0 = eng.live_tiles(), eng.screened_blocks()
            c0 = eng.pass_counts()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            for _ in range(iters):
                eng.half_step(0, 0, n, 0, sp)
                eng.half_step(1, 0, m, 0, sp)
            e1.record(stream)
            eng.grad(0, n, G.data_ptr(), sp)
            e2.record(stream)
            torch.cuda.synchronize()
            l1, b1 = eng.live_tiles(), eng.screened_blocks()
            c1 = eng.pass_counts()
            print(f"order={order:7s} rep {rep}: iterations {e0.elapsed_time(e1):8.1f} ms, grad "
                  f"{e1.elapsed_time(e2):6.1f} ms, live fraction {(l1 - l0) / max(1, b1 - b0):.4f}, "
                  f"passes { {k: c1[k] - c0[k] for k in c1} }", flush=True)
        # results in the original order agree across orders
        fo = np.empty(n)
        fo[px] = f.cpu().numpy()
        print(f"   f[0:3] in original order: {fo[:3]}", flush=True)
        eng.close()


if __name__ == "__main__":
    main()
