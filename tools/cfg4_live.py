#!/usr/bin/env python3
"""Live fraction of the LSE passes at cfg4 (n = m = 1e5, d = 1024, eps = 0.1): the key
tiles each pass's epilogue could not skip (tile granularity, both orientations)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import bench
    import paper_2602_03067_b200 as fsk
    n, m, d, eps, iters = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
    X, Y = bench.make_inputs(n, m, d)
    a, b = bench.uniform_weights(n), bench.uniform_weights(m)
    eng = fsk.Engine(0, X, a, Y, b, mode="tensor")
    eng.set_eps(eps)
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    g = torch.empty(m, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())
    eng.init_potentials()
    for it in range(iters):
        eng.half_step(0, 0, n)
        eng.half_step(1, 0, m)
        torch.cuda.synchronize()
        print(f"it {it}: live tiles f-side {eng.live_set_fraction(0):.4f}  "
              f"g-side {eng.live_set_fraction(1):.4f}", flush=True)


if __name__ == "__main__":
    main()
