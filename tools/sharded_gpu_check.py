#!/usr/bin/env python3
"""Multi-rank check of the sharded driver with the real B200 engine.

Only one GPU is reachable from this environment, and NCCL refuses two ranks on
one device, so the ranks share cuda:0 and exchange the potentials over gloo
(CUDA tensors). Everything else is the production path: one fsk.Engine per
rank, row shards of f and g, in-place all-gathers after every half-step, the
lagged marginal violation, gradient rows per rank. The result is compared with
a single-engine run of the same problem.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/sharded_gpu_check.py
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> int:
    import torch
    import torch.distributed as dist

    import paper_2602_03067_b200 as fsk
    from paper_2602_03067_b200.sharded import ShardPlan, ShardedSinkhorn

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    n, m, d, eps, iters = 6000, 5000, 64, 0.1, 6
    if len(sys.argv) > 1:   # e.g. 65536 65536 64 0.05 10 (exercises the warm-bound passes)
        n, m, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
        eps, iters = float(sys.argv[4]), int(sys.argv[5])
    rng = np.random.default_rng(3)
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d)) * 0.9 + 0.1
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    dev = torch.device("cuda", 0)

    eng = fsk.Engine(0, X, a, Y, b, mode="tensor")
    eng.set_eps(eps)
    plan = ShardPlan(rank, world, n, m)
    solver = ShardedSinkhorn(eng, plan, dev, dist)
    solver.init()
    viol = solver.iterate(iters, track_violation=True)
    lo, hi = plan.f_bounds[rank]
    G = torch.empty((max(hi - lo, 1), d), dtype=torch.float32, device=dev)
    solver.grad_shard(G)
    torch.cuda.synchronize()
    f_sh, g_sh = solver.f[:n].cpu().numpy(), solver.g[:m].cpu().numpy()
    parts = [None] * world
    dist.all_gather_object(parts, (lo, hi, G[: hi - lo].cpu().numpy()))

    ok = True
    if rank == 0:
        ref = fsk.Engine(0, X, a, Y, b, mode="tensor")
        ref.set_eps(eps)
        f = torch.empty(n, dtype=torch.float32, device=dev)
        g = torch.empty(m, dtype=torch.float32, device=dev)
        ref.bind(f.data_ptr(), g.data_ptr())
        ref.init_potentials()
        for _ in range(iters):
            ref.half_step(0, 0, n)
            ref.half_step(1, 0, m)
        v = torch.zeros(1, dtype=torch.float64, device=dev)
        f_save = f.clone()
        ref.half_step(0, 0, n, v.data_ptr())
        f.copy_(f_save)
        Gr = torch.empty((n, d), dtype=torch.float32, device=dev)
        ref.grad(0, n, Gr.data_ptr())
        torch.cuda.synchronize()
        Gs = np.zeros((n, d), dtype=np.float32)
        for plo, phi, part in parts:
            Gs[plo:phi] = part
        df = np.abs(f_sh - f.cpu().numpy()).max() / max(1.0, np.abs(f.cpu().numpy()).max())
        dg = np.abs(g_sh - g.cpu().numpy()).max() / max(1.0, np.abs(g.cpu().numpy()).max())
        dG = np.abs(Gs - Gr.cpu().numpy()).max() / np.abs(Gr.cpu().numpy()).max()
        dv = abs(viol - v.item()) / max(1e-30, abs(v.item()))
        print(f"[sharded x{world}] f {df:.2e} g {dg:.2e} grad {dG:.2e} viol {dv:.2e}", flush=True)
        # row shards run the same kernels on the same rows: identical up to the
        # order of the per-split partial sums
        # warm-bound passes seed each row's running max per shard and pair query tiles
        # into different units: agreement to fp32 rounding (cf. the warm-vs-cold test)
        ok = df <= 1e-6 and dg <= 1e-6 and dG <= 2e-4 and dv <= 1e-5
        print("[sharded] OK" if ok else "[sharded] MISMATCH", flush=True)
        ref.close()
    eng.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
