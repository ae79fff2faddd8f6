#!/usr/bin/env python3
"""Per-rank device time of the row-sharded cfg3 step, measured on ONE B200.

Only one GPU is reachable here, so the N-GPU run of `bench.py --gpus N` cannot be
timed directly. This tool measures what each rank's GPU would execute in it: a
full-problem engine runs the exact bench step once and records the potential
vector after every half-step (what the in-place all-gather leaves in every
rank's buffer); then, for every rank r of every world size N, a second engine
runs rank r's shard of every half-step (rows `ShardPlan(r, N).f_bounds[r]` /
`g_bounds[r]`, the same calls `paper_2602_03067_b200.sharded` makes) with the
recorded full vector copied in after each half-step in place of the all-gather,
and then its rows of the gradient. Each rank's half-steps and gradient are timed
with CUDA events on the launching stream; the copies standing in for the
all-gathers are outside the timed intervals. The shard rows are compared with the
full run (max |difference| reported).

projected step(N) = max over ranks (sum of the rank's half-step and gradient times)
                    + 20 x the all-gather of a 4 MB fp32 potential vector (stated
                    as an assumption, `--gather-us`, not measured here).

    python tools/shard_projection.py [--worlds 1 2 4 8] [--gather-us 25] [--json out]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> int:
    import torch

    import bench
    import paper_2602_03067_b200 as fsk
    from paper_2602_03067_b200.sharded import ShardPlan

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--worlds", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--gather-us", type=float, default=25.0)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--json")
    args = ap.parse_args()

    n, m, d, eps, iters = bench.CONFIGS[args.config]
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    X, Y = bench.make_inputs(n, m, d)
    a, b = bench.uniform_weights(n), bench.uniform_weights(m)

    # the full run: the potential vector after every half-step
    full = fsk.Engine(0, X, a, Y, b)
    full.set_eps(eps)
    F = torch.zeros(n, dtype=torch.float32, device="cuda")
    G = torch.zeros(m, dtype=torch.float32, device="cuda")
    full.bind(F.data_ptr(), G.data_ptr())
    full.init_potentials(sptr)
    f_trace, g_trace = [], []
    for _ in range(iters):
        full.half_step(0, 0, n, 0, sptr)
        f_trace.append(F.clone())
        full.half_step(1, 0, m, 0, sptr)
        g_trace.append(G.clone())
    grad_full = torch.empty((n, d), dtype=torch.float32, device="cuda")
    full.grad(0, n, grad_full.data_ptr(), sptr)
    torch.cuda.synchronize()
    del full

    eng = fsk.Engine(0, X, a, Y, b)
    eng.set_eps(eps)
    f = torch.zeros(n, dtype=torch.float32, device="cuda")
    g = torch.zeros(m, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())

    def rank_step(plan, r, timed):
        flo, fhi = plan.f_bounds[r]
        glo, ghi = plan.g_bounds[r]
        ev = []

        def mark():
            if timed:
                ev.append(torch.cuda.Event(enable_timing=True))
                ev[-1].record(stream)

        eng.init_potentials(sptr)
        keep = []   # shard rows after each half-step, compared after the step (no syncs)
        for k in range(iters):
            mark()
            eng.half_step(0, flo, fhi, 0, sptr)
            mark()
            if timed:
                keep.append((f[flo:fhi].clone(), f_trace[k][flo:fhi]))
            f.copy_(f_trace[k])                       # the all-gather's result
            mark()
            eng.half_step(1, glo, ghi, 0, sptr)
            mark()
            if timed:
                keep.append((g[glo:ghi].clone(), g_trace[k][glo:ghi]))
            g.copy_(g_trace[k])
        out = torch.empty((max(fhi - flo, 1), d), dtype=torch.float32, device="cuda")
        mark()
        eng.grad(flo, fhi, out.data_ptr(), sptr)
        mark()
        torch.cuda.synchronize()
        if not timed:
            return None
        diff = max((float((u - w).abs().max()) for u, w in keep if u.numel()), default=0.0)
        gdiff = float((out[:fhi - flo] - grad_full[flo:fhi]).abs().max()) if fhi > flo else 0.0
        t = [ev[i].elapsed_time(ev[i + 1]) for i in range(0, len(ev), 2)]
        return {"half_ms": sum(t[:-1]), "grad_ms": t[-1], "step_ms": sum(t),
                "max_abs_diff_potentials": diff, "max_abs_diff_grad": gdiff,
                "rows": [flo, fhi]}

    res = {"config": args.config, "n": n, "m": m, "d": d, "iters": iters,
           "gather_us_assumed": args.gather_us, "worlds": {}}
    for N in args.worlds:
        ranks = []
        for r in range(N):
            plan = ShardPlan(r, N, n, m)
            for _ in range(args.warmup):
                rank_step(plan, r, False)
            ranks.append(rank_step(plan, r, True))
        worst = max(x["step_ms"] for x in ranks)
        proj = worst + 2 * iters * args.gather_us / 1e3
        res["worlds"][N] = {"ranks": ranks, "max_rank_step_ms": worst,
                            "projected_step_ms": proj,
                            "projected_it_s": iters / (proj / 1e3),
                            "max_abs_diff": max(max(x["max_abs_diff_potentials"],
                                                    x["max_abs_diff_grad"]) for x in ranks)}
        print(f"N={N}: max rank step {worst:.1f} ms, projected {iters / (proj / 1e3):.2f} it/s, "
              f"per-rank {[round(x['step_ms'], 1) for x in ranks]}, max |shard - full| "
              f"{res['worlds'][N]['max_abs_diff']:.2e}", flush=True)
    base = res["worlds"].get(1, {}).get("projected_it_s")
    if base:
        for N, w in res["worlds"].items():
            w["projected_speedup"] = w["projected_it_s"] / base
    if args.json:
        Path(args.json).write_text(json.dumps(res, indent=1))
    return 0


if __name__ == "__main__":
    sys.exit(main())
