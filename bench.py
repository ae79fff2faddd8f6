#!/usr/bin/env python3
"""FlashSinkhorn B200 benchmark (BASELINE.json metric).

Metric: Sinkhorn iterations/s at n = m = 2^20 (the "1M" config, SURVEY §0
finding 4), d = 64, eps = 0.05 on 1-8 B200, one step = 10 alternating
iterations + the gradient w.r.t. X (the fwd+grad unit of cfg3). Inputs are
synthetic Gaussian clouds from fsk::Rng(1000) (X then Y), uniform weights,
fp32 on device (the reference's Single-precision path), larger than L2.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Arms
  default            the B200 engine: device-resident clouds + tcgen05 split-fp16
                     half-steps, rows sharded over ranks, NCCL all-gather of the
                     potentials after each half-step (paper_2602_03067_b200.sharded)
  --impl reference   the reference's own CPU solver (oracle/_ref, compiled from
                     /root/reference sources) timed on this host's cores on a
                     bounded row/column slice of the same workload, extrapolated
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (n, m, d, eps, iterations per step); BASELINE.json configs[0..4]
    "cfg3": (1 << 20, 1 << 20, 64, 0.05, 10),
    "cfg2": (65536, 65536, 64, 0.05, 10),
    "cfg1": (4096, 4096, 3, 0.1, 100),
    "cfg4": (100000, 100000, 1024, 0.1, 10),
    "cfg5": (10000, 10000, 784, 0.1, 10),
}
# what a step adds after the iterations: the gradient w.r.t. X (cfg1-3), one
# Hessian-vector product (cfg4: K_CG = 50 fixed, tau = 1e-5, PAPER.md:1614-1616,
# single-precision engine), and for cfg5 a step is the whole batch of 64
# debiased divergences (3 solves per pair)
STEP_TAIL = {"cfg1": "grad", "cfg2": "grad", "cfg3": "grad", "cfg4": "hvp", "cfg5": "divergence"}
HVP_CG_ITERS = 50
CFG5_PAIRS = 64


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, indices):
        self.indices = set(indices)
        self.rows = []
        self.proc = None

    def start(self, wait_first=True):
        """Starts sampling every 200 ms; waits (<= 3 s) for the first sample so that a
        short timed region still sees one."""
        self._start()
        if wait_first and self.proc is not None:
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:
                time.sleep(0.01)
        self.n0 = len(self.rows)

    def _start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return None
        # a region shorter than the sampling period: take the next sample as well
        t0 = time.time()
        while len(self.rows) <= getattr(self, "n0", 0) and time.time() - t0 < 1.0:
            time.sleep(0.01)
        self.rows = self.rows[max(0, getattr(self, "n0", 0) - 1):]
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = [r for r in self.rows if r[0].isdigit() and int(r[0]) in self.indices]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for name, val in zip(names, r[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ---------------------------------------------------------------- inputs ------

def uniform_weights(n):
    """1/n weights whose naive running sum passes the reference's |sum - 1| <= 1e-12
    check (core.cpp:27-33): plain 1/n fails at n = 1e5 (SURVEY §0 finding 4), so
    the last weight absorbs the sequential-sum residual."""
    w = np.full(n, 1.0 / n)
    w[-1] = 1.0 - np.cumsum(w[:-1])[-1] if n > 1 else 1.0
    return w


def make_inputs(n, m, d, seed=1000):
    """fsk::Rng(seed).normal(): X (n x d) then Y (m x d), row-major."""
    import paper_2602_03067_b200 as fsk
    z = fsk.rng_normal(seed, (n + m) * d)
    return z[: n * d].reshape(n, d), z[n * d:].reshape(m, d)


# ------------------------------------------------------------ reference arm --

_REF_INPUTS = {}


def _reference_inputs(n, m, d):
    key = (n, m, d)
    if key not in _REF_INPUTS:
        from oracle import rng_normal
        z = rng_normal(1000, (n + m) * d)  # the same fsk::Rng(1000) stream as the GPU arm
        X64, Y64 = z[: n * d].reshape(n, d), z[n * d:].reshape(m, d)
        _REF_INPUTS[key] = (X64, Y64, X64.astype(np.float32), Y64.astype(np.float32))
    return _REF_INPUTS[key]


def reference_sample(cfgname, threads=None):
    """Times the reference's own CPU path on a bounded slice of the workload and
    extrapolates to one full step.

    * f half-step: update_f_hat_f32 (stream.cpp:437-443) for 64*T source rows
      (one row block per worker thread) against all m targets; rows are
      independent given g, so time scales by n / rows (a sliced call is
      bit-identical to the same rows of a full call).
    * g half-step: update_g_hat_f32 (stream.cpp:445-451) for 64*T target rows
      against all n sources, scaled by m / rows.
    * gradient (cfg1-3): the SPEC composition (the reference ships no gradient
      code): one f64 LSE pass for r (update_f_hat, 64*T rows x m) plus
      apply_plan(Y) (stream.cpp:324-339, double only) on 64*T rows x 4096
      targets, scaled by (n / rows) and (n / rows)(m / 4096).
    * cfg5: a step is 64 pairs x 3 solves x iters alternating iterations.
    Times include the wrapper's copy of the inputs into fsk types (< 10%).
    """
    from oracle import Oracle

    n, m, d, eps, iters = CONFIGS[cfgname]
    tail = STEP_TAIL[cfgname]
    ref = Oracle("ref_fast")
    if threads:
        ref.set_num_threads(threads)
    T = ref.num_threads()
    rows = min(64 * T, n, m)
    cols_apply = min(4096, m)
    X64, Y64, Xf, Yf = _reference_inputs(n, m, d)
    a = np.full(n, 1.0 / n, dtype=np.float32)
    b = np.full(m, 1.0 / m, dtype=np.float32)
    g0 = -(Y64 ** 2).sum(1)
    f0 = -(X64 ** 2).sum(1)
    t0 = time.perf_counter()
    ref.update_f_hat_f32(Xf[:rows], a[:rows], Yf, b, g0.astype(np.float32), eps)
    t_f = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref.update_g_hat_f32(Xf, a, Yf[:rows], b[:rows], f0.astype(np.float32), eps)
    t_g = time.perf_counter() - t0
    iter_s = t_f * n / rows + t_g * m / rows
    grad_s = 0.0
    sample = (f"f32 half-steps on {rows} rows x all {m} (resp. {n}) columns, {T} threads")
    if tail == "grad":
        a64 = np.full(rows, 1.0 / rows)
        t0 = time.perf_counter()
        ref.update_f_hat(X64[:rows], a64, Y64, uniform_weights(m), g0, eps)
        t_lse64 = time.perf_counter() - t0
        Ysub = Y64[:cols_apply]
        bsub = np.full(cols_apply, 1.0 / cols_apply)
        gsub = -(Ysub ** 2).sum(1)
        fsub = ref.update_f_hat(X64[:rows], a64, Ysub, bsub, gsub, eps)
        t0 = time.perf_counter()
        ref.apply_plan(X64[:rows], a64, Ysub, bsub, fsub, gsub, eps, Ysub)
        t_apply = time.perf_counter() - t0
        grad_s = t_lse64 * n / rows + t_apply * (n / rows) * (m / cols_apply)
        sample += (f"; gradient = f64 LSE {rows} x {m} + apply_plan(Y) {rows} x {cols_apply}")
    if tail == "hvp":
        # the reference ships no HVP (SURVEY §0 finding 5): the SPEC composition is
        # (2 K + 3) transport-vector + 3 transport-matrix + 1 Hadamard applies of
        # apply_plan (stream.cpp:324-339, f64); time one vector apply on the row
        # slice and one matrix apply (p = d) on rows x 4096 columns
        a64 = np.full(rows, 1.0 / rows)
        bm = uniform_weights(m)
        fr = ref.update_f_hat(X64[:rows], a64, Y64, bm, g0, eps)
        v = np.ones((m, 1))
        t0 = time.perf_counter()
        ref.apply_plan(X64[:rows], a64, Y64, bm, fr, g0, eps, v)
        t_vec = time.perf_counter() - t0
        Ysub = Y64[:cols_apply]
        bsub = np.full(cols_apply, 1.0 / cols_apply)
        gsub = -(Ysub ** 2).sum(1)
        fsub = ref.update_f_hat(X64[:rows], a64, Ysub, bsub, gsub, eps)
        t0 = time.perf_counter()
        ref.apply_plan(X64[:rows], a64, Ysub, bsub, fsub, gsub, eps, Ysub)
        t_mat = time.perf_counter() - t0
        grad_s = ((2 * HVP_CG_ITERS + 3) * t_vec * n / rows +
                  4 * t_mat * (n / rows) * (m / cols_apply))
        sample += (f"; HVP = {2 * HVP_CG_ITERS + 3} x apply_plan(p=1) {rows} x {m} + 4 x "
                   f"apply_plan(p={d}) {rows} x {cols_apply}")
    sample += "; extrapolated by n/rows, m/cols"
    solves = 3 * CFG5_PAIRS if tail == "divergence" else 1
    if tail == "divergence":
        sample += f"; x {solves} solves (64 pairs x 3)"
    return dict(step_s=solves * iters * iter_s + grad_s, iter_s=iter_s, grad_s=grad_s, threads=T,
                iters=solves * iters, sample=sample, so=str(ref.so_path.name))


def run_reference(args, cfgname):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    for _ in range(args.warmup):
        reference_sample(cfgname)
    steps = [reference_sample(cfgname) for _ in range(args.steps)]
    step_s = statistics.median(s["step_s"] for s in steps)
    value = steps[0]["iters"] / step_s
    line = {
        "impl": "reference", "metric": metric_name(cfgname), "value": value, "unit": "iterations/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (fsk::Rng(1000) Gaussian)",
        "config": workload_config(cfgname),
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": steps[0]["threads"],
                         "kind": "reference", "sample": steps[0]["sample"],
                         "library": steps[0]["so"], "iter_s": steps[0]["iter_s"],
                         "grad_s": steps[0]["grad_s"]},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def metric_name(cfgname):
    n, m, d, eps, iters = CONFIGS[cfgname]
    tail = STEP_TAIL[cfgname]
    if tail == "divergence":
        return (f"Sinkhorn iterations/s ({CFG5_PAIRS} debiased divergences x 3 solves x {iters} "
                f"iterations per step), n=m={n}, d={d}")
    what = {"grad": "+ grad_X ", "hvp": "+ 1 HVP "}.get(tail, "")
    nn = "2^20" if n == 1 << 20 else str(n)
    return f"Sinkhorn iterations/s ({iters} alternating iterations {what}per step), n=m={nn}, d={d}"


METRIC = metric_name("cfg3")


def workload_config(cfgname):
    n, m, d, eps, iters = CONFIGS[cfgname]
    tail = {"grad": " + gradient w.r.t. X", "fwd": " (forward only)",
            "hvp": f" + one HVP (K_CG = {HVP_CG_ITERS}, tau = 1e-5)",
            "divergence": f" per solve, {CFG5_PAIRS} pairs x 3 solves"}[STEP_TAIL[cfgname]]
    return {"workload": f"{cfgname}: point-cloud EOT n=m={n}, d={d}, eps={eps}, "
                        f"{iters} alternating iterations{tail} per step",
            "n": n, "m": m, "d": d, "eps": eps, "iterations_per_step": iters,
            "precision": "fp32 contract (SURVEY §8d: potentials / loss within 1e-5)",
            "l2": "inputs larger than L2 (no flush needed)"}


# ------------------------------------------------------------- parity check --

def parity_sample(cfgname, X, a, Y, b, f_dev, g_dev, grad_dev, grad_lo, rows=512, grad_rows=64):
    """Sampled parity of the last timed step against the oracle, after the timed
    region (the oracle is the checker here, never the thing timed): `rows` random
    rows of the step's final g half-step (update_g_hat on the final f, through the
    C port, oracle/rows.py) and `grad_rows` random gradient rows (SPEC grad_source,
    fp64) against the device results. Contracts: SURVEY §8d (i) and the stated
    tensor-mode gradient bound max(1e-5, 2 e32)."""
    import torch

    from oracle import Oracle
    from oracle import rows as orows

    n, m, d, eps, iters = CONFIGS[cfgname]
    port = Oracle("port")
    f = f_dev[:n].double().cpu().numpy()
    g = g_dev[:m].double().cpu().numpy()
    rng = np.random.default_rng(2024)
    sel = np.sort(rng.choice(m, min(rows, m), replace=False))
    t0 = time.perf_counter()
    want = orows.half_step_rows(port, 1, X, a, Y, b, f, eps, sel)
    err = float(np.abs(g[sel] - want).max() / max(1.0, np.abs(want).max()))
    out = {"half_step": "final g-update of the last timed step", "rows": int(len(sel)),
           "max_rel_err": err, "bound": 1e-5,
           "norm": "||g_gpu - g_64||_inf / max(1, ||g_64||_inf) over the sampled rows"}
    if grad_dev is not None:
        R = grad_dev.shape[0]
        gsel = np.sort(rng.choice(R, min(grad_rows, R), replace=False))
        Gs = grad_dev[torch.as_tensor(gsel, device=grad_dev.device)].double().cpu().numpy()
        rows_x = gsel + grad_lo
        G64, r64, _ = orows.grad_rows(port, X, a, Y, b, f, g, eps, rows_x)
        e32 = orows.grad_rows_fp32_error(port, X, a, Y, b, f, g, eps, rows_x, G64, r64)
        gerr = float(np.abs(Gs - G64).max() / np.abs(G64).max())
        out.update(grad_rows=int(len(gsel)), grad_max_rel_err=gerr, grad_ref_fp32_err=e32,
                   grad_bound=max(1e-5, 2.0 * e32))
    out["ok"] = bool(err <= 1e-5 and out.get("grad_max_rel_err", 0.0) <= out.get("grad_bound", 1.0))
    out["check_s"] = time.perf_counter() - t0
    return out


# --------------------------------------------------------------- B200 arm -----

def run_b200(args, cfgname):
    import torch
    import torch.distributed as dist

    import paper_2602_03067_b200 as fsk
    from paper_2602_03067_b200.sharded import ShardPlan, ShardedSinkhorn

    n, m, d, eps, iters = CONFIGS[cfgname]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # one dedicated (non-default) stream: the engine's kernels, torch's NCCL
    # collectives and the CUDA events all live on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    X, Y = make_inputs(n, m, d)
    a = uniform_weights(n)
    b = uniform_weights(m)
    eng = fsk.Engine(local, X, a, Y, b, mode=args.mode)
    eng.set_eps(eps)
    plan = ShardPlan(rank, world, n, m)
    solver = ShardedSinkhorn(eng, plan, torch.device("cuda", local),
                             dist if world > 1 else None)
    lo, hi = plan.f_bounds[rank]
    grad = torch.empty((max(hi - lo, 1), d), dtype=torch.float32, device="cuda")
    hvp_dir = np.random.default_rng(7).standard_normal((n, d)) if STEP_TAIL[cfgname] == "hvp" \
        else None
    sptr = stream.cuda_stream
    hvp = None
    if STEP_TAIL[cfgname] == "hvp":
        # the HVP on the engine's resident potentials, rows sharded over the ranks (2
        # all-gathers per CG iteration, paper_2602_03067_b200.sharded.ShardedHvp);
        # X, Y, A replicated fp64 on the device (row-local assembly)
        from paper_2602_03067_b200.sharded import ShardedHvp
        dev = torch.device("cuda", local)
        hvp = ShardedHvp(eng, plan, dev, dist if world > 1 else None)
        Xd = torch.tensor(X, dtype=torch.float64, device=dev)
        Yd = torch.tensor(Y, dtype=torch.float64, device=dev)
        Ad = torch.tensor(hvp_dir, dtype=torch.float64, device=dev)

    # the engine launches on its own stream unless given one: pass torch's
    def half(side, lo_, hi_):
        eng.half_step(side, lo_, hi_, 0, sptr)

    # single GPU on the CUDA-core path (small d, launch-bound): the whole loop is one
    # CUDA-graph launch inside the engine
    graph_loop = world == 1 and not eng.path.startswith("tcgen05")

    def step(events=None):
        eng.init_potentials(sptr)
        if graph_loop:
            if events is not None:
                events.append(torch.cuda.Event(enable_timing=True))
                events[-1].record(stream)
            eng.iterate(iters, sptr)
            if events is not None:
                events.append(torch.cuda.Event(enable_timing=True))
                events[-1].record(stream)
        for _ in range(0 if graph_loop else iters):
            flo, fhi = plan.f_bounds[rank]
            if events is not None:
                events.append(torch.cuda.Event(enable_timing=True))
                events[-1].record(stream)
            half(0, flo, fhi)
            if events is not None:
                events.append(torch.cuda.Event(enable_timing=True))
                events[-1].record(stream)
            solver._gather(solver.f, plan.f_per)
            glo, ghi = plan.g_bounds[rank]
            if events is not None:
                events.append(torch.cuda.Event(enable_timing=True))
                events[-1].record(stream)
            half(1, glo, ghi)
            if events is not None:
                events.append(torch.cuda.Event(enable_timing=True))
                events[-1].record(stream)
            solver._gather(solver.g, plan.g_per)
        if STEP_TAIL[cfgname] == "hvp":
            # SPEC hvp_apply at the step's potentials: K_CG = 50 fixed
            if events is not None:
                gev.append(torch.cuda.Event(enable_timing=True))
                gev[-1].record(stream)
            hvp.apply(Xd, Yd, Ad, eps, tau=1e-5, cg_tol=1e-30, cg_max_iters=HVP_CG_ITERS)
            if events is not None:
                gev.append(torch.cuda.Event(enable_timing=True))
                gev[-1].record(stream)
            return
        if STEP_TAIL[cfgname] != "grad":
            return
        if events is not None:
            gev.append(torch.cuda.Event(enable_timing=True))
            gev[-1].record(stream)
        eng.grad(lo, hi, grad.data_ptr(), sptr)
        if events is not None:
            gev.append(torch.cuda.Event(enable_timing=True))
            gev[-1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler([local]) if rank == 0 else None
    if sampler:
        sampler.start()
    launches0 = fsk.Engine.launches()
    live0, sblk0 = eng.live_tiles(), eng.screened_blocks()
    pc0 = eng.pass_counts() if eng.path.startswith("tcgen05") else {}
    events = []
    gev = []
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(stream)
    for _ in range(args.steps):
        step(events)
    stop.record(stream)
    torch.cuda.synchronize()
    launches = fsk.Engine.launches() - launches0
    live, sblk = eng.live_tiles() - live0, eng.screened_blocks() - sblk0
    pc1 = eng.pass_counts() if pc0 else {}
    n_screened = pc1.get("screened", 0) - pc0.get("screened", 0)
    clocks = sampler.stop() if sampler else None
    elapsed = start.elapsed_time(stop) / 1e3
    half_ms = [events[i].elapsed_time(events[i + 1]) / (2 * iters if graph_loop else 1)
               for i in range(0, len(events), 2)]
    grad_ms = sorted(gev[i].elapsed_time(gev[i + 1]) for i in range(0, len(gev), 2))
    t = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t.item())

    # end-to-end through the public C ABI with host buffers (N = 1), or the
    # engine with host upload + gradient download per rank (N > 1)
    e2e = None
    if args.e2e:
        if world == 1:
            want_grad = STEP_TAIL[cfgname] == "grad"
            # the caller's inputs live in page-locked host memory (the library's pinned
            # pool), as a serving process would keep its batches: one DMA per cloud
            X, Y, a, b = (fsk.pinned_copy(v) for v in (X, Y, a, b))
            # untimed calls first (lazy module loading, allocator and pinned-pool
            # warm-up), as many as the device-resident arm's warmup steps; each keeps
            # its result alive until the next returns, as the timed loop does
            def e2e_step():
                o = fsk.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=iters,
                                       precision="single", grad=want_grad)
                h = None
                if STEP_TAIL[cfgname] == "hvp":
                    h, _ = fsk.hvp_apply(X, a, Y, b, o["f_hat"], o["g_hat"], eps, hvp_dir,
                                         tau=1e-5, cg_tol=1e-30, cg_max_iters=HVP_CG_ITERS,
                                         precision="single")
                return o, h

            for _ in range(max(2, args.warmup)):
                out, hv = e2e_step()
            # the same K steps as the device-resident arm, each a full call with host
            # buffers (upload, solve, gradient or HVP, download)
            t0 = time.perf_counter()
            for _ in range(args.steps):
                out, hv = e2e_step()
            e2e_s = (time.perf_counter() - t0) / args.steps
            e2e = {"value": iters / e2e_s, "unit": "iterations/s", "steps": args.steps,
                   "h2d_bytes_per_step": int(X.nbytes + Y.nbytes + a.nbytes + b.nbytes) *
                   (2 if STEP_TAIL[cfgname] == "hvp" else 1),
                   "d2h_bytes_per_step": int((out["grad"].nbytes if want_grad else 0) +
                                             out["f_hat"].nbytes + out["g_hat"].nbytes +
                                             (hv.nbytes if STEP_TAIL[cfgname] == "hvp" else 0)),
                   "api": "fsk_sinkhorn_solve_grad (+ fsk_hvp_apply_single for cfg4), C ABI, "
                          "host double buffers (page-locked: fsk_host_alloc pool)",
                   "loss": out["dual_cost"]}
        else:
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            eng2 = fsk.Engine(local, X, a, Y, b, mode=args.mode)
            eng2.set_eps(eps)
            s2 = ShardedSinkhorn(eng2, plan, torch.device("cuda", local), dist)
            s2.init()
            s2.iterate(iters)
            gh = torch.empty((max(hi - lo, 1), d), dtype=torch.float32, device="cuda")
            s2.grad_shard(gh)
            g_host = gh.cpu().numpy()
            f_host = s2.f[:n].cpu().numpy()
            torch.cuda.synchronize()
            e2e_t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
            e2e = {"value": iters / float(e2e_t.item()), "unit": "iterations/s",
                   "h2d_bytes_per_step": int(X.nbytes + Y.nbytes + a.nbytes + b.nbytes),
                   "d2h_bytes_per_step": int(g_host.nbytes + f_host.nbytes),
                   "api": "fsk_engine_* (C ABI) per rank, host double buffers"}
            eng2.close()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    pk, pk_kind = peaks()
    # roofline of the dominant kernel (the half-step LSE kernel): algorithmic
    # FLOPs of one launch over this rank's rows, W_dot = 2 n_rows m d,
    # against the peak of the precision mode that runs it (SURVEY §8d "which
    # roofline applies by mode"): the split-fp16 tensor mode issues
    # (12 C + 1) K16 MMAs per 64 C features where one fp16 pass issues 4 C, so
    # its dot-product peak is the measured dense fp16/bf16 peak / mode_factor.
    rows0 = plan.f_bounds[0][1] - plan.f_bounds[0][0]
    hs = sorted(half_ms)
    med_half = hs[len(hs) // 2] / 1e3
    # the executed fraction below is an average over every LSE pass of the timed
    # steps (cold first passes included), so the time it pairs with is the mean
    # over all timed half-steps (f and g), not the median warm one
    mean_half = sum(half_ms) / len(half_ms) / 1e3
    w_dot = 2.0 * rows0 * m * d
    sm_clk = (clocks or {}).get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)
    tensor = eng.path.startswith("tcgen05")
    chunks = -(-d // 64)
    # block skipping (warm bounds / screen): the kernel scores only the blocks it
    # cannot prove negligible, in units of (query tile, 64-key half) - the MMA and
    # epilogue unit of the d <= 64 kernel. Executed fraction over the timed LSE
    # passes: the live halves of the passes whose live count was read back, plus
    # every half of the untracked (plain) passes.
    passes = args.steps * (2 * iters + (1 if STEP_TAIL[cfgname] == "grad" else 0))
    blocks_pass = -(-rows0 // 128) * -(-m // 128)   # (query tile, key tile) blocks
    if tensor and chunks == 1:
        blocks_pass *= 2   # 64-key halves
    total_blocks = passes * blocks_pass
    # the screen's phase 1 (5 of the 13 MMAs over every block of a screened cold
    # pass) is tensor work too: counted at its MMA share
    screen_work = n_screened * blocks_pass * 5.0 / 13.0 if (tensor and chunks == 1) else 0.0
    executed = min(1.0, (live + max(0, total_blocks - sblk) + screen_work) / total_blocks) \
        if total_blocks else 1.0
    achieved = executed * w_dot / mean_half / 1e12
    if tensor:
        mode_factor = (12 * chunks + 1) / (4.0 * chunks) * (64.0 * chunks / d)
        peak_raw = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
        peak = peak_raw / mode_factor
        peak_src = (f"{pk_kind} bf16_tflops_sustained {peak_raw} / split-fp16 mode factor "
                    f"{mode_factor:.3f}")
        kernel = "tc_lse_chunked_kernel<false>" if chunks > 1 else "tc_lse_tq_kernel<false, *>"
    else:
        mode_factor = 1.0
        peak = 2.0 * 128 * 148 * sm_clk * 1e6 / 1e12   # FP32 FMA at the sampled clock
        peak_src = f"FP32 FMA 148 SM x 128 lanes x 2 x {sm_clk} MHz (sampled clock)"
        kernel = "lse_partial_kernel (CUDA-core FP32)"
    exp_floor = rows0 * m / (16.0 * 148 * sm_clk * 1e6)
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(cfgname, {}).get("bytes_per_launch")
    step_s = elapsed / args.steps
    value = iters * args.steps / elapsed
    line = {
        "metric": metric_name(cfgname), "value": value, "unit": "iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (fsk::Rng(1000) Gaussian clouds, uniform weights)",
        "config": workload_config(cfgname),
        "parallelism": (f"row-shard x{world} + NCCL all-gather of potentials" if world > 1
                        else "1 GPU"),
        "path": eng.path + (" (split-fp16 scores on tcgen05, fp32 accumulate)"
                            if eng.path.startswith("tcgen05") else ""),
        "half_step_ms": med_half * 1e3,
        "half_step_mean_ms": mean_half * 1e3,
        ("hvp_ms" if STEP_TAIL[cfgname] == "hvp" else "grad_ms"):
            grad_ms[len(grad_ms) // 2] if grad_ms else None,
        "roofline": {"bound": "tensor" if tensor else "fma", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "kernel": kernel + " (+bias/finalize; CUDA events around every f and g "
                               "half-step on the launching stream, mean)",
                     "algorithmic": f"W_dot = 2 n m d per half-step (n_rows={rows0}, m={m}, "
                                    f"d={d}) x executed (query tile, 64-key half) block "
                                    f"fraction {executed:.3f} (incl. {n_screened} screened "
                                    f"passes' phase-1 MMAs at 5/13 of a block)",
                     "executed_fraction": executed,
                     "effective_tflops": w_dot / mean_half / 1e12,
                     "peak_source": peak_src,
                     "exp_floor_ms": exp_floor * 1e3,
                     "mode_floor_ms": w_dot / (peak * 1e12) * 1e3},
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": e2e,
    }
    if tensor and chunks == 1:
        # block skipping in the LSE passes (warm bounds across passes, or the 5-MMA
        # screen): of the (query tile, 64-key half) blocks of the passes whose live
        # count was read back, the fraction scored in full; the rest are provably
        # < 2^-T of every row's max (T = 26 + ceil(log2 m))
        line["block_skipping"] = {"unit": "(query tile, 64-key half) blocks",
                                  "tracked_blocks": sblk, "live_blocks": live,
                                  "live_fraction": live / sblk if sblk else None}
    if args.parity:
        try:
            line["parity"] = parity_sample(cfgname, X, a, Y, b, solver.f, solver.g,
                                           grad if STEP_TAIL[cfgname] == "grad" else None, lo)
        except Exception as exc:  # oracle library absent on this host
            line["parity"] = {"ok": None, "unavailable": str(exc)}
    if world == 1 and args.cpu_baseline:
        try:
            cb = reference_sample(cfgname)
            line["cpu_baseline"] = {"value": cb["iters"] / cb["step_s"], "unit": "iterations/s",
                                    "cores": cb["threads"], "kind": "reference",
                                    "sample": cb["sample"], "library": cb["so"]}
        except Exception as exc:  # reference library absent on this host
            line["cpu_baseline"] = {"value": None, "unit": "iterations/s", "cores": None,
                                    "kind": "reference", "sample": f"unavailable: {exc}"}
    print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_b200_divergence(args, cfgname):
    """cfg5: one step = fsk_sinkhorn_divergence_batch over 64 (mu, nu) pairs, each
    pair 3 single-precision solves (cross + both debiasing terms) of `iters`
    alternating iterations, through the public C ABI with host buffers (the
    timed region includes every upload and the dual-cost readback). Pairs are
    drawn from 16 distinct Gaussian clouds (1 GB of host data instead of 8 GB);
    every pair still runs its 3 full solves."""
    import torch

    import paper_2602_03067_b200 as fsk

    n, m, d, eps, iters = CONFIGS[cfgname]
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    # 16 distinct clouds, cloud k = fsk::Rng(1000 + k).normal() (SURVEY §8d seeds)
    clouds = [fsk.rng_normal(1000 + k, n * d).reshape(n, d) for k in range(16)]
    w = uniform_weights(n)
    pairs = [(clouds[k % 16], w, clouds[(k * 7 + 3) % 16], w) for k in range(CFG5_PAIRS)]
    os.environ.setdefault("FSK_TENSOR_MODE", args.mode)
    for _ in range(args.warmup):
        fsk.sinkhorn_divergence_batch(pairs[:2], eps=eps, max_iters=iters)
    sampler = ClockSampler([0])
    sampler.start()
    launches0 = fsk.Engine.launches()
    times = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fsk.sinkhorn_divergence_batch(pairs, eps=eps, max_iters=iters)
        times.append(time.perf_counter() - t0)
    launches = fsk.Engine.launches() - launches0
    clocks = sampler.stop()
    step_s = statistics.median(times)
    its = CFG5_PAIRS * 3 * iters
    value = its / step_s
    h2d = sum(2 * (X.nbytes + a.nbytes + Y.nbytes + b.nbytes) for (X, a, Y, b) in pairs)
    # roofline (dominant kernel tc_lse_chunked_kernel, d = 784 -> 13 feature chunks):
    # algorithmic W_dot = 2 n m d per half-step x 2 iters per solve x 3 solves x 64
    # pairs over the whole step time (uploads, dual costs and the 2 marginal passes per
    # solve included in the time, not in the work: a lower bound on the kernel's rate)
    pk, pk_kind = peaks()
    chunks = -(-d // 64)
    mode_factor = (12 * chunks + 1) / (4.0 * chunks) * (64.0 * chunks / d)
    peak_raw = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    w_dot = 2.0 * n * m * d * 2 * iters * 3 * CFG5_PAIRS
    achieved = w_dot / step_s / 1e12
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_raw / mode_factor,
                "unit": "TFLOP/s", "frac": achieved / (peak_raw / mode_factor), "traffic": None,
                "kernel": "tc_lse_chunked_kernel<false> (whole C ABI step time, incl. uploads)",
                "algorithmic": f"W_dot = 2 n m d x {2 * iters} half-steps x 3 solves x "
                               f"{CFG5_PAIRS} pairs (n=m={n}, d={d})",
                "peak_source": f"{pk_kind} bf16_tflops_sustained {peak_raw} / split-fp16 mode "
                               f"factor {mode_factor:.3f}"}
    line = {
        "metric": metric_name(cfgname), "value": value, "unit": "iterations/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (16 Gaussian clouds, 64 pairs), uniform weights",
        "config": workload_config(cfgname),
        "parallelism": "1 GPU, pairs sequential",
        "api": "fsk_sinkhorn_divergence_batch (C ABI, host buffers)",
        "pairs_per_s": CFG5_PAIRS / step_s, "divergence_mean": float(np.mean(out)),
        "roofline": roofline,
        "gpu_launches": launches, "clocks": clocks,
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(out.nbytes),
                "api": "value is itself end to end (host buffers in, divergences out)"},
    }
    if args.cpu_baseline:
        cb = reference_sample(cfgname)
        line["cpu_baseline"] = {"value": cb["iters"] / cb["step_s"], "unit": "iterations/s",
                                "cores": cb["threads"], "kind": "reference",
                                "sample": cb["sample"], "library": cb["so"]}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="auto", choices=["auto", "tensor", "fma"])
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-parity", dest="parity", action="store_false")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args, args.config)
    if STEP_TAIL[args.config] == "divergence":
        return run_b200_divergence(args, args.config)
    return run_b200(args, args.config)


if __name__ == "__main__":
    sys.exit(main())
