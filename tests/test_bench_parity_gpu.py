"""Parity at the benchmarked configurations, through the same engine calls bench.py
times (VERDICT r1 "what's weak" 1).

cfg2 / cfg3: the exact bench step - fsk::Rng(1000) Gaussian clouds, uniform
weights, eps = 0.05, 10 alternating iterations from the reference init
(solver.cpp:27-32) with warm bounds and the screen ON (the 89%-skip machinery
the headline relies on) - with sampled rows of every checked half-step compared
with the oracle on the potential that went into it, and sampled gradient rows
at the final potentials.

Contracts:
  half-step  ||f_gpu - f_64||_inf <= 1e-5 max(1, ||f_64||_inf) on the sampled rows
  gradient   ||G_gpu - G_64||_inf <= max(1e-5, 2 e32) ||G_64||_inf, e32 = the error
             the reference's own fp32 half-step puts into the same rows
"""
import os
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _bench():
    sys.path.insert(0, str(ROOT))
    import bench
    return bench


def run_bench_step(fsk, torch, cfg, check_half_steps):
    """One bench step (init + iters alternating half-steps + grad) on the engine with
    the input potential of every half-step in `check_half_steps` captured."""
    bench = _bench()
    n, m, d, eps, iters = bench.CONFIGS[cfg]
    X, Y = bench.make_inputs(n, m, d)
    a, b = bench.uniform_weights(n), bench.uniform_weights(m)
    eng = fsk.Engine(0, X, a, Y, b)
    eng.set_eps(eps)
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    g = torch.empty(m, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())
    s = torch.cuda.Stream()
    sp = s.cuda_stream
    eng.init_potentials(sp)
    captured = {}
    for k in range(2 * iters):
        side = k % 2
        if k in check_half_steps:
            s.synchronize()
            pin = (g if side == 0 else f).cpu().numpy().astype(np.float64)
        eng.half_step(side, 0, n if side == 0 else m, 0, sp)
        if k in check_half_steps:
            s.synchronize()
            out = (f if side == 0 else g).cpu().numpy().astype(np.float64)
            captured[k] = (pin, out)
    G = torch.empty((n, d), dtype=torch.float32, device="cuda")
    eng.grad(0, n, G.data_ptr(), sp)
    s.synchronize()
    res = dict(X=X, Y=Y, a=a, b=b, eps=eps, f=f.cpu().numpy().astype(np.float64),
               g=g.cpu().numpy().astype(np.float64), G=G, captured=captured,
               live=eng.live_tiles(), blocks=eng.screened_blocks(), path=eng.path)
    eng.close()
    return res


@pytest.mark.parametrize("cfg,checks,rows", [
    ("cfg2", tuple(range(20)), 1024),
    ("cfg3", (0, 1, 2, 9, 18, 19), 1024),
])
def test_bench_step_parity(fsk, port, cfg, checks, rows):
    torch = pytest.importorskip("torch")
    from oracle import rows as orows

    assert os.environ.get("FSK_WARM", "1") != "0" and os.environ.get("FSK_SCREEN", "1") != "0"
    r = run_bench_step(fsk, torch, cfg, set(checks))
    X, Y, a, b, eps = r["X"], r["Y"], r["a"], r["b"], r["eps"]
    n, m = len(X), len(Y)
    assert r["path"].startswith("tcgen05")
    live_frac = r["live"] / max(1, r["blocks"])
    print(f"{cfg}: tracked blocks {r['blocks']}, live fraction {live_frac:.3f}")
    if cfg == "cfg3":
        # the skip machinery is what is under test: most blocks must have been skipped
        assert r["blocks"] > 0 and live_frac < 0.5
    rng = np.random.default_rng(77)
    worst = 0.0
    for k in checks:
        side = k % 2
        pin, out = r["captured"][k]
        R = n if side == 0 else m
        sel = np.sort(rng.choice(R, rows, replace=False))
        want = orows.half_step_rows(port, side, X, a, Y, b, pin, eps, sel)
        err = np.abs(out[sel] - want).max() / max(1.0, np.abs(want).max())
        worst = max(worst, err)
        print(f"{cfg} half-step {k} ({'f' if side == 0 else 'g'}): rel err {err:.2e}")
        assert err <= 1e-5, (k, err)
    # gradient rows at the final potentials
    gsel = np.sort(rng.choice(n, 256, replace=False))
    Gs = r["G"][torch.as_tensor(gsel, device="cuda")].cpu().numpy().astype(np.float64)
    G64, r64, _ = orows.grad_rows(port, X, a, Y, b, r["f"], r["g"], eps, gsel)
    e32 = orows.grad_rows_fp32_error(port, X, a, Y, b, r["f"], r["g"], eps, gsel, G64, r64)
    gerr = np.abs(Gs - G64).max() / np.abs(G64).max()
    print(f"{cfg} gradient rows: rel err {gerr:.2e} (reference fp32 path {e32:.2e}); "
          f"worst half-step {worst:.2e}")
    assert gerr <= max(1e-5, 2.0 * e32)


def test_dense_mode_matches_skipping_mode_cfg2(fsk, port):
    """The same cfg2 bench step with warm bounds and the screen OFF (every block
    scored) gives potentials within the contract of the skipping run: the skips
    drop only terms provably < 2^-58 of each row's max."""
    torch = pytest.importorskip("torch")
    out = {}
    for flag in ("1", "0"):
        os.environ["FSK_WARM"] = flag
        os.environ["FSK_SCREEN"] = flag
        try:
            out[flag] = run_bench_step(fsk, torch, "cfg2", set())
        finally:
            os.environ.pop("FSK_WARM", None)
            os.environ.pop("FSK_SCREEN", None)
    for key in ("f", "g"):
        ref = out["0"][key]
        err = np.abs(out["1"][key] - ref).max() / max(1.0, np.abs(ref).max())
        print(f"cfg2 {key}: skipping vs dense rel {err:.2e}")
        assert err <= 1e-5


def _solved_potentials(fsk, X, a, Y, b, eps, iters=10):
    s = fsk.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=iters, precision="single")
    return s["f_hat"], s["g_hat"]


@pytest.mark.parametrize("plan_cache", ["0", "1"])
def test_cfg4_single_precision_hvp_against_oracle(fsk, plan_cache):
    """cfg4's HVP path (d = 1024: chunked tcgen05 transport-vector passes, device CG,
    tensor-core matrix / Hadamard applies; plan cache off = the default, and on) at
    n = 2048, m = 1900 against the SPEC composition (oracle/compose.py) evaluated on
    the dense fp64 plan (oracle/dense.py DenseOps), same potentials, same direction,
    same fixed K_CG = 50 (cg_tol 1e-30, the bench setting), tau = 1e-5.
    Bound (stated tensor-mode HVP bound, like the gradient's): relative Frobenius
    error <= max(1e-5, 2 e32), e32 = the error of the same composition on the plan
    whose scores are evaluated in the reference's own fp32 arithmetic and order
    (DenseOps fp32_scores="reference", stream.cpp:61-79 / :421-434). At d = 1024,
    eps = 0.1 the score terms reach ~1.4e4 log2 units and cancel to a few hundred, so
    fp32 arithmetic alone moves plan entries by ~1e-3 relative."""
    from oracle import compose
    from oracle.dense import DenseOps
    bench = _bench()
    n, m, d, eps = 2048, 1900, 1024, 0.1
    z = fsk.rng_normal(1000, (n + m) * d)
    X, Y = z[: n * d].reshape(n, d), z[n * d:].reshape(m, d)
    a, b = bench.uniform_weights(n), bench.uniform_weights(m)
    f, g = _solved_potentials(fsk, X, a, Y, b, eps)
    A = np.random.default_rng(7).standard_normal((n, d))
    os.environ["FSK_PLAN_CACHE"] = plan_cache
    try:
        led = fsk.Ledger()
        H, info = fsk.hvp_apply(X, a, Y, b, f, g, eps, A, tau=1e-5, cg_tol=1e-30,
                                cg_max_iters=50, precision="single", ledger=led)
    finally:
        os.environ.pop("FSK_PLAN_CACHE", None)
    ws = compose.Workspace(DenseOps(), X, a, Y, b, f, g, eps)
    H64, it64, _ = compose.hvp_apply(ws, A, tau=1e-5, tol=1e-30, max_iters=50)
    ws32 = compose.Workspace(DenseOps(fp32_scores="reference"), X, a, Y, b, f, g, eps)
    H32 = compose.hvp_apply(ws32, A, tau=1e-5, tol=1e-30, max_iters=50)[0]
    rel = np.linalg.norm(H - H64) / np.linalg.norm(H64)
    e32 = np.linalg.norm(H32 - H64) / np.linalg.norm(H64)
    print(f"cfg4-shape HVP (plan cache {plan_cache}): rel Frobenius {rel:.2e} "
          f"(reference fp32 score arithmetic {e32:.2e}), CG {info['cg_iters']} vs {it64}")
    assert info["cg_iters"] == it64 == 50
    assert led.transport_vector_applies == 2 * 50 + 3
    assert rel <= max(1e-5, 2.0 * e32)


def test_cfg4_hvp_peak_memory_contract(fsk):
    """peak allocation during hvp_apply <= c (n + m) d scalars, never
    n m. At the cfg4 shape (n = m = 1e5, d = 1024) the default single-precision HVP
    stays under 16 (n + m) d fp32 scalars (13 GB; n m fp32 = 40 GB), and the opt-in
    plan cache (FSK_PLAN_CACHE=1, 31 GB of plan blocks) is shown to break it, so
    the check has teeth."""
    bench = _bench()
    n = m = 100000
    d = 1024
    z = fsk.rng_normal(1000, (n + m) * d)
    X, Y = z[: n * d].reshape(n, d), z[n * d:].reshape(m, d)
    del z
    a, b = bench.uniform_weights(n), bench.uniform_weights(m)
    f, g = _solved_potentials(fsk, X, a, Y, b, 0.1, iters=3)
    A = np.random.default_rng(7).standard_normal((n, d))
    bound = 16 * (n + m) * d * 4
    peaks = {}
    for flag in ("0", "1"):
        os.environ["FSK_PLAN_CACHE"] = flag
        try:
            fsk.device_peak_bytes(0, reset=True)
            fsk.hvp_apply(X, a, Y, b, f, g, 0.1, A, tau=1e-5, cg_tol=1e-30, cg_max_iters=3,
                          precision="single")
            peaks[flag] = fsk.device_peak_bytes(0)
        finally:
            os.environ.pop("FSK_PLAN_CACHE", None)
    print(f"HVP peak device bytes: default {peaks['0'] / 2**30:.2f} GiB, plan cache "
          f"{peaks['1'] / 2**30:.2f} GiB, bound 16 (n+m) d fp32 = {bound / 2**30:.2f} GiB")
    assert 0 < peaks["0"] <= bound
    assert peaks["1"] > bound


def test_cfg5_divergence_batch_against_oracle(fsk, port):
    """cfg5's path (d = 784, chunked tcgen05 kernels, single precision, the batched
    C ABI entry) against the port's fp64 solves: per pair S = OT(mu,nu) -
    OT(mu,mu)/2 - OT(nu,nu)/2 after 10 alternating iterations each (solver.cpp:145-159).
    Bound: |S_gpu - S_64| <= 1e-5 (|OT_xy| + |OT_xx|/2 + |OT_yy|/2) (the loss
    contract of SURVEY §8d ii applied to the three dual costs)."""
    bench = _bench()
    d, eps, iters = 784, 0.1, 10
    rng = np.random.default_rng(1000)
    sizes = [640, 640, 700]
    clouds = [rng.standard_normal((k, d)) for k in sizes]
    ws = [bench.uniform_weights(k) for k in sizes]
    idx = [(0, 1), (1, 2)]
    pairs = [(clouds[i], ws[i], clouds[j], ws[j]) for i, j in idx]
    got = fsk.sinkhorn_divergence_batch(pairs, eps=eps, max_iters=iters)
    for k, (X, a, Y, b) in enumerate(pairs):
        ot = [port.sinkhorn_solve(P, p, Q, q, eps=eps, max_iters=iters)["dual_cost"]
              for P, p, Q, q in ((X, a, Y, b), (X, a, X, a), (Y, b, Y, b))]
        want = ot[0] - 0.5 * ot[1] - 0.5 * ot[2]
        scale = abs(ot[0]) + 0.5 * abs(ot[1]) + 0.5 * abs(ot[2])
        err = abs(got[k] - want) / scale
        print(f"cfg5 pair {k}: S_gpu {got[k]:.9g} S_64 {want:.9g} err/scale {err:.2e}")
        assert err <= 1e-5
