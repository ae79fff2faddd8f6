"""Parity of the CUDA path (called through the C ABI) with the oracle.

Double-precision ops must meet the reference's own test tolerances
(1e-12 potentials / 1e-10 transport, test_stream.cpp); single precision meets
the SURVEY §8(d) contract: ||df||_inf <= 1e-5 max(1, ||f||_inf) against the
reference's fp64 half-step, loss within 1e-5 relative.
"""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import compose, dense
from oracle.rng import Rng, random_measure

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(1.0, np.abs(np.asarray(b)).max())


def test_reference_test_stream_suite_on_b200():
    """proj/tests/test_stream.cpp, unmodified, against libfsk_b200.so: 16/16."""
    exe = ROOT / "tests" / "refsuite" / "_bin" / "test_stream_b200"
    assert exe.exists(), "refsuite binary missing (built by __graft_entry__.build())"
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr[-4000:]
    assert "16 passed | 0 failed" in out.stdout


def test_half_steps_golden(fsk, golden):
    G = golden
    out = fsk.update_f_hat(G["fu_X"], G["fu_a"], G["fu_Y"], G["fu_b"], G["fu_g"], 0.1, (16, 24))
    assert np.all(np.abs(out - G["fu_out"]) <= 1e-12 * (1 + np.abs(G["fu_out"])))
    out = fsk.update_g_hat(G["gu_X"], G["gu_a"], G["gu_Y"], G["gu_b"], G["gu_f"], 0.2, (8, 8))
    assert np.abs(out - G["gu_out"]).max() < 1e-12
    out = fsk.update_f_hat(G["tl_X"], G["tl_a"], G["tl_Y"], G["tl_b"], G["tl_g"], 0.15, (5, 7))
    assert np.all(np.abs(out - G["tl_out"]) <= 1e-12 * (1 + np.abs(G["tl_out"])))


def test_transport_golden(fsk, golden):
    G = golden
    args = (G["tr_X"], G["tr_a"], G["tr_Y"], G["tr_b"], G["tr_f"], G["tr_g"], 0.3)
    for got, want in [(fsk.apply_plan(*args, G["tr_V"]), G["tr_PV"]),
                      (fsk.apply_plan_adjoint(*args, G["tr_U"]), G["tr_PtU"]),
                      (fsk.apply_hadamard_plan(*args, G["tr_A"], G["tr_B"], G["tr_V"][:, :2]),
                       G["tr_HV"])]:
        assert np.abs(got - want).max() <= 1e-10 * (1 + np.abs(want).max())
    r, c = fsk.induced_marginals(*args)
    assert np.abs(r - G["tr_r"]).max() <= 1e-12 * np.abs(G["tr_r"]).max()
    assert np.abs(c - G["tr_c"]).max() <= 1e-12 * np.abs(G["tr_c"]).max()
    fs, gs = fsk.symmetric_update(*args)
    assert rel(fs, G["tr_sym_f"]) < 1e-12 and rel(gs, G["tr_sym_g"]) < 1e-12
    assert abs(fsk.dual_cost(*args) - float(G["tr_dual"])) < 1e-10


def test_label_augmented_golden(fsk, golden):
    G = golden
    cost = dict(lambda1=0.5, lambda2=0.5, label_cost=G["lab_W"])
    out = fsk.update_f_hat(G["lab_X"], G["lab_a"], G["lab_Y"], G["lab_b"], G["lab_g"], 0.25,
                           cost=cost, la=G["lab_la"], lb=G["lab_lb"])
    assert np.all(np.abs(out - G["lab_out"]) <= 1e-12 * (1 + np.abs(G["lab_out"])))


@pytest.mark.parametrize("sch", ["alternating", "symmetric"])
def test_solver_double_golden(fsk, golden, sch):
    G = golden
    s = fsk.sinkhorn_solve(G["sv_X"], G["sv_a"], G["sv_Y"], G["sv_b"], eps=0.2, max_iters=40,
                           schedule=sch)
    key = f"sv_d{sch[0]}"
    assert rel(s["f_hat"], G[key + "_f"]) < 1e-11
    assert s["iterations"] == int(G[key + "_s"][0])
    assert abs(s["dual_cost"] - G[key + "_s"][2]) < 1e-10
    assert abs(s["marginal_violation"] - G[key + "_s"][1]) < 1e-9


@pytest.mark.parametrize("sch", ["alternating", "symmetric"])
def test_solver_single_golden(fsk, golden, sch):
    G = golden
    s = fsk.sinkhorn_solve(G["sv_X"], G["sv_a"], G["sv_Y"], G["sv_b"], eps=0.2, max_iters=40,
                           schedule=sch, precision="single")
    key = f"sv_s{sch[0]}"
    assert rel(s["f_hat"], G[key + "_f"]) < 1e-5
    assert abs(s["dual_cost"] - G[key + "_s"][2]) <= 1e-5 * abs(G[key + "_s"][2])


def test_solver_tolerance_and_scaling_golden(fsk, golden):
    G = golden
    X, a, Y, b = G["sv_X"], G["sv_a"], G["sv_Y"], G["sv_b"]
    s = fsk.sinkhorn_solve(X, a, Y, b, eps=0.2, max_iters=2000, marginal_tol=1e-9)
    assert abs(s["iterations"] - int(G["sv_tol_s"][0])) <= 1
    assert abs(s["dual_cost"] - G["sv_tol_s"][2]) < 1e-9
    if s["iterations"] == int(G["sv_tol_s"][0]):
        # the fused lagged check reports the reference's violation of the same iterate
        assert abs(s["marginal_violation"] - G["sv_tol_s"][1]) <= 1e-6 * G["sv_tol_s"][1]
    s = fsk.sinkhorn_solve(X, a, Y, b, eps=0.2, max_iters=300, eps_scaling_factor=0.8,
                           extra_iters_at_final_eps=20)
    assert np.array_equal(s["eps_history"], G["sv_sc_hist"])
    assert rel(s["f_hat"], G["sv_sc_f"]) < 1e-10
    d = fsk.sinkhorn_divergence(X, a, Y, b, eps=0.2, max_iters=60)
    assert abs(d - float(G["sv_div"])) < 1e-10


def test_cfg1_golden(fsk, golden):
    """BASELINE cfg1 through the device-resident fp64 solver."""
    G = golden
    u = np.full(4096, 1.0 / 4096)
    s = fsk.sinkhorn_solve(G["cfg1_X"], u, G["cfg1_Y"], u, eps=0.1, max_iters=100)
    assert rel(s["f_hat"], G["cfg1_f"]) < 1e-11
    assert abs(s["dual_cost"] - G["cfg1_s"][2]) <= 1e-11 * abs(G["cfg1_s"][2])


def test_f32_half_step_contract(fsk, golden):
    G = golden
    out = fsk.update_f_hat_f32(G["f32_X"], G["f32_a"], G["f32_Y"], G["f32_b"], G["f32_g"], 0.05)
    ref64 = G["f32_out64"]
    assert np.abs(out - ref64).max() <= 1e-5 * max(1.0, np.abs(ref64).max())
    # and it is at least as close to fp64 as the reference's own fp32 path, up to 4x
    ref32_err = np.abs(G["f32_out"] - ref64).max()
    assert np.abs(out - ref64).max() <= max(4 * ref32_err, 1e-6 * np.abs(ref64).max())


@pytest.mark.parametrize("n,m,d", [(200, 300, 3), (513, 257, 16), (640, 384, 64), (300, 200, 40)])
def test_f32_half_steps_random(fsk, port, n, m, d):
    rng = np.random.default_rng(n + m + d)
    X = rng.normal(size=(n, d))
    Y = rng.normal(size=(m, d))
    a = np.full(n, 1.0 / n)
    b = rng.random(m) + 0.5
    b /= b.sum()
    g = -(Y ** 2).sum(1) * 0.9
    for eps in (0.05, 0.5):
        want = port.update_f_hat(X, a, Y, b, g, eps)
        got = fsk.update_f_hat_f32(X, a, Y, b, g, eps)
        assert np.abs(got - want).max() <= 1e-5 * max(1.0, np.abs(want).max()), (eps,)
        f = want
        want_g = port.update_g_hat(X, a, Y, b, f, eps)
        got_g = fsk.update_g_hat_f32(X, a, Y, b, f, eps)
        assert np.abs(got_g - want_g).max() <= 1e-5 * max(1.0, np.abs(want_g).max())


def test_gradient_and_barycentric(fsk, port):
    rng = Rng(11)
    X, a = random_measure(rng, 96, 3, False)
    Y, b = random_measure(rng, 80, 3, False)
    s = port.sinkhorn_solve(X, a, Y, b, eps=0.3, max_iters=50)
    f, g = s["f_hat"], s["g_hat"]
    ws = compose.Workspace(port, X, a, Y, b, f, g, 0.3)
    Gs = fsk.grad_source(X, a, Y, b, f, g, 0.3)
    assert np.abs(Gs - compose.grad_source(ws)).max() <= 1e-10 * np.abs(Gs).max()
    Gt = fsk.grad_target(X, a, Y, b, f, g, 0.3)
    assert np.abs(Gt - compose.grad_target(ws)).max() <= 1e-10 * np.abs(Gt).max()
    T = fsk.barycentric_projection(X, a, Y, b, f, g, 0.3)
    assert np.abs(T - compose.barycentric_projection(ws)).max() <= 1e-10


def test_solve_grad_single(fsk, port):
    rng = np.random.default_rng(3)
    n, m, d = 512, 384, 64
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d))
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    s = fsk.sinkhorn_solve(X, a, Y, b, eps=1.0, max_iters=10, precision="single", grad=True)
    r = port.sinkhorn_solve(X, a, Y, b, eps=1.0, max_iters=10, precision="double")
    assert np.abs(s["f_hat"] - r["f_hat"]).max() <= 1e-5 * np.abs(r["f_hat"]).max()
    assert abs(s["dual_cost"] - r["dual_cost"]) <= 1e-5 * abs(r["dual_cost"])
    # gradient contract (SURVEY §8d ii): at the returned (fp32) potentials, within
    # max(1e-5, 2x) the error of the reference's own fp32 arithmetic
    from test_tensor_gpu import grad_errors
    e_gpu, e32, _ = grad_errors(port, X, a, Y, b, s["f_hat"], s["g_hat"], 1.0, s["grad"])
    assert e_gpu <= max(1e-5, 2.0 * e32)
    # end to end against the fp64 solve: dominated by the fp32 storage of the
    # potentials (|f_hat| ~ |x|^2 ~ 64, ulp 7.6e-6, enters r through exp(df/eps))
    ws64 = compose.Workspace(port, X, a, Y, b, r["f_hat"], r["g_hat"], 1.0)
    G64 = compose.grad_source(ws64)
    assert np.abs(s["grad"] - G64).max() <= 1e-4 * np.abs(G64).max()


def test_hvp_against_dense_and_composition(fsk, port):
    rng = Rng(5)
    X, a = random_measure(rng, 48, 3, False)
    Y, b = random_measure(rng, 40, 3, False)
    eps = 0.5
    s = port.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=3000, marginal_tol=1e-12)
    f, g = s["f_hat"], s["g_hat"]
    A = np.random.default_rng(1).normal(size=X.shape)
    led = fsk.Ledger()
    H, info = fsk.hvp_apply(X, a, Y, b, f, g, eps, A, tau=0.0, cg_tol=1e-12, cg_max_iters=500,
                            ledger=led)
    P = dense.dense_plan(X, a, Y, b, f, g, eps)
    Hd = dense.dense_hvp(dense.dense_hessian(X, Y, P, eps), A)
    assert np.linalg.norm(H - Hd) <= 1e-8 * np.linalg.norm(Hd)
    K = info["cg_iters"]
    assert led.transport_vector_applies == 2 * K + 3
    assert led.transport_matrix_applies == 3
    assert led.hadamard_applies == 1
    # default damping (SPEC acceptance 4 bound)
    H2, _ = fsk.hvp_apply(X, a, Y, b, f, g, eps, A)
    assert np.linalg.norm(H2 - Hd) <= 2e-2 * np.linalg.norm(Hd)


def test_ledger_matches_reference(fsk, ref):
    rng = Rng(89)
    X, a = random_measure(rng, 45, 5)
    Y, b = random_measure(rng, 33, 5)
    s = ref.sinkhorn_solve(X, a, Y, b, eps=0.5, max_iters=3, tiles=(8, 16))
    f, g = s["f_hat"], s["g_hat"]
    led = fsk.Ledger()
    fsk.sinkhorn_solve(X, a, Y, b, eps=0.5, max_iters=3, tiles=(8, 16), ledger=led)
    # 3 iterations (2 half-steps each) + marginals + dual_cost(marginals)
    expect = 3 * (fsk.io_count("f_update", 45, 33, 5, tiles=(8, 16)) +
                  fsk.io_count("g_update", 45, 33, 5, tiles=(8, 16))) + \
        2 * fsk.io_count("induced_marginals", 45, 33, 5, tiles=(8, 16))
    assert led.total_scalars() == expect
    assert led.kernel_invocations == 3 * 2 + 2


def test_numerical_error_on_overflow(fsk):
    X = np.array([[0.0], [1.0]])
    w = np.array([0.5, 0.5])
    with pytest.raises(fsk.NumericalError):
        fsk.apply_plan(X, w, X, w, [800.0, 800.0], [0.0, 0.0], 1.0, np.ones((2, 1)))


def test_break_lse_negative_control(fsk, port):
    """Flipping the online rescale must break every multi-tile stream
    (stream.cpp:81-87); our kernels stream 64-column tiles, so use m > 64."""
    rng = np.random.default_rng(9)
    X, Y = rng.normal(size=(64, 4)), rng.normal(size=(700, 4))
    a, b = np.full(64, 1 / 64), np.full(700, 1 / 700)
    g = rng.normal(size=700)
    good = port.update_f_hat(X, a, Y, b, g, 0.1)
    fsk.debug_break_lse(True)
    try:
        # a broken recurrence must be caught: either wrong potentials or the
        # reference's own NumericalError on a non-finite one (stream.cpp:127-130);
        # which one depends on how often the running max moves, i.e. on tiling
        for fn, tol in ((fsk.update_f_hat, 1e-6), (fsk.update_f_hat_f32, 1e-3)):
            try:
                bad = fn(X, a, Y, b, g, 0.1)
                assert np.abs(bad - good).max() > tol
            except fsk.NumericalError:
                pass
    finally:
        fsk.debug_break_lse(False)
    assert np.abs(fsk.update_f_hat(X, a, Y, b, g, 0.1) - good).max() < 1e-12


@pytest.mark.parametrize("tol", [1e-3, 1e-6, 1e-9])
def test_fused_convergence_matches_reference_stop(fsk, port, tol):
    """N1: the drop-in fp64 solver's early stop runs the reference's check
    (solver.cpp:51-60) as a by-product of the next f-update (one extra pass at the
    stop instead of two marginal passes per iteration): same stopping iterate, the
    same violation to 1e-6 relative, the same dual cost, and the reference ledger."""
    rng = np.random.default_rng(31)
    n, m, d = 300, 260, 5
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d)) * 0.8 + 0.1
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    led = fsk.Ledger()
    s = fsk.sinkhorn_solve(X, a, Y, b, eps=0.3, max_iters=500, marginal_tol=tol, ledger=led)
    r = port.sinkhorn_solve(X, a, Y, b, eps=0.3, max_iters=500, marginal_tol=tol)
    assert abs(s["iterations"] - r["iterations"]) <= 1
    if s["iterations"] == r["iterations"]:
        assert abs(s["marginal_violation"] - r["marginal_violation"]) <= \
            1e-6 * r["marginal_violation"]
        assert rel(s["f_hat"], r["f_hat"]) < 1e-10
        assert abs(s["dual_cost"] - r["dual_cost"]) <= 1e-10 * abs(r["dual_cost"])
    assert s["marginal_violation"] <= tol or s["iterations"] == 500
    # ledger (closed forms, solver.cpp:36-66): every iteration at the final eps runs
    # the reference's check (induced_marginals), plus dual_cost's marginals at the stop
    # (or the final marginals + dual_cost when the cap is hit)
    K = s["iterations"]
    stopped = s["marginal_violation"] <= tol
    expect = K * (fsk.io_count("f_update", n, m, d) + fsk.io_count("g_update", n, m, d)) + \
        (K + (1 if stopped else 2)) * fsk.io_count("induced_marginals", n, m, d)
    assert led.total_scalars() == expect
