"""The tcgen05 split-fp16 half-step (fp32-accurate tensor-core path) and the
device engine, against the oracle.

Contract: ||f_gpu - f_ref64||_inf <= 1e-5 max(1, ||f_ref64||_inf)
for one half-step from identical inputs.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def contract(got, want):
    return np.abs(got - want).max() / max(1.0, np.abs(want).max())


def grad_errors(port, X, a, Y, b, f, g, eps, got):
    """Gradient contract (SURVEY §8d ii, tensor-mode statement): at identical
    potentials, ||G_gpu - G_64||_inf <= max(1e-5, 2 e32) ||G_64||_inf where e32 is
    the error the reference's own fp32 arithmetic makes on the same inputs.

    G = 2(diag(r) X - P Y) and r_i = a_i exp((f_i - f+_i)/eps) turns an absolute
    score error delta into a relative gradient error delta/eps: no fp32 evaluation
    of f+ (|f+| ~ |x|^2) reaches 1e-5 at eps = 0.05. e32 recomputes r with f+ from
    the reference's update_f_hat_f32 (stream.cpp:437-443), P Y in fp64."""
    from oracle import compose
    ws = compose.Workspace(port, X, a, Y, b, f, g, eps)
    G64 = compose.grad_source(ws)
    fp32 = port.update_f_hat_f32(X, a, Y, b, g, eps).astype(np.float64)
    r32 = a * np.exp((f - fp32) / eps)
    G32 = 2.0 * (r32[:, None] * X - (r32 / ws.r)[:, None] * ws.PY)
    scale = np.abs(G64).max()
    return np.abs(got - G64).max() / scale, np.abs(G32 - G64).max() / scale, G64


@pytest.fixture()
def tensor_mode():
    os.environ["FSK_TENSOR_MODE"] = "tensor"
    yield
    os.environ.pop("FSK_TENSOR_MODE", None)


@pytest.mark.parametrize("n,m,d", [(128, 128, 64), (384, 320, 64), (1000, 777, 64),
                                   (515, 1300, 33), (260, 513, 16), (129, 131, 3),
                                   # chunked kernel (d > 64): cfg4 / cfg5 feature dims
                                   (300, 421, 784), (260, 300, 1024), (129, 200, 100),
                                   (640, 700, 128)])
@pytest.mark.parametrize("eps", [0.05, 1.0])
def test_tensor_half_step_parity(fsk, port, tensor_mode, n, m, d, eps):
    rng = np.random.default_rng(n * 7 + m + d)
    X = rng.normal(size=(n, d))
    Y = rng.normal(size=(m, d)) + 0.3
    a = np.full(n, 1.0 / n)
    b = rng.random(m) + 0.2
    b /= b.sum()
    g = -(Y ** 2).sum(1) + rng.normal(size=m)
    want = port.update_f_hat(X, a, Y, b, g, eps)
    got = fsk.update_f_hat_f32(X, a, Y, b, g, eps)
    assert contract(got, want) <= 1e-5
    wg = port.update_g_hat(X, a, Y, b, want, eps)
    gg = fsk.update_g_hat_f32(X, a, Y, b, want, eps)
    assert contract(gg, wg) <= 1e-5


def test_tensor_scaling_invariance(fsk, port, tensor_mode):
    """Large / tiny coordinates exercise the power-of-two operand scaling."""
    rng = np.random.default_rng(1)
    for s in (1e-3, 40.0):
        X = rng.normal(size=(300, 64)) * s
        Y = rng.normal(size=(200, 64)) * s
        a, b = np.full(300, 1 / 300), np.full(200, 1 / 200)
        g = -(Y ** 2).sum(1)
        eps = 0.1 * s * s
        want = port.update_f_hat(X, a, Y, b, g, eps)
        got = fsk.update_f_hat_f32(X, a, Y, b, g, eps)
        assert contract(got, want) <= 1e-5, s


def test_tensor_solver_matches_fp64(fsk, port, tensor_mode):
    rng = np.random.default_rng(5)
    n, m, d = 700, 650, 64
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d))
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    s = fsk.sinkhorn_solve(X, a, Y, b, eps=0.5, max_iters=10, precision="single", grad=True)
    r = port.sinkhorn_solve(X, a, Y, b, eps=0.5, max_iters=10, precision="double")
    r32 = port.sinkhorn_solve(X, a, Y, b, eps=0.5, max_iters=10, precision="single")
    err = contract(s["f_hat"], r["f_hat"])
    err32 = contract(r32["f_hat"], r["f_hat"])
    assert err <= max(1e-5, 2 * err32)
    assert abs(s["dual_cost"] - r["dual_cost"]) <= 1e-5 * abs(r["dual_cost"])


def test_tensor_solver_eps_scaling(fsk, port, tensor_mode):
    """eps-scaling on the tensor path (operand images and bias rebuilt at every
    eps of the schedule, warm state reset): same eps history as the reference,
    potentials and loss within the fp32 solve contract."""
    rng = np.random.default_rng(8)
    n, m, d = 600, 520, 64
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d)) * 0.9
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    kw = dict(eps=0.3, max_iters=40, eps_scaling_factor=0.7, extra_iters_at_final_eps=5)
    s = fsk.sinkhorn_solve(X, a, Y, b, precision="single", **kw)
    r = port.sinkhorn_solve(X, a, Y, b, precision="double", **kw)
    r32 = port.sinkhorn_solve(X, a, Y, b, precision="single", **kw)
    assert np.array_equal(np.asarray(s["eps_history"]), np.asarray(r["eps_history"]))
    assert s["iterations"] == r["iterations"]
    err = contract(s["f_hat"], r["f_hat"])
    err32 = contract(r32["f_hat"], r["f_hat"])
    print(f"eps-scaled solve: tensor {err:.2e}, reference fp32 {err32:.2e}")
    assert err <= max(1e-5, 2 * err32)
    assert abs(s["dual_cost"] - r["dual_cost"]) <= 1e-5 * abs(r["dual_cost"])


def test_tensor_solver_symmetric_schedule(fsk, port, tensor_mode):
    """Symmetric (Jacobi) schedule on the tensor path: both half-steps from the old
    pair, averaged in the finalize; fp32 solve contract against the reference."""
    rng = np.random.default_rng(9)
    n, m, d = 640, 580, 64
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d)) + 0.1
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    kw = dict(eps=0.4, max_iters=25, schedule="symmetric")
    s = fsk.sinkhorn_solve(X, a, Y, b, precision="single", **kw)
    r = port.sinkhorn_solve(X, a, Y, b, precision="double", **kw)
    r32 = port.sinkhorn_solve(X, a, Y, b, precision="single", **kw)
    err = contract(s["f_hat"], r["f_hat"])
    err32 = contract(r32["f_hat"], r["f_hat"])
    print(f"symmetric solve: tensor {err:.2e}, reference fp32 {err32:.2e}")
    assert err <= max(1e-5, 2 * err32)
    assert abs(s["dual_cost"] - r["dual_cost"]) <= 1e-5 * abs(r["dual_cost"])


def test_engine_row_shards_reproduce_full_half_step(fsk, port):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(11)
    n, m, d = 1100, 900, 64
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d))
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    for mode in ("tensor", "fma"):
        eng = fsk.Engine(0, X, a, Y, b, mode=mode)
        eng.set_eps(0.2)
        f = torch.empty(n, dtype=torch.float32, device="cuda")
        g = torch.empty(m, dtype=torch.float32, device="cuda")
        eng.bind(f.data_ptr(), g.data_ptr())
        eng.init_potentials()
        viol = torch.zeros(1, dtype=torch.float64, device="cuda")
        # f-update in 3 uneven shards, then g-update in 2
        for lo, hi in [(0, 300), (300, 777), (777, n)]:
            eng.half_step(0, lo, hi)
        for lo, hi in [(0, 512), (512, m)]:
            eng.half_step(1, lo, hi)
        torch.cuda.synchronize()
        f0 = -(X ** 2).sum(1)
        g0 = -(Y ** 2).sum(1)
        fw = port.update_f_hat(X, a, Y, b, g0, 0.2)
        gw = port.update_g_hat(X, a, Y, b, fw, 0.2)
        assert contract(f.cpu().numpy(), fw) <= 1e-5, mode
        assert contract(g.cpu().numpy(), gw) <= 1e-5, mode
        # lagged violation from the next f-update equals sum |r - a| of the iterate
        eng.half_step(0, 0, n, viol.data_ptr())
        torch.cuda.synchronize()
        r, c = port.induced_marginals(X, a, Y, b, fw, gw, 0.2)
        want_v = np.abs(r - a).sum()
        assert abs(viol.item() - want_v) <= 2e-2 * want_v + 1e-6, mode
        G = torch.empty((n, d), dtype=torch.float32, device="cuda")
        eng.grad(0, n, G.data_ptr())
        torch.cuda.synchronize()
        eng.close()
        del f0


@pytest.mark.parametrize("n,m,d", [(1000, 777, 64), (515, 1300, 33), (260, 513, 16),
                                   (129, 131, 3), (2048, 4096, 64),
                                   # d > 64: general apply kernel (V = Y) + gradient epilogue
                                   (400, 350, 100), (260, 300, 1024)])
@pytest.mark.parametrize("eps", [0.05, 1.0])
def test_tensor_fused_gradient_parity(fsk, port, n, m, d, eps):
    """Fused tcgen05 transport kernel (K3): grad_X at the engine's own potentials
    against the fp64 SPEC composition 2(diag(r) X - P Y).
    Contract (SURVEY §8d ii): ||dG||_inf <= 1e-5 ||G||_inf."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(n + 3 * m + d)
    X = rng.normal(size=(n, d))
    Y = rng.normal(size=(m, d)) * 0.8 + 0.2
    a = rng.random(n) + 0.5
    a /= a.sum()
    b = np.full(m, 1.0 / m)
    eng = fsk.Engine(0, X, a, Y, b, mode="tensor")
    assert eng.path == "tcgen05-split3"
    eng.set_eps(eps)
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    g = torch.empty(m, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())
    eng.init_potentials()
    for _ in range(3):
        eng.half_step(0, 0, n)
        eng.half_step(1, 0, m)
    G = torch.empty((n, d), dtype=torch.float32, device="cuda")
    eng.grad(0, n, G.data_ptr())
    # a ragged row shard of the same gradient
    lo, hi = 77, min(n, 77 + 300)
    Gs = torch.empty((hi - lo, d), dtype=torch.float32, device="cuda")
    eng.grad(lo, hi, Gs.data_ptr())
    torch.cuda.synchronize()
    fh = f.cpu().numpy().astype(np.float64)
    gh = g.cpu().numpy().astype(np.float64)
    e_gpu, e32, want = grad_errors(port, X, a, Y, b, fh, gh, eps, G.cpu().numpy())
    print(f"grad rel err gpu {e_gpu:.2e} ref-fp32 {e32:.2e}")
    assert e_gpu <= max(1e-5, 2.0 * e32)
    # the row shard reproduces the same rows of the full gradient (to rounding: a
    # ragged shard pairs its query tiles into different units, so the screened
    # live sets and running-max seeds of those rows can differ)
    dsh = np.abs(Gs.cpu().numpy() - G.cpu().numpy()[lo:hi]).max()
    print(f"shard vs full max |diff| {dsh:.3e}")
    assert dsh <= 1e-6 * np.abs(G.cpu().numpy()).max()
    eng.close()


def test_tensor_fused_gradient_cfg2_rows(fsk, port):
    """cfg2 shape (n = m = 65536, d = 64, eps = 0.05): fused gradient on the full
    problem, 256 sampled rows checked against the fp64 composition restricted to
    those rows (rows are independent given the potentials)."""
    torch = pytest.importorskip("torch")
    n = m = 65536
    d, eps = 64, 0.05
    z = fsk.rng_normal(1000, (n + m) * d)
    X, Y = z[: n * d].reshape(n, d), z[n * d:].reshape(m, d)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    eng = fsk.Engine(0, X, a, Y, b, mode="tensor")
    eng.set_eps(eps)
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    g = torch.empty(m, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())
    eng.init_potentials()
    for _ in range(2):
        eng.half_step(0, 0, n)
        eng.half_step(1, 0, m)
    G = torch.empty((n, d), dtype=torch.float32, device="cuda")
    eng.grad(0, n, G.data_ptr())
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(0).choice(n, 256, replace=False))
    fh = f.cpu().numpy().astype(np.float64)
    gh = g.cpu().numpy().astype(np.float64)
    # the oracle on the row slice: G_i is linear in a_i, so renormalise the slice
    # weights (the oracle validates sum(a) = 1) and scale back
    wsum = a[rows].sum()
    got = G.cpu().numpy()[rows] / wsum
    assert np.all(np.isfinite(got))
    e_gpu, e32, _ = grad_errors(port, X[rows], a[rows] / wsum, Y, b, fh[rows], gh, eps, got)
    print(f"cfg2 grad rel err gpu {e_gpu:.2e} ref-fp32 {e32:.2e}")
    assert e_gpu <= max(1e-5, 2.0 * e32)
    eng.close()


@pytest.mark.parametrize("n,m,d", [(700, 513, 64), (300, 421, 100), (515, 260, 33)])
@pytest.mark.parametrize("side", [0, 1])
def test_tensor_transport_vector_parity(fsk, port, n, m, d, side):
    """K1 VEC mode: P v / P^T u on the tensor cores against the fp64 apply_plan /
    apply_plan_adjoint (stream.cpp:324-357) at the engine's potentials. Signed v:
    the bound is relative to (P |v|) so cancellation is not charged to the kernel."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(7 * n + m + d + side)
    X = rng.normal(size=(n, d)) * 0.4
    Y = rng.normal(size=(m, d)) * 0.4 + 0.1
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    eps = 0.5
    eng = fsk.Engine(0, X, a, Y, b, mode="tensor")
    eng.set_eps(eps)
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    g = torch.empty(m, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())
    eng.init_potentials()
    for _ in range(4):
        eng.half_step(0, 0, n)
        eng.half_step(1, 0, m)
    cols, rows = (m, n) if side == 0 else (n, m)
    v = rng.normal(size=cols)
    vd = torch.tensor(v, dtype=torch.float32, device="cuda")
    out = torch.empty(rows, dtype=torch.float64, device="cuda")
    eng.transport_vec(side, vd.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    fh = f.cpu().numpy().astype(np.float64)
    gh = g.cpu().numpy().astype(np.float64)
    v32 = v.astype(np.float32).astype(np.float64)
    fn = port.apply_plan if side == 0 else port.apply_plan_adjoint
    want = fn(X, a, Y, b, fh, gh, eps, v32[:, None])[:, 0]
    scale = fn(X, a, Y, b, fh, gh, eps, np.abs(v32)[:, None])[:, 0]
    err = (np.abs(out.cpu().numpy() - want) / scale).max()
    # as for the gradient, (P v)_i = r_i (P~ v)_i carries the marginal r_i =
    # w_i exp((pot_i - pot+_i)/eps): contract max(1e-5, 2 e32) with e32 the error
    # the reference's own fp32 half-step (stream.cpp:437-451) puts into r
    r64, c64 = port.induced_marginals(X, a, Y, b, fh, gh, eps)
    if side == 0:
        p32 = port.update_f_hat_f32(X, a, Y, b, gh, eps).astype(np.float64)
        m32 = a * np.exp((fh - p32) / eps) / r64
    else:
        p32 = port.update_g_hat_f32(X, a, Y, b, fh, eps).astype(np.float64)
        m32 = b * np.exp((gh - p32) / eps) / c64
    e32 = (np.abs(want * (m32 - 1.0)) / scale).max()
    print(f"transport-vector side {side}: max rel err {err:.2e} (ref-fp32 {e32:.2e})")
    assert err <= max(1e-5, 2.0 * e32)
    eng.close()


@pytest.mark.parametrize("d", [64, 100])
def test_single_precision_hvp_matches_fp64(fsk, port, tensor_mode, d):
    """fsk_hvp_apply_single (tcgen05 transport-vector applies, fp32 matrix applies)
    against the fp64 engine on the same inputs; CG run to convergence in both."""
    rng = np.random.default_rng(d)
    n, m = 400, 300
    X = rng.normal(size=(n, d)) * 0.3
    Y = rng.normal(size=(m, d)) * 0.3 + 0.05
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    eps = 0.5
    s = port.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=200)
    f, g = s["f_hat"], s["g_hat"]
    A = rng.normal(size=X.shape)
    H64, i64 = fsk.hvp_apply(X, a, Y, b, f, g, eps, A, tau=1e-5, cg_tol=1e-9, cg_max_iters=400)
    led = fsk.Ledger()
    H32, i32 = fsk.hvp_apply(X, a, Y, b, f, g, eps, A, tau=1e-5, cg_tol=1e-9, cg_max_iters=400,
                             precision="single", ledger=led)
    rel = np.linalg.norm(H32 - H64) / np.linalg.norm(H64)
    print(f"single-precision HVP d={d}: rel Frobenius {rel:.2e}, CG {i32['cg_iters']} vs "
          f"{i64['cg_iters']}")
    assert rel <= 1e-3
    assert led.transport_vector_applies == 2 * i32["cg_iters"] + 3


@pytest.mark.parametrize("cold_screen", ["0", "1"])
def test_warm_bounds_match_cold_passes(fsk, cold_screen):
    """Warm bounds (gap bounds carried across LSE passes and moved by the bias
    change) only drop blocks provably < 2^-58 of every row's max: 10 iterations +
    gradient agree with FSK_WARM=0 / FSK_SCREEN=0 to fp32 rounding. With
    cold_screen the first pass of each side is screened and its phase 1 seeds the
    gap bounds."""
    torch = pytest.importorskip("torch")
    n = m = 1 << 18
    d, eps = 64, 0.05
    z = fsk.rng_normal(1001, (n + m) * d)
    X, Y = z[: n * d].reshape(n, d), z[n * d:].reshape(m, d)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    out = {}
    for warm in ("1", "0"):
        os.environ["FSK_WARM"] = warm
        os.environ["FSK_SCREEN"] = cold_screen if warm == "1" else "0"
        try:
            eng = fsk.Engine(0, X, a, Y, b, mode="tensor")
            eng.set_eps(eps)
            f = torch.empty(n, dtype=torch.float32, device="cuda")
            g = torch.empty(m, dtype=torch.float32, device="cuda")
            eng.bind(f.data_ptr(), g.data_ptr())
            eng.init_potentials()
            for _ in range(10):
                eng.half_step(0, 0, n)
                eng.half_step(1, 0, m)
            G = torch.empty((n, d), dtype=torch.float32, device="cuda")
            eng.grad(0, n, G.data_ptr())
            torch.cuda.synchronize()
            out[warm] = (f.cpu().numpy(), g.cpu().numpy(), G.cpu().numpy())
            eng.close()
        finally:
            os.environ.pop("FSK_WARM", None)
            os.environ.pop("FSK_SCREEN", None)
    fw, gw, Gw = out["1"]
    fc, gc, Gc = out["0"]
    assert np.abs(fw - fc).max() <= 1e-6 * max(1.0, np.abs(fc).max())
    assert np.abs(gw - gc).max() <= 1e-6 * max(1.0, np.abs(gc).max())
    # warm passes seed each row's running max with a lower bound, which moves the
    # reference point of the online LSE: f and g differ by fp32 rounding, and one
    # ulp of f / eps perturbs every P_ij by that much relative - the gradient
    # (a difference of two such sums) inherits it
    floor = 2.0 ** -23 * max(np.abs(fc).max(), np.abs(gc).max()) / eps
    assert np.abs(Gw - Gc).max() <= max(1e-5, floor) * np.abs(Gc).max()


def test_screened_lse_matches_unscreened(fsk):
    """The 5-MMA screen only drops tiles whose terms are all < 2^-58 of the row max:
    screened and unscreened f/g updates agree to fp32 rounding. n = m = 2^18 at
    eps = 0.05 is concentrated enough for most tiles to be screened out."""
    torch = pytest.importorskip("torch")
    n = m = 1 << 18
    d, eps = 64, 0.05
    z = fsk.rng_normal(1000, (n + m) * d)
    X, Y = z[: n * d].reshape(n, d), z[n * d:].reshape(m, d)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    out = {}
    for flag in ("1", "0"):
        os.environ["FSK_SCREEN"] = flag  # adaptive screening vs the plain kernel
        os.environ["FSK_WARM"] = "0"     # (warm bounds replace the screen when on)
        try:
            eng = fsk.Engine(0, X, a, Y, b, mode="tensor")
            eng.set_eps(eps)
        finally:
            os.environ.pop("FSK_SCREEN", None)
        f = torch.empty(n, dtype=torch.float32, device="cuda")
        g = torch.empty(m, dtype=torch.float32, device="cuda")
        eng.bind(f.data_ptr(), g.data_ptr())
        eng.init_potentials()
        for _ in range(3):
            eng.half_step(0, 0, n)
            eng.half_step(1, 0, m)
        # gradient: with screening its K3 pass streams only the LSE pass's live tiles
        G = torch.empty((n, d), dtype=torch.float32, device="cuda")
        eng.grad(0, n, G.data_ptr())
        torch.cuda.synchronize()
        out[flag] = (f.cpu().numpy(), g.cpu().numpy(), eng.live_tiles(), eng.screened_blocks(),
                     G.cpu().numpy())
        eng.close()
        os.environ.pop("FSK_WARM", None)
    fs, gs, live, blocks, Gs = out["1"]
    fu, gu, live_u, blocks_u, Gu = out["0"]
    assert np.abs(Gs - Gu).max() <= 1e-5 * np.abs(Gu).max()
    assert blocks_u == 0 and blocks > 0
    print(f"screen live fraction {live / blocks:.3f}")
    assert live < blocks
    assert np.abs(fs - fu).max() <= 1e-6 * max(1.0, np.abs(fu).max())
    assert np.abs(gs - gu).max() <= 1e-6 * max(1.0, np.abs(gu).max())


@pytest.mark.parametrize("n,m,d,p", [(700, 513, 64, 64), (300, 421, 100, 130), (515, 260, 33, 1),
                                     (260, 300, 1024, 200)])
@pytest.mark.parametrize("side", [0, 1])
def test_tensor_transport_matrix_parity(fsk, port, n, m, d, p, side):
    """General tcgen05 transport-matrix kernel (any d, any V, p in passes of 128
    columns) against the fp64 apply_plan / apply_plan_adjoint (stream.cpp:324-357),
    with the marginal-scaled contract of the transport-vector test."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3 * n + m + d + p + side)
    X = rng.normal(size=(n, d)) * 0.4
    Y = rng.normal(size=(m, d)) * 0.4 + 0.1
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    eps = 0.5 if d < 512 else 2.0
    eng = fsk.Engine(0, X, a, Y, b, mode="tensor")
    eng.set_eps(eps)
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    g = torch.empty(m, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())
    eng.init_potentials()
    for _ in range(4):
        eng.half_step(0, 0, n)
        eng.half_step(1, 0, m)
    cols, rows = (m, n) if side == 0 else (n, m)
    V = rng.normal(size=(cols, p))
    Vd = torch.tensor(V, dtype=torch.float32, device="cuda")
    out = torch.empty((rows, p), dtype=torch.float32, device="cuda")
    eng.transport_mat(side, Vd.data_ptr(), p, out.data_ptr())
    torch.cuda.synchronize()
    fh = f.cpu().numpy().astype(np.float64)
    gh = g.cpu().numpy().astype(np.float64)
    V32 = V.astype(np.float32).astype(np.float64)
    fn = port.apply_plan if side == 0 else port.apply_plan_adjoint
    want = fn(X, a, Y, b, fh, gh, eps, V32)
    scale = fn(X, a, Y, b, fh, gh, eps, np.abs(V32))
    err = (np.abs(out.cpu().numpy() - want) / scale).max()
    r64, c64 = port.induced_marginals(X, a, Y, b, fh, gh, eps)
    if side == 0:
        p32 = port.update_f_hat_f32(X, a, Y, b, gh, eps).astype(np.float64)
        m32 = a * np.exp((fh - p32) / eps) / r64
    else:
        p32 = port.update_g_hat_f32(X, a, Y, b, fh, eps).astype(np.float64)
        m32 = b * np.exp((gh - p32) / eps) / c64
    e32 = (np.abs(want * (m32 - 1.0)[:, None]) / scale).max()
    print(f"transport-matrix side {side} d={d} p={p}: max rel err {err:.2e} (ref-fp32 {e32:.2e})")
    assert err <= max(1e-5, 2.0 * e32)
    eng.close()


@pytest.mark.parametrize("n,m,d,p", [(700, 513, 64, 64), (300, 421, 100, 130), (260, 300, 1024, 70)])
def test_tensor_transport_hadamard_parity(fsk, port, n, m, d, p):
    """Hadamard mode of the general tensor apply: (P (.) A Y^T) V against the fp64
    apply_hadamard_plan (stream.cpp:359-375, B = Y), marginal-scaled contract."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5 * n + m + d + p)
    X = rng.normal(size=(n, d)) * 0.4
    Y = rng.normal(size=(m, d)) * 0.4 + 0.1
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    eps = 0.5 if d < 512 else 2.0
    eng = fsk.Engine(0, X, a, Y, b, mode="tensor")
    eng.set_eps(eps)
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    g = torch.empty(m, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())
    eng.init_potentials()
    for _ in range(4):
        eng.half_step(0, 0, n)
        eng.half_step(1, 0, m)
    A = rng.normal(size=(n, d))
    V = rng.normal(size=(m, p))
    Ad = torch.tensor(A, dtype=torch.float32, device="cuda")
    Vd = torch.tensor(V, dtype=torch.float32, device="cuda")
    out = torch.empty((n, p), dtype=torch.float32, device="cuda")
    eng.transport_hadamard(Ad.data_ptr(), Vd.data_ptr(), p, out.data_ptr())
    torch.cuda.synchronize()
    fh = f.cpu().numpy().astype(np.float64)
    gh = g.cpu().numpy().astype(np.float64)
    A32 = A.astype(np.float32).astype(np.float64)
    V32 = V.astype(np.float32).astype(np.float64)
    Y32 = Y.astype(np.float32).astype(np.float64)
    want = port.apply_hadamard_plan(X, a, Y, b, fh, gh, eps, A32, Y32, V32)
    # scale: the same plan with |W| |V| (no cancellation charged to the kernel)
    Wabs = np.abs(A32 @ Y32.T)
    r64, _ = port.induced_marginals(X, a, Y, b, fh, gh, eps)
    P = port.apply_plan(X, a, Y, b, fh, gh, eps, np.eye(m)) if m <= 600 else None
    scale = (P * Wabs) @ np.abs(V32)
    err = (np.abs(out.cpu().numpy() - want) / scale).max()
    p32 = port.update_f_hat_f32(X, a, Y, b, gh, eps).astype(np.float64)
    m32 = a * np.exp((fh - p32) / eps) / r64
    e32 = (np.abs(want * (m32 - 1.0)[:, None]) / scale).max()
    print(f"hadamard d={d} p={p}: max rel err {err:.2e} (ref-fp32 {e32:.2e})")
    assert err <= max(1e-5, 2.0 * e32)
    eng.close()


@pytest.fixture()
def graph_path():
    """fsk_engine_iterate on the CUDA graph of per-half-step launches (the persistent
    small-problem kernel disabled)."""
    os.environ["FSK_PERSIST"] = "0"
    yield
    os.environ.pop("FSK_PERSIST", None)


def test_engine_iterate_graph_matches_loop(fsk, graph_path):
    """fsk_engine_iterate (CUDA graph on the CUDA-core path) reproduces the per-call
    half-step loop bit for bit, on first capture and on replay."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(21)
    n, m, d = 1000, 900, 3
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d))
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    s = torch.cuda.Stream()
    res = []
    for use_iterate in (False, True, True):
        eng = fsk.Engine(0, X, a, Y, b, mode="fma")
        eng.set_eps(0.1)
        f = torch.empty(n, dtype=torch.float32, device="cuda")
        g = torch.empty(m, dtype=torch.float32, device="cuda")
        eng.bind(f.data_ptr(), g.data_ptr())
        for rep in range(2):  # second round replays the captured graph
            eng.init_potentials(s.cuda_stream)
            if use_iterate:
                eng.iterate(7, s.cuda_stream)
            else:
                for _ in range(7):
                    eng.half_step(0, 0, n, 0, s.cuda_stream)
                    eng.half_step(1, 0, m, 0, s.cuda_stream)
        s.synchronize()
        res.append((f.cpu().numpy(), g.cpu().numpy()))
        eng.close()
    for fr, gr in res[1:]:
        assert np.array_equal(fr, res[0][0]) and np.array_equal(gr, res[0][1])


def test_engine_iterate_graph_follows_eps_and_rebinding(fsk, graph_path):
    """An eps-annealing loop (set_eps(e_k); iterate(k)) and a rebinding of g must not
    replay a graph captured for the old eps / old buffer: every iterate() equals the
    per-call half-step loop at the current eps and buffers."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(22)
    n, m, d = 800, 700, 3
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d))
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    s = torch.cuda.Stream()

    def run(use_iterate):
        eng = fsk.Engine(0, X, a, Y, b, mode="fma")
        f = torch.empty(n, dtype=torch.float32, device="cuda")
        g = torch.empty(m, dtype=torch.float32, device="cuda")
        g2 = torch.empty(m, dtype=torch.float32, device="cuda")
        eng.bind(f.data_ptr(), g.data_ptr())
        eng.set_eps(1.0)
        eng.init_potentials(s.cuda_stream)
        out = []
        for eps, gbuf in ((1.0, g), (0.5, g), (0.25, g), (0.25, g2)):
            if gbuf is g2:
                g2.copy_(g)
                eng.bind(f.data_ptr(), g2.data_ptr())
            eng.set_eps(eps)
            if use_iterate:
                eng.iterate(3, s.cuda_stream)
            else:
                for _ in range(3):
                    eng.half_step(0, 0, n, 0, s.cuda_stream)
                    eng.half_step(1, 0, m, 0, s.cuda_stream)
            s.synchronize()
            out.append((f.cpu().numpy().copy(), gbuf.cpu().numpy().copy()))
        eng.close()
        return out

    want, got = run(False), run(True)
    for (fw, gw), (fg, gg) in zip(want, got):
        assert np.array_equal(fw, fg) and np.array_equal(gw, gg)


@pytest.mark.parametrize("n,m,d", [(1, 1, 64), (1, 300, 64), (300, 1, 64), (2, 3, 100), (1, 1, 1024),
                                   (127, 129, 65)])
def test_tensor_degenerate_shapes(fsk, port, tensor_mode, n, m, d):
    """Single-point measures and tile-boundary sizes through the tensor kernels
    (half-steps both ways and the gradient) against the fp64 oracle."""
    rng = np.random.default_rng(n * 1000 + m + d)
    X = rng.normal(size=(n, d)) * 0.5
    Y = rng.normal(size=(m, d)) * 0.5
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    g = -(Y ** 2).sum(1)
    eps = 0.5
    want = port.update_f_hat(X, a, Y, b, g, eps)
    got = fsk.update_f_hat_f32(X, a, Y, b, g, eps)
    assert contract(got, want) <= 1e-5
    wg = port.update_g_hat(X, a, Y, b, want, eps)
    gg = fsk.update_g_hat_f32(X, a, Y, b, want, eps)
    assert contract(gg, wg) <= 1e-5
    s = fsk.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=3, precision="single", grad=True)
    r = port.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=3, precision="double")
    assert abs(s["dual_cost"] - r["dual_cost"]) <= 1e-5 * max(1.0, abs(r["dual_cost"]))
    assert np.all(np.isfinite(s["grad"]))


@pytest.mark.parametrize("precision", ["single", "double"])
def test_divergence_batch_matches_single_calls(fsk, precision):
    """fsk_sinkhorn_divergence_batch (uploads each distinct cloud once per call and
    serves repeats from device copies) returns exactly what per-pair
    sinkhorn_divergence calls return; pairs reuse clouds in both roles."""
    rng = np.random.default_rng(11)
    d = 100 if precision == "single" else 8
    clouds = [rng.normal(size=(300 + 37 * i, d)) * (1.0 + 0.1 * i) for i in range(3)]
    ws = [np.full(len(c), 1.0 / len(c)) for c in clouds]
    idx = [(0, 1), (1, 2), (2, 0), (0, 1), (1, 1)]
    pairs = [(clouds[i], ws[i], clouds[j], ws[j]) for i, j in idx]
    got = fsk.sinkhorn_divergence_batch(pairs, eps=0.5, max_iters=8, precision=precision)
    want = [fsk.sinkhorn_divergence(X, a, Y, b, eps=0.5, max_iters=8, precision=precision)
            for X, a, Y, b in pairs]
    assert np.array_equal(got, np.array(want)), (got, want)
    assert got[0] == got[3]


def test_hvp_plan_cache_matches_recomputed_scores(fsk, port):
    """d > 64: the HVP's transport-vector passes sweep the live plan blocks kept in
    HBM (build_plan); with FSK_PLAN_CACHE=0 they recompute the scores. Both runs use
    the same fp32 plan entries, so they agree to accumulation-order rounding."""
    rng = np.random.default_rng(3)
    n, m, d = 700, 650, 100
    X = rng.normal(size=(n, d)) * 0.3
    Y = rng.normal(size=(m, d)) * 0.3 + 0.05
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    eps = 0.5
    s = port.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=100)
    A = rng.normal(size=X.shape)
    out = {}
    for flag in ("1", "0"):
        os.environ["FSK_PLAN_CACHE"] = flag
        try:
            out[flag], _ = fsk.hvp_apply(X, a, Y, b, s["f_hat"], s["g_hat"], eps, A, tau=1e-5,
                                         cg_tol=1e-30, cg_max_iters=30, precision="single")
        finally:
            os.environ.pop("FSK_PLAN_CACHE", None)
    rel = np.linalg.norm(out["1"] - out["0"]) / np.linalg.norm(out["0"])
    print(f"plan cache vs recomputed: rel Frobenius {rel:.2e}")
    assert rel <= 1e-5


@pytest.mark.parametrize("precision", ["double", "single"])
def test_warm_start_continues_the_solve(fsk, precision):
    """f3: fsk_sinkhorn_solve_warm from the potentials of a 10-iteration solve, run
    10 more iterations, is the 20-iteration solve (bit-identical in fp64: same
    kernels, same inputs; single precision to rounding of the skip decisions)."""
    rng = np.random.default_rng(5)
    n, m, d = 3000, 2600, 64
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d)) + 0.1
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    s10 = fsk.sinkhorn_solve(X, a, Y, b, eps=0.1, max_iters=10, precision=precision)
    s20 = fsk.sinkhorn_solve(X, a, Y, b, eps=0.1, max_iters=20, precision=precision, grad=True)
    w = fsk.sinkhorn_solve(X, a, Y, b, eps=0.1, max_iters=10, precision=precision, grad=True,
                           f_init=s10["f_hat"], g_init=s10["g_hat"])
    if precision == "double":
        assert np.array_equal(w["f_hat"], s20["f_hat"]) and np.array_equal(w["g_hat"], s20["g_hat"])
        assert w["dual_cost"] == s20["dual_cost"]
    else:
        assert contract(w["f_hat"], s20["f_hat"]) <= 1e-6
        assert abs(w["dual_cost"] - s20["dual_cost"]) <= 1e-7 * abs(s20["dual_cost"])
    assert np.abs(w["grad"] - s20["grad"]).max() <= 1e-5 * np.abs(s20["grad"]).max()
    with pytest.raises(fsk.ValidationError):
        fsk.sinkhorn_solve(X, a, Y, b, eps=0.1, max_iters=3, f_init=s10["f_hat"])


def test_engine_warm_resolve_runs_no_screened_pass(fsk):
    """f3 on the device engine: continuing a solve from its own potentials (a warm
    re-solve) keeps every LSE pass on the warm bounds - zero screened cold passes -
    while the cold start needed them."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(6)
    n = m = 1 << 17
    d = 64
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d))
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    eng = fsk.Engine(0, X, a, Y, b)
    eng.set_eps(0.05)
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    g = torch.empty(m, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())
    eng.init_potentials()
    eng.iterate(10)
    c0 = eng.pass_counts()
    eng.iterate(10)   # warm re-solve: continue from the current potentials
    c1 = eng.pass_counts()
    torch.cuda.synchronize()
    print(f"cold solve passes {c0}, warm re-solve adds "
          f"{ {k: c1[k] - c0[k] for k in c1} }")
    assert c0["screened"] >= 1
    assert c1["screened"] == c0["screened"]
    assert c1["warm"] - c0["warm"] >= 18
    eng.close()


@pytest.mark.parametrize("n,m", [(20000, 18000), (65536, 65536)])
def test_run_to_run_bit_identical(fsk, n, m):
    """SPEC.md:300 (bit-exact regardless of parallelism): two independent solves +
    gradients of the same problem on the tensor path (screen / warm-bound decisions,
    split partials, fixed-order violation reductions) return identical bits."""
    rng = np.random.default_rng(n)
    X, Y = rng.normal(size=(n, 64)), rng.normal(size=(m, 64))
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    outs = [fsk.sinkhorn_solve(X, a, Y, b, eps=0.05, max_iters=10, precision="single",
                               grad=True) for _ in range(2)]
    for key in ("f_hat", "g_hat", "grad"):
        assert np.array_equal(outs[0][key], outs[1][key]), key
    assert outs[0]["dual_cost"] == outs[1]["dual_cost"]
    assert outs[0]["marginal_violation"] == outs[1]["marginal_violation"]


def test_engine_solves_history_independent(fsk):
    """A solve restarted on the same engine (init_potentials) forgets the warm
    bounds and pass-kind history of the previous solve: the second solve, after a
    different one in between, returns the first one's bits (skip decisions are a
    function of the problem and the pass, not of what ran before)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(77)
    n = m = 1 << 17
    X, Y = rng.normal(size=(n, 64)), rng.normal(size=(m, 64))
    u = np.full(n, 1.0 / n)
    eng = fsk.Engine(0, X, u, Y, u, mode="tensor")
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    g = torch.empty(m, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())
    outs = []
    for eps in (0.05, 0.07, 0.05):
        eng.set_eps(eps)
        eng.init_potentials()
        for _ in range(6):
            eng.half_step(0, 0, n)
            eng.half_step(1, 0, m)
        G = torch.empty((n, 64), dtype=torch.float32, device="cuda")
        eng.grad(0, n, G.data_ptr())
        torch.cuda.synchronize()
        outs.append((f.cpu().numpy().copy(), g.cpu().numpy().copy(), G.cpu().numpy()))
    assert eng.pass_counts()["warm"] > 0
    for a_, b_ in zip(outs[0], outs[2]):
        assert np.array_equal(a_, b_)
    eng.close()


def test_device_decided_passes_match_host_decided(fsk):
    """Large problems decide warm vs cold on the device (no host read-back): the
    same decisions and bits as the host-decided path (FSK_DEVICE_DECIDE=0), and the
    same pass-kind counts."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(404)
    n = m = 1 << 18
    X, Y = rng.normal(size=(n, 64)), rng.normal(size=(m, 64))
    u = np.full(n, 1.0 / n)
    out = {}
    for flag in ("1", "0"):
        os.environ["FSK_DEVICE_DECIDE"] = flag
        try:
            eng = fsk.Engine(0, X, u, Y, u, mode="tensor")
            eng.set_eps(0.05)
            f = torch.empty(n, dtype=torch.float32, device="cuda")
            g = torch.empty(m, dtype=torch.float32, device="cuda")
            eng.bind(f.data_ptr(), g.data_ptr())
            eng.init_potentials()
            for _ in range(8):
                eng.half_step(0, 0, n)
                eng.half_step(1, 0, m)
            G = torch.empty((n, 64), dtype=torch.float32, device="cuda")
            eng.grad(0, n, G.data_ptr())
            torch.cuda.synchronize()
            out[flag] = (f.cpu().numpy(), g.cpu().numpy(), G.cpu().numpy(), eng.pass_counts())
            eng.close()
        finally:
            os.environ.pop("FSK_DEVICE_DECIDE", None)
    for a_, b_ in zip(out["1"][:3], out["0"][:3]):
        assert np.array_equal(a_, b_)
    assert out["1"][3] == out["0"][3]
    assert out["1"][3]["warm"] > 0 and out["1"][3]["screened"] > 0


@pytest.mark.parametrize("switch", ["FSK_LEAN_ISSUE", "FSK_HALF_LOAD"])
def test_issue_and_load_switches_bit_identical(fsk, switch):
    """The d <= 64 kernel's lean MMA-chain issue (one elect per chain, descriptors by
    32-bit adds) and its half-tile key loads (a stage with one needed 64-key half
    loads only that half) change how the same MMAs are issued and fed, not what
    they compute: screened, warm and transport-vector passes and the gradient give
    the same bits with each switch on and off (read per call)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(405)
    n = m = 1 << 18
    X, Y = rng.normal(size=(n, 64)), rng.normal(size=(m, 64))
    u = np.full(n, 1.0 / n)
    v = torch.tensor(rng.normal(size=m), dtype=torch.float32, device="cuda")
    out = {}
    for flag in ("1", "0"):
        os.environ[switch] = flag
        try:
            eng = fsk.Engine(0, X, u, Y, u, mode="tensor")
            eng.set_eps(0.05)
            f = torch.empty(n, dtype=torch.float32, device="cuda")
            g = torch.empty(m, dtype=torch.float32, device="cuda")
            eng.bind(f.data_ptr(), g.data_ptr())
            eng.init_potentials()
            for _ in range(6):
                eng.half_step(0, 0, n)
                eng.half_step(1, 0, m)
            G = torch.empty((n, 64), dtype=torch.float32, device="cuda")
            eng.grad(0, n, G.data_ptr())
            pv = torch.empty(n, dtype=torch.float64, device="cuda")
            eng.transport_vec(0, v.data_ptr(), pv.data_ptr())
            torch.cuda.synchronize()
            out[flag] = (f.cpu().numpy(), g.cpu().numpy(), G.cpu().numpy(), pv.cpu().numpy(),
                         eng.pass_counts())
            eng.close()
        finally:
            os.environ.pop(switch, None)
    for a_, b_ in zip(out["1"][:4], out["0"][:4]):
        assert np.array_equal(a_, b_)
    assert out["1"][4] == out["0"][4]


def test_persistent_small_solve(fsk, port, golden):
    """cfg1-class problems (keys fit in shared memory, d <= 16): the whole iteration
    loop is one cooperative kernel (small_solve.cu). Engine iterate and the drop-in
    single-precision solve against the fp64 oracle / the reference golden cfg1
    (fp32 contract), eps changes and rebinding honoured, and the same iterate as
    the per-launch path to fp32 rounding."""
    torch = pytest.importorskip("torch")
    G = golden
    X, Y = G["cfg1_X"], G["cfg1_Y"]
    n, m = len(X), len(Y)
    u = np.full(n, 1.0 / n)
    s = fsk.sinkhorn_solve(X, u, Y, u, eps=0.1, max_iters=100, precision="single", grad=True)
    assert contract(s["f_hat"], G["cfg1_f"]) <= 1e-5
    assert abs(s["dual_cost"] - G["cfg1_s"][2]) <= 1e-5 * abs(G["cfg1_s"][2])
    eng = fsk.Engine(0, X, u, Y, u, mode="fma")
    f = torch.empty(n, dtype=torch.float32, device="cuda")
    g = torch.empty(m, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())
    ref_f, ref_g = -(X ** 2).sum(1), -(Y ** 2).sum(1)
    eng.init_potentials()
    for eps, its in ((0.5, 4), (0.1, 6)):
        eng.set_eps(eps)
        eng.iterate(its)
        for _ in range(its):
            ref_f = port.update_f_hat(X, u, Y, u, ref_g, eps)
            ref_g = port.update_g_hat(X, u, Y, u, ref_f, eps)
        torch.cuda.synchronize()
        assert contract(f.cpu().numpy(), ref_f) <= 1e-5
        assert contract(g.cpu().numpy(), ref_g) <= 1e-5
    # the per-launch path from the same state agrees to fp32 rounding
    f2, g2 = f.clone(), g.clone()
    eng.iterate(5)
    eng.bind(f2.data_ptr(), g2.data_ptr())
    os.environ["FSK_PERSIST"] = "0"
    try:
        eng.iterate(5)
    finally:
        os.environ.pop("FSK_PERSIST", None)
    torch.cuda.synchronize()
    assert contract(f2.cpu().numpy(), f.cpu().numpy().astype(np.float64)) <= 1e-6
    eng.close()


def _labeled_engine_half_steps(fsk, X, a, Y, b, g0, eps, cost, la, lb, mode):
    torch = pytest.importorskip("torch")
    n, m = len(X), len(Y)
    eng = fsk.Engine(0, X, a, Y, b, mode=mode, cost=cost, la=la, lb=lb)
    eng.set_eps(eps)
    f = torch.zeros(n, dtype=torch.float32, device="cuda")
    g = torch.tensor(g0, dtype=torch.float32, device="cuda")
    eng.bind(f.data_ptr(), g.data_ptr())
    eng.half_step(0, 0, n)
    torch.cuda.synchronize()
    fo = f.cpu().numpy().astype(np.float64)
    eng.half_step(1, 0, m)
    torch.cuda.synchronize()
    go = g.cpu().numpy().astype(np.float64)
    G = torch.empty((n, X.shape[1]), dtype=torch.float32, device="cuda")
    eng.grad(0, n, G.data_ptr())
    torch.cuda.synchronize()
    path = eng.path
    eng.close()
    return fo, go, G.cpu().numpy().astype(np.float64), path


@pytest.mark.parametrize("mode", ["tensor", "fma"])
def test_label_augmented_golden_fp32(fsk, golden, port, mode):
    """f1: the label-augmented cost (stream.cpp:73-77) on the fp32 engine - the tensor
    path applies lambda2 W / eps in the chunked kernels' epilogues - against the
    reference golden f-update (lab_*) at the fp32 contract."""
    G = golden
    cost = dict(lambda1=0.5, lambda2=0.5, label_cost=G["lab_W"])
    fo, go, _, path = _labeled_engine_half_steps(fsk, G["lab_X"], G["lab_a"], G["lab_Y"],
                                                 G["lab_b"], G["lab_g"], 0.25, cost, G["lab_la"],
                                                 G["lab_lb"], mode)
    assert path.startswith("tcgen05" if mode == "tensor" else "fma")
    assert contract(fo, G["lab_out"]) <= 1e-5
    want_g = port.update_g_hat(G["lab_X"], G["lab_a"], G["lab_Y"], G["lab_b"], fo, 0.25,
                               cost=cost, la=G["lab_la"], lb=G["lab_lb"])
    assert contract(go, want_g) <= 1e-5


@pytest.mark.parametrize("n,m,d,V", [(600, 520, 784, 10), (700, 333, 64, 5), (300, 257, 100, 64)])
def test_label_augmented_tensor_path_vs_oracle(fsk, port, n, m, d, V):
    """Labelled OTDD-style problems (d = 784 as cfg5, 10 classes; ragged shapes; V = 64,
    the table limit) on the tensor path: both half-steps against the port (fp32
    contract) and the gradient rows against the SPEC composition on the port's
    labelled transport (the stated tensor-mode gradient bound)."""
    from oracle import compose
    rng = np.random.default_rng(n + V)
    X = rng.normal(size=(n, d)) * 0.1
    Y = rng.normal(size=(m, d)) * 0.1 + 0.01
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    la, lb = rng.integers(0, V, n), rng.integers(0, V, m)
    W = rng.random((V, V)) * 2.0
    cost = dict(lambda1=0.8, lambda2=0.6, label_cost=W)
    eps = 0.5
    g0 = -0.8 * (Y ** 2).sum(1)
    fo, go, Gg, path = _labeled_engine_half_steps(fsk, X, a, Y, b, g0, eps, cost, la, lb, "tensor")
    assert path.startswith("tcgen05")
    fw = port.update_f_hat(X, a, Y, b, g0, eps, cost=cost, la=la, lb=lb)
    assert contract(fo, fw) <= 1e-5
    gw = port.update_g_hat(X, a, Y, b, fo, eps, cost=cost, la=la, lb=lb)
    assert contract(go, gw) <= 1e-5
    # gradient at the engine's potentials (fo, go): SPEC grad_source, G = 2 (diag(r) X - P Y)
    # (the convention of fsk_grad_source for every cost)
    f64, g64 = fo, go

    class LabOps:
        def __getattr__(self, name):
            fn = getattr(port, name)
            return lambda *args, **kw: fn(*args, cost=cost, la=la, lb=lb, **kw)

    ws = compose.Workspace(LabOps(), X, a, Y, b, f64, g64, eps)
    G64 = compose.grad_source(ws)
    err = np.abs(Gg - G64).max() / np.abs(G64).max()
    print(f"labelled n={n} m={m} d={d} V={V}: f {contract(fo, fw):.2e} g {contract(go, gw):.2e} "
          f"grad {err:.2e}")
    assert err <= 1e-4
