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


@pytest.fixture()
def tensor_mode():
    os.environ["FSK_TENSOR_MODE"] = "tensor"
    yield
    os.environ.pop("FSK_TENSOR_MODE", None)


@pytest.mark.parametrize("n,m,d", [(128, 128, 64), (384, 320, 64), (1000, 777, 64),
                                   (515, 1300, 33), (260, 513, 16), (129, 131, 3)])
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
