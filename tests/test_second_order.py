"""lanczos_min_eig / parameter_hvp."""
import numpy as np
import pytest

from paper_2602_03067_b200.second_order import lanczos_min_eig, parameter_hvp


def test_lanczos_diagonal_operator():
    diag = np.arange(1.0, 41.0)
    assert abs(lanczos_min_eig(lambda v: diag * v, 40, tol=1e-10) - 1.0) <= 1e-8


def test_lanczos_seeded_symmetric_and_negation():
    rng = np.random.default_rng(4)
    A = rng.normal(size=(32, 32))
    A = A + A.T
    want = np.linalg.eigvalsh(A)
    got = lanczos_min_eig(lambda v: A @ v, 32, subspace=8, tol=1e-10, max_restarts=2000)
    assert abs(got - want[0]) <= 1e-6 * max(1.0, abs(want[0]))
    neg = lanczos_min_eig(lambda v: -(A @ v), 32, subspace=8, tol=1e-10, max_restarts=2000)
    assert abs(neg + want[-1]) <= 1e-6 * max(1.0, abs(want[-1]))


def test_parameter_hvp_lift_project():
    rng = np.random.default_rng(1)
    X = rng.normal(size=(8, 2))
    T = rng.normal(size=(8, 8))
    T = T @ T.T
    hv = lambda U: T @ U  # a data-space operator acting column-wise
    v = rng.normal(size=(2, 2))
    assert np.allclose(parameter_hvp(X, hv, v), (X.T @ T @ X @ v).reshape(-1))
    assert np.allclose(parameter_hvp(X, hv, np.zeros(4)), 0.0)
    u = rng.normal(size=4)
    w = rng.normal(size=4)
    assert abs(parameter_hvp(X, hv, u) @ w - parameter_hvp(X, hv, w) @ u) <= 1e-10


@pytest.mark.gpu
def test_lanczos_on_streaming_hvp_matches_dense_hessian(fsk, port):
    """lambda_min of the streaming HVP (GPU, fp64) against the dense Hessian
    (the eigh restatement of dense.cpp:185-265) at desk scale."""
    from oracle import dense
    from oracle.rng import Rng, random_measure
    rng = Rng(17)
    X, a = random_measure(rng, 24, 2, False)
    Y, b = random_measure(rng, 20, 2, False)
    eps = 0.5
    s = port.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=3000, marginal_tol=1e-12)
    f, g = s["f_hat"], s["g_hat"]
    H = dense.dense_hessian(X, Y, dense.dense_plan(X, a, Y, b, f, g, eps), eps)
    want = np.linalg.eigvalsh(0.5 * (H + H.T))[0]
    mv = lambda v: fsk.hvp_apply(X, a, Y, b, f, g, eps, v.reshape(X.shape), tau=0.0,
                                 cg_tol=1e-12, cg_max_iters=500)[0].reshape(-1)
    got = lanczos_min_eig(mv, X.size, subspace=X.size, tol=1e-9, max_restarts=5)
    assert abs(got - want) <= 1e-6 * max(1.0, abs(want))
