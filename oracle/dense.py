"""Numpy restatement of the reference dense backend (proj/src/dense.cpp).

TEST INFRASTRUCTURE ONLY (desk-scale oracle). dense.cpp needs Eigen3 (absent),
so it cannot be compiled here; this restatement follows it line by line and
uses numpy.linalg.eigh in place of Eigen::SelfAdjointEigenSolver for the
Hessian pseudo-inverse (dense.cpp:210-218). That is the only third-party
arithmetic on the path (Eigen3 >= 3.3, version unpinned by
proj/CMakeLists.txt:19); the restatement is anchored on the published formula
(SPEC.md dense_hessian, Appendix C) and cross-checked against the
streaming SPEC composition in tests.
"""
from __future__ import annotations

import numpy as np


def dense_cost(X, Y, cost=None, la=None, lb=None):
    """dense.cpp:68-89."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    diff = X[:, None, :] - Y[None, :, :]
    C = np.einsum("ijt,ijt->ij", diff, diff)
    if cost is not None:
        W = np.asarray(cost["label_cost"])
        C = cost["lambda1"] * C + cost["lambda2"] * W[np.asarray(la)[:, None], np.asarray(lb)[None, :]]
    return C


def _row_lse(z):
    mx = z.max(axis=1, keepdims=True)
    return (mx + np.log(np.exp(z - mx).sum(axis=1, keepdims=True)))[:, 0]


def dense_sinkhorn(X, a, Y, b, eps=0.1, schedule="alternating", max_iters=100, cost=None,
                   la=None, lb=None):
    """dense.cpp:91-135 (flat eps schedule, no tolerance). Returns shifted (f_hat, g_hat)."""
    C = dense_cost(X, Y, cost, la, lb)
    loga, logb = np.log(a), np.log(b)
    f = np.zeros(len(a))
    g = np.zeros(len(b))
    for _ in range(max_iters):
        if schedule == "alternating":
            f = -eps * _row_lse((g[None, :] - C) / eps + logb[None, :])
            g = -eps * _row_lse(((f[:, None] - C) / eps + loga[:, None]).T)
        else:
            fn = 0.5 * f - 0.5 * eps * _row_lse((g[None, :] - C) / eps + logb[None, :])
            gn = 0.5 * g - 0.5 * eps * _row_lse(((f[:, None] - C) / eps + loga[:, None]).T)
            f, g = fn, gn
    s = 1.0 if cost is None else cost["lambda1"]
    alpha = s * (np.asarray(X) ** 2).sum(1)
    beta = s * (np.asarray(Y) ** 2).sum(1)
    return f - alpha, g - beta


def dense_plan(X, a, Y, b, f_hat, g_hat, eps, cost=None, la=None, lb=None):
    """dense.cpp:142-164: P_ij = a_i b_j exp((f_i + g_j - C_ij)/eps), unshifted potentials."""
    C = dense_cost(X, Y, cost, la, lb)
    s = 1.0 if cost is None else cost["lambda1"]
    f = np.asarray(f_hat) + s * (np.asarray(X) ** 2).sum(1)
    g = np.asarray(g_hat) + s * (np.asarray(Y) ** 2).sum(1)
    P = np.asarray(a)[:, None] * np.asarray(b)[None, :] * np.exp((f[:, None] + g[None, :] - C) / eps)
    if not np.all(np.isfinite(P)):
        raise FloatingPointError("dense_plan overflow, potentials are not stabilized")
    return P


def dense_gradient(X, Y, P):
    """dense.cpp:166-183: G = 2 (diag(P 1) X - P Y)."""
    return 2.0 * (P.sum(1)[:, None] * np.asarray(X) - P @ np.asarray(Y))


def dense_hessian(X, Y, P, eps, pinv_threshold=1e-10):
    """dense.cpp:185-265: (1/eps) R^T H^+ R + E, stored (n d) x (n d)."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    n, d = X.shape
    m = Y.shape[0]
    if n > 512 or m > 512:
        raise ValueError("dense_hessian is desk-scale only (n, m <= 512)")
    r = P.sum(1)
    c = P.sum(0)
    H = np.zeros((n + m, n + m))
    H[np.arange(n), np.arange(n)] = r
    H[n + np.arange(m), n + np.arange(m)] = c
    H[:n, n:] = P
    H[n:, :n] = P.T
    evals, evecs = np.linalg.eigh(H)
    lmax = np.abs(evals).max()
    inv = np.where(evals > pinv_threshold * lmax, 1.0 / np.where(evals == 0, 1, evals), 0.0)
    Hdag = (evecs * inv) @ evecs.T
    PY = P @ Y
    R = np.zeros((n + m, n * d))
    for k in range(n):
        R[k, k * d:(k + 1) * d] = 2.0 * (X[k] * r[k] - PY[k])
    for k in range(n):
        # R(n+j, k*d+t) = 2 (x_kt - y_jt) P_kj
        R[n:, k * d:(k + 1) * d] = 2.0 * (X[k][None, :] - Y) * P[k][:, None]
    T = R.T @ (Hdag @ R) / eps
    for k in range(n):
        diff = X[k][None, :] - Y  # m x d
        blk = -(4.0 / eps) * np.einsum("j,jt,jl->tl", P[k], diff, diff)
        blk[np.arange(d), np.arange(d)] += 2.0 * r[k]
        T[k * d:(k + 1) * d, k * d:(k + 1) * d] += blk
    return T


def dense_hvp(T, A):
    """dense.cpp:267-279."""
    A = np.asarray(A, dtype=np.float64)
    return (T @ A.reshape(-1)).reshape(A.shape)


def dense_primal_objective(X, a, Y, b, P, eps, cost=None, la=None, lb=None):
    """dense.cpp:281-295: <C,P> + eps KL(P || a (x) b)."""
    C = dense_cost(X, Y, cost, la, lb)
    ab = np.asarray(a)[:, None] * np.asarray(b)[None, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        kl = np.where(P > 0, P * np.log(P / ab) - P + ab, ab)
    return float((C * P).sum() + eps * kl.sum())


class DenseOps:
    """The stream-op interface of ``oracle.Oracle`` (apply_plan, apply_plan_adjoint,
    apply_hadamard_plan, induced_marginals) over the materialised fp64 plan
    P_ij = a_i b_j exp((f_i + g_j + 2 <x_i, y_j>)/eps) (shifted potentials,
    stream.cpp:140-207 / :377-404 evaluated densely), so ``compose.Workspace`` /
    ``compose.hvp_apply`` run at d = 1024 in seconds where the streaming port's
    per-column transport (stream.cpp:182-186) would take hours. Pinned against the
    port in tests/test_oracle.py. Squared-Euclidean cost only."""

    def __init__(self, fp32_scores=False):
        # fp32_scores="reference": S_ij evaluated in the reference's single-precision
        # arithmetic and order (make_ctx_f32 stream.cpp:421-434 + score_tile
        # stream.cpp:61-79 over float: keys x (2.0f/eps), bias (g + eps logf(w))/eps
        # first, then += x_t * k_t sequentially in t, each product and sum rounded to
        # fp32, no FMA), the rest in fp64. The HVP on that plan is what the reference's
        # own fp32 arithmetic does to the result: the "e32" of the tensor-mode bounds.
        # fp32_scores=True: the same in fp32 BLAS order (sgemm), a milder variant.
        self.fp32_scores = fp32_scores

    def _plan(self, X, a, Y, b, f_hat, g_hat, eps):
        X = np.asarray(X, dtype=np.float64)
        Y = np.asarray(Y, dtype=np.float64)
        key = (id(X), id(Y), id(f_hat), id(g_hat), float(eps))
        if getattr(self, "_key", None) != key:
            if self.fp32_scores == "reference":
                e32 = np.float32(eps)
                k32 = Y.astype(np.float32) * (np.float32(2.0) / e32)
                bias32 = (np.asarray(g_hat).astype(np.float32) +
                          e32 * np.log(np.asarray(b).astype(np.float32))) / e32
                S32 = np.empty((X.shape[0], Y.shape[0]), dtype=np.float32)
                S32[:] = bias32[None, :]
                X32 = X.astype(np.float32)
                prod = np.empty_like(S32)
                for t in range(X.shape[1]):
                    np.multiply.outer(X32[:, t], k32[:, t], out=prod)
                    S32 += prod
                S = S32.astype(np.float64)
                S += (np.asarray(f_hat, dtype=np.float64) / eps + np.log(a))[:, None]
            elif self.fp32_scores:
                k32 = Y.astype(np.float32) * np.float32(2.0 / eps)
                bias32 = ((np.asarray(g_hat).astype(np.float32) +
                           np.float32(eps) * np.log(np.asarray(b).astype(np.float32))) /
                          np.float32(eps)).astype(np.float32)
                S = ((X.astype(np.float32) @ k32.T) + bias32[None, :]).astype(np.float64)
                S += (np.asarray(f_hat, dtype=np.float64) / eps + np.log(a))[:, None]
            else:
                S = (2.0 / eps) * (X @ Y.T)
                S += (np.asarray(f_hat, dtype=np.float64) / eps + np.log(a))[:, None]
                S += (np.asarray(g_hat, dtype=np.float64) / eps + np.log(b))[None, :]
            self._P = np.exp(S)
            if not np.all(np.isfinite(self._P)):
                raise FloatingPointError("dense plan overflow, potentials are not stabilized")
            self._key = key
            self._refs = (X, Y, f_hat, g_hat)   # keep the ids alive while cached
        return self._P

    def apply_plan(self, X, a, Y, b, f_hat, g_hat, eps, V, tiles=None):
        return self._plan(X, a, Y, b, f_hat, g_hat, eps) @ np.asarray(V, dtype=np.float64)

    def apply_plan_adjoint(self, X, a, Y, b, f_hat, g_hat, eps, U, tiles=None):
        return self._plan(X, a, Y, b, f_hat, g_hat, eps).T @ np.asarray(U, dtype=np.float64)

    def apply_hadamard_plan(self, X, a, Y, b, f_hat, g_hat, eps, A, B, V, tiles=None):
        P = self._plan(X, a, Y, b, f_hat, g_hat, eps)
        return (P * (np.asarray(A) @ np.asarray(B).T)) @ np.asarray(V, dtype=np.float64)

    def induced_marginals(self, X, a, Y, b, f_hat, g_hat, eps, tiles=None):
        P = self._plan(X, a, Y, b, f_hat, g_hat, eps)
        return P.sum(1), P.sum(0)
