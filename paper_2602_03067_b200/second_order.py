"""Second-order consumers of the HVP.

lanczos_min_eig  restarted Lanczos with full reorthogonalisation for the smallest
                 algebraic eigenvalue of a symmetric operator given as a matvec
                 (the paper's "coarse diagnostic" of the parameter Hessian,
                 Appendix H.3); every matvec is one streaming HVP on the GPU.
parameter_hvp    H_W v = X^T T(X v) for the shuffled-regression parameterisation
                 Y_hat = X W (§4.2): lift, data-space HVP, project.
"""
from __future__ import annotations

import numpy as np


def lanczos_min_eig(matvec, dim: int, subspace: int = 6, tol: float = 1e-8,
                    max_restarts: int = 200, seed: int = 0) -> float:
    """Smallest algebraic eigenvalue of a symmetric operator (SPEC lanczos_min_eig).

    Each cycle builds an orthonormal Krylov basis of size `subspace` from the
    current start vector (full reorthogonalisation, one matvec per basis vector,
    the products kept for the Rayleigh-Ritz step), takes the smallest Ritz pair
    and restarts from its Ritz vector until ||A u - theta u|| <= tol max(1, |theta|).
    A breakdown (invariant subspace) ends the cycle early; a degenerate start
    restarts from a new seeded random vector."""
    rng = np.random.default_rng(seed)
    k = max(1, min(subspace, dim))
    v = rng.standard_normal(dim)
    v /= np.linalg.norm(v)
    theta = np.inf
    for _ in range(max_restarts):
        V = np.zeros((dim, k))
        AV = np.zeros((dim, k))
        V[:, 0] = v
        m = k
        for j in range(k):
            AV[:, j] = np.asarray(matvec(V[:, j]), dtype=np.float64)
            if j + 1 == k:
                break
            w = AV[:, j].copy()
            for _ in range(2):  # full reorthogonalisation (twice is enough)
                w -= V[:, : j + 1] @ (V[:, : j + 1].T @ w)
            beta = np.linalg.norm(w)
            if beta <= 1e-12 * max(1.0, np.linalg.norm(AV[:, j])):
                m = j + 1
                break
            V[:, j + 1] = w / beta
        H = V[:, :m].T @ AV[:, :m]
        evals, evecs = np.linalg.eigh(0.5 * (H + H.T))
        theta = float(evals[0])
        u = V[:, :m] @ evecs[:, 0]
        r = AV[:, :m] @ evecs[:, 0] - theta * u
        if np.linalg.norm(r) <= tol * max(1.0, abs(theta)) or m == dim:
            return theta
        nu = np.linalg.norm(u)
        v = u / nu if np.isfinite(nu) and nu > 1e-14 else rng.standard_normal(dim)
        v /= np.linalg.norm(v)
    return theta


def parameter_hvp(X_design, data_hvp, v):
    """H_W v = X^T T(X v) (SPEC parameter_hvp): v is d x p flattened, X_design
    n x d, data_hvp maps an n x p data-space direction to its HVP."""
    X = np.asarray(X_design, dtype=np.float64)
    d = X.shape[1]
    V = np.asarray(v, dtype=np.float64).reshape(d, -1)
    return (X.T @ np.asarray(data_hvp(X @ V), dtype=np.float64)).reshape(-1)
