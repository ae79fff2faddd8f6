"""SPEC compositions the reference never implemented, built from its stream ops.

TEST INFRASTRUCTURE ONLY. The reference ships no gradient / HVP code
(SURVEY.md §0 finding 5); SPEC.md prescribes them as compositions of the
streaming operators. These restatements run over an ``oracle.Oracle`` backend
and are the parity targets for the product's fused CUDA implementations:

  barycentric_projection, grad_source, grad_target   <- SPEC.md:378-430 (autodiff)
  explicit_term, build_rhs, schur_apply, cg_solve,
  hvp_apply                                          <- SPEC.md:432-542 (hvp),
                                                        PAPER.md:1242-1462 (Thm. 3.5)
"""
from __future__ import annotations

import numpy as np


class Workspace:
    """HvpWorkspace: cached P Y and induced marginals."""

    def __init__(self, ops, X, a, Y, b, f_hat, g_hat, eps, tiles=(64, 64)):
        self.ops, self.X, self.a, self.Y, self.b = ops, X, a, Y, b
        self.f, self.g, self.eps, self.tiles = f_hat, g_hat, eps, tiles
        self.PY = ops.apply_plan(X, a, Y, b, f_hat, g_hat, eps, Y, tiles)
        self.r, self.c = ops.induced_marginals(X, a, Y, b, f_hat, g_hat, eps, tiles)
        self.counts = dict(vector=1 if Y.shape[1] == 1 else 0, matrix=0 if Y.shape[1] == 1 else 1,
                           hadamard=0)

    def P(self, V):
        V = np.asarray(V, dtype=np.float64)
        v1 = V.ndim == 1
        out = self.ops.apply_plan(self.X, self.a, self.Y, self.b, self.f, self.g, self.eps,
                                  V[:, None] if v1 else V, self.tiles)
        self.counts["vector" if (v1 or V.shape[1] == 1) else "matrix"] += 1
        return out[:, 0] if v1 else out

    def Pt(self, U):
        U = np.asarray(U, dtype=np.float64)
        v1 = U.ndim == 1
        out = self.ops.apply_plan_adjoint(self.X, self.a, self.Y, self.b, self.f, self.g,
                                          self.eps, U[:, None] if v1 else U, self.tiles)
        self.counts["vector" if (v1 or U.shape[1] == 1) else "matrix"] += 1
        return out[:, 0] if v1 else out


def barycentric_projection(ws: Workspace):
    """T = diag(r)^-1 P Y."""
    return ws.PY / ws.r[:, None]


def grad_source(ws: Workspace):
    """G = 2 (diag(r) X - P Y)."""
    return 2.0 * (ws.r[:, None] * ws.X - ws.PY)


def grad_target(ws: Workspace):
    """G = 2 (diag(c) Y - P^T X)."""
    return 2.0 * (ws.c[:, None] * ws.Y - ws.Pt(ws.X))


def explicit_term(ws: Workspace, A):
    """E.A = B1 - (4/eps)(B2 - B3 - B4 + B5)."""
    X, PY, r, eps = ws.X, ws.PY, ws.r, ws.eps
    u = (X * A).sum(1)
    uP = (PY * A).sum(1)
    B5 = ws.ops.apply_hadamard_plan(ws.X, ws.a, ws.Y, ws.b, ws.f, ws.g, eps, A, ws.Y, ws.Y,
                                    ws.tiles)
    ws.counts["hadamard"] += 1
    return 2.0 * r[:, None] * A - (4.0 / eps) * ((r * u)[:, None] * X - u[:, None] * PY
                                                  - uP[:, None] * X + B5)


def build_rhs(ws: Workspace, A):
    """r1 = 2 (r u - u_P), r2 = 2 (P^T u - <P^T A, Y>_row)."""
    u = (ws.X * A).sum(1)
    uP = (ws.PY * A).sum(1)
    r1 = 2.0 * (ws.r * u - uP)
    r2 = 2.0 * (ws.Pt(u) - (ws.Pt(A) * ws.Y).sum(1))
    return r1, r2


def schur_apply(ws: Workspace, v, tau):
    """S_tau v = c v - P^T diag(r)^-1 P v + tau v."""
    return ws.c * v - ws.Pt(ws.P(v) / ws.r) + tau * v


def cg_solve(apply, rhs, tol=1e-6, max_iters=50):
    """Unpreconditioned CG from 0. Returns (x, iters, rel_residual)."""
    x = np.zeros_like(rhs)
    rnorm0 = np.linalg.norm(rhs)
    if rnorm0 == 0.0:
        return x, 0, 0.0
    res = rhs.copy()
    p = res.copy()
    rs = res @ res
    it = 0
    while it < max_iters:
        Ap = apply(p)
        alpha = rs / (p @ Ap)
        x += alpha * p
        res -= alpha * Ap
        it += 1
        rs_new = res @ res
        if np.sqrt(rs_new) <= tol * rnorm0:
            break
        p = res + (rs_new / rs) * p
        rs = rs_new
    return x, it, float(np.sqrt(res @ res) / rnorm0)


def hvp_apply(ws: Workspace, A, tau=1e-5, tol=1e-6, max_iters=50):
    """G = (1/eps) R^T w + E.A (Thm. 3.5)."""
    A = np.asarray(A, dtype=np.float64)
    r1, r2 = build_rhs(ws, A)
    rhs = r2 - ws.Pt(r1 / ws.r)
    w2, iters, res = cg_solve(lambda v: schur_apply(ws, v, tau), rhs, tol, max_iters)
    Pw2 = ws.P(w2)
    w1 = (r1 - Pw2) / ws.r
    RTw = 2.0 * ((ws.r * w1)[:, None] * ws.X - w1[:, None] * ws.PY + Pw2[:, None] * ws.X
                 - ws.P(w2[:, None] * ws.Y))
    return RTw / ws.eps + explicit_term(ws, A), iters, res
