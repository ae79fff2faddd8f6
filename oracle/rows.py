"""Row-sliced fp64 restatements for parity checks at benchmark sizes.

TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py's parity
check after the timed region). Never on the product path.

At n = m = 2^20 the full oracle is hours of CPU time, but every row of a
half-step / transport output depends only on its own query point and the whole
key side ("a sliced update_f_hat is bit-identical to the
same rows of a full run"). So parity at the benchmarked configuration checks a
random sample of rows:

* half-step rows: ``Oracle("port").update_f_hat`` / ``update_g_hat`` on the row
  slice (weights of the query slice renormalised: they do not enter the
  half-step, stream.cpp:209-251), bit-identical to the reference on those rows;
* transport rows: ``transport_rows`` below, a numpy fp64 restatement of
  apply_core (stream.cpp:140-207) over key chunks - out_i = a_i e^{f_i/eps + m_i}
  sum_j e^{S_ij - m_i} V_j with S_ij = (2/eps)<x_i, y_j> + (g_j + eps log b_j)/eps.
  Not bit-faithful (BLAS order, numpy exp), fp64-accurate (~1e-13 relative), which
  is all a 1e-5 contract needs; pinned against the port in tests/test_oracle.py;
* gradient rows: SPEC grad_source composed from those,
  G_i = 2 (r_i x_i - (P Y)_i), r_i = a_i exp((f_i - f+_i)/eps) (stream.cpp:377-404).
"""
from __future__ import annotations

import numpy as np


def slice_weights(k: int) -> np.ndarray:
    """Uniform weights for a k-row query slice whose naive sum passes the reference's
    |sum - 1| <= 1e-12 validation (core.cpp:27-33)."""
    w = np.full(k, 1.0 / k)
    if k > 1:
        w[-1] = 1.0 - np.cumsum(w[:-1])[-1]
    return w


def half_step_rows(port, side, X, a, Y, b, pot_other, eps, rows):
    """Rows `rows` of update_f_hat (side 0: rows of X, keys Y, pot_other = g) or
    update_g_hat (side 1: rows of Y, keys X, pot_other = f), through the C port."""
    rows = np.asarray(rows)
    w = slice_weights(len(rows))
    if side == 0:
        return port.update_f_hat(X[rows], w, Y, b, pot_other, eps)
    return port.update_g_hat(X, a, Y[rows], w, pot_other, eps)


def transport_rows(Xr, ar, fr, Y, b, g, eps, V, chunk=1 << 15):
    """(P V)[rows] in fp64 (apply_core, stream.cpp:140-207), keys streamed in chunks
    with the same online max rescaling as the reference."""
    Xr = np.asarray(Xr, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    V2 = V[:, None] if V.ndim == 1 else V
    R, m = Xr.shape[0], Y.shape[0]
    bias = (np.asarray(g, dtype=np.float64) + eps * np.log(np.asarray(b, dtype=np.float64))) / eps
    mrow = np.full(R, -np.inf)
    acc = np.zeros((R, V2.shape[1]))
    for j0 in range(0, m, chunk):
        j1 = min(m, j0 + chunk)
        S = Xr @ (Y[j0:j1] * (2.0 / eps)).T + bias[j0:j1][None, :]
        mnew = np.maximum(mrow, S.max(1))
        acc *= np.exp(mrow - mnew)[:, None]
        acc += np.exp(S - mnew[:, None]) @ V2[j0:j1]
        mrow = mnew
    out = (np.asarray(ar, dtype=np.float64) * np.exp(np.asarray(fr) / eps + mrow))[:, None] * acc
    return out[:, 0] if V.ndim == 1 else out


def grad_rows(port, X, a, Y, b, f, g, eps, rows):
    """SPEC grad_source on the rows `rows` of X:
    G_i = 2 (r_i x_i - (P Y)_i) with r_i = a_i exp((f_i - f+_i)/eps)."""
    rows = np.asarray(rows)
    f = np.asarray(f, dtype=np.float64)
    fplus = half_step_rows(port, 0, X, a, Y, b, g, eps, rows)
    r = a[rows] * np.exp((f[rows] - fplus) / eps)
    PY = transport_rows(X[rows], a[rows], f[rows], Y, b, g, eps, Y)
    return 2.0 * (r[:, None] * X[rows] - PY), r, fplus


def grad_rows_fp32_error(port, X, a, Y, b, f, g, eps, rows, G64, r64, PY=None):
    """The error the reference's own fp32 half-step (update_f_hat_f32,
    stream.cpp:437-443) puts into the same gradient rows through r: e32 =
    ||G32 - G64||_inf / ||G64||_inf with f+ from the fp32 path, P Y in fp64
    (the tensor-mode gradient contract)."""
    rows = np.asarray(rows)
    w = slice_weights(len(rows))
    fp32 = port.update_f_hat_f32(X[rows], w, Y, b, g, eps).astype(np.float64)
    r32 = a[rows] * np.exp((np.asarray(f, dtype=np.float64)[rows] - fp32) / eps)
    PYr = (G64 / -2.0 + r64[:, None] * X[rows]) if PY is None else PY
    G32 = 2.0 * (r32[:, None] * X[rows] - (r32 / r64)[:, None] * PYr)
    return np.abs(G32 - G64).max() / np.abs(G64).max()
