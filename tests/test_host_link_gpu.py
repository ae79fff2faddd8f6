"""Host link of the single-precision solve entry points (C ABI, host buffers).

* Device ingest (DevProblem::ingest): the caller's doubles are narrowed on the
  device, which also runs validate_measure's coordinate finiteness scan and forms
  alpha = |x|^2, beta = |y|^2 and the initial potentials (solver.cpp:27-32). Its
  results are bit-identical to the host path (FSK_DEVICE_INGEST=0), and the
  deferred scan raises the reference's error in the reference's order
  (core.cpp:18-81: the first failing check of source, then target, then config).
* Page-locked buffers (fsk_host_alloc pool): pinned inputs and outputs move by one
  DMA and give the same bits as pageable ones.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fsk():
    import paper_2602_03067_b200 as m
    if m.lib().fsk_device_count() < 1:
        pytest.skip("no CUDA device")
    return m


def _problem(n, m, d, seed=5):
    rng = np.random.default_rng(seed)
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d))
    return X, np.full(n, 1.0 / n), Y, np.full(m, 1.0 / m)


@pytest.mark.parametrize("n,m,d,eps,iters", [(4096, 4096, 3, 0.1, 30),     # persistent small solve
                                             (3000, 2500, 64, 0.05, 8),    # tensor path
                                             (1 << 17, 1 << 17, 64, 0.05, 6)])  # staged sizes
def test_device_ingest_matches_host_path(fsk, monkeypatch, n, m, d, eps, iters):
    X, a, Y, b = _problem(n, m, d)
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("FSK_DEVICE_INGEST", flag)
        outs.append(fsk.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=iters, precision="single",
                                       grad=True))
    for key in ("f_hat", "g_hat", "grad"):
        assert np.array_equal(outs[0][key], outs[1][key]), key
    assert outs[0]["dual_cost"] == outs[1]["dual_cost"]
    assert outs[0]["marginal_violation"] == outs[1]["marginal_violation"]


def test_pinned_buffers_same_bits(fsk):
    X, a, Y, b = _problem(1 << 16, 1 << 16, 64, seed=9)
    ref = fsk.sinkhorn_solve(X, a, Y, b, eps=0.05, max_iters=5, precision="single", grad=True)
    Xp, Yp, ap, bp = (fsk.pinned_copy(v) for v in (X, Y, a, b))
    out = fsk.sinkhorn_solve(Xp, ap, Yp, bp, eps=0.05, max_iters=5, precision="single", grad=True)
    for key in ("f_hat", "g_hat", "grad"):
        assert np.array_equal(ref[key], out[key]), key
    assert ref["dual_cost"] == out["dual_cost"]
    # outputs of >= 8 MB come from the pinned pool; the block returns to it on release
    G = out["grad"]
    assert G.nbytes >= (8 << 20) and G.base is not None
    del out, G


def test_pinned_pool_roundtrip(fsk):
    a = fsk.pinned_empty((1000, 3))
    a[...] = 7.0
    assert a.shape == (1000, 3) and a.dtype == np.float64 and float(a.sum()) == 21000.0
    p = a.__array_interface__["data"][0]
    del a
    b = fsk.pinned_empty((1000, 3))
    b[...] = 1.0
    assert float(b.sum()) == 3000.0 and p != 0
    with pytest.raises(fsk.DeviceError):
        fsk._check(fsk.lib().fsk_host_free(12345))


@pytest.mark.parametrize("where", ["src", "tgt"])
def test_deferred_finiteness_error(fsk, where):
    X, a, Y, b = _problem(5000, 4000, 64)
    (X if where == "src" else Y)[1234, 7] = np.nan
    with pytest.raises(fsk.ValidationError, match="non-finite coordinate in measure"):
        fsk.sinkhorn_solve(X, a, Y, b, eps=0.05, max_iters=3, precision="single", grad=True)


def test_deferred_finiteness_error_order(fsk):
    """Non-finite source coordinates come before a bad target weight and a bad config
    (the reference's check order), also when the finiteness scan is deferred."""
    X, a, Y, b = _problem(5000, 4000, 64)
    X[3, 3] = np.inf
    b = b.copy()
    b[0] = -1.0
    with pytest.raises(fsk.ValidationError, match="non-finite coordinate in measure"):
        fsk.sinkhorn_solve(X, a, Y, b, eps=0.05, max_iters=3, precision="single")
    X2, a2, Y2, b2 = _problem(5000, 4000, 64)
    Y2[0, 0] = np.nan
    with pytest.raises(fsk.ValidationError, match="non-finite coordinate in measure"):
        fsk.sinkhorn_solve(X2, a2, Y2, b2, eps=-1.0, max_iters=3, precision="single")
    X3, a3, Y3, b3 = _problem(5000, 4000, 64)
    b3 = b3.copy()
    b3[0] = 0.0
    with pytest.raises(fsk.ValidationError, match="strictly positive"):
        fsk.sinkhorn_solve(X3, a3, Y3, b3, eps=0.05, max_iters=3, precision="single")


@pytest.mark.parametrize("n,m", [(1 << 16, 1 << 16), (1 << 18, 1 << 18)])
def test_overlapped_gradient_download_same_bits(fsk, monkeypatch, n, m):
    """With a page-locked gradient output the gradient runs between the two marginal
    passes and downloads on a copy stream (FSK_OVERLAP_GRAD): same bits as the
    sequential order."""
    X, a, Y, b = _problem(n, m, 64, seed=11)
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("FSK_OVERLAP_GRAD", flag)
        outs.append(fsk.sinkhorn_solve(X, a, Y, b, eps=0.05, max_iters=6, precision="single",
                                       grad=True))
    for key in ("f_hat", "g_hat", "grad"):
        assert np.array_equal(outs[0][key], outs[1][key]), key
    assert outs[0]["dual_cost"] == outs[1]["dual_cost"]
    assert outs[0]["marginal_violation"] == outs[1]["marginal_violation"]
