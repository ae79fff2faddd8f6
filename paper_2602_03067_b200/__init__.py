"""B200-native FlashSinkhorn engine - Python host binding.

This package is a thin ctypes mirror of the C ABI in include/fsk_b200.h (the
drop-in boundary for the reference's fsk::stream / fsk::solver API,
/root/reference/proj/include/fsk/{stream,solver}.hpp). Every numeric result is
computed by the sm_100a kernels in libfsk_b200.so; there is no CPU fallback:
importing works anywhere, but any compute call fails loudly
(``DeviceError``) when the library or a CUDA device is missing.

Names and argument meaning follow the reference operations:

    update_f_hat, update_g_hat, symmetric_update, apply_plan,
    apply_plan_adjoint, apply_hadamard_plan, induced_marginals,
    update_f_hat_f32, update_g_hat_f32, io_count_*, tiles_fit_sram,
    sinkhorn_solve, dual_cost, sinkhorn_divergence(_mixed)

plus the SPEC modules the reference never implemented: grad_source,
grad_target, barycentric_projection, sinkhorn_solve_grad, hvp_apply, and the
device-resident ``Engine`` used for sharded multi-GPU runs.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "_build" / "libfsk_b200.so"


class ValidationError(RuntimeError):
    """fsk::ValidationError (proj/include/fsk/core.hpp:16-18)."""


class NumericalError(RuntimeError):
    """fsk::NumericalError (proj/include/fsk/core.hpp:21-23)."""


class DeviceError(RuntimeError):
    """CUDA / library failure (no CPU fallback exists)."""


class _Measure(C.Structure):
    _fields_ = [("points", C.c_void_p), ("weights", C.c_void_p), ("labels", C.c_void_p),
                ("n", C.c_int64), ("d", C.c_int64)]


class _Cost(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lambda1", C.c_double), ("lambda2", C.c_double),
                ("label_cost", C.c_void_p), ("num_labels", C.c_int64)]


class _Tiles(C.Structure):
    _fields_ = [("block_rows", C.c_int64), ("block_cols", C.c_int64)]


class Ledger(C.Structure):
    """fsk::IoLedger counters (proj/include/fsk/ledger.hpp:12-40)."""
    _fields_ = [("slow_to_fast_scalars", C.c_uint64), ("fast_to_slow_scalars", C.c_uint64),
                ("kernel_invocations", C.c_uint64), ("transport_vector_applies", C.c_uint64),
                ("transport_matrix_applies", C.c_uint64), ("hadamard_applies", C.c_uint64)]

    def total_scalars(self) -> int:
        return int(self.slow_to_fast_scalars + self.fast_to_slow_scalars)


class _Config(C.Structure):
    _fields_ = [("eps", C.c_double), ("schedule", C.c_int32), ("max_iters", C.c_int32),
                ("marginal_tol", C.c_double), ("eps_scaling_factor", C.c_double),
                ("extra_iters_at_final_eps", C.c_int32), ("precision", C.c_int32)]


class _Report(C.Structure):
    _fields_ = [("f_hat", C.c_void_p), ("g_hat", C.c_void_p), ("eps_history", C.c_void_p),
                ("eps_history_cap", C.c_int64), ("iterations", C.c_int32),
                ("marginal_violation", C.c_double), ("dual_cost", C.c_double),
                ("eps", C.c_double)]


class _HvpConfig(C.Structure):
    _fields_ = [("tau", C.c_double), ("cg_tol", C.c_double), ("cg_max_iters", C.c_int32)]


class _HvpReport(C.Structure):
    _fields_ = [("cg_iters", C.c_int32), ("cg_rel_residual", C.c_double),
                ("converged", C.c_int32)]


_lib = None


def lib() -> C.CDLL:
    """Loads libfsk_b200.so (raises DeviceError when it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DeviceError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                              "(the B200 engine has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        L.fsk_last_error.restype = C.c_char_p
        L.fsk_version.restype = C.c_char_p
        L.fsk_engine_path.restype = C.c_char_p
        L.fsk_engine_kernel_launches.restype = C.c_int64
        L.fsk_engine_screen_live_tiles.restype = C.c_uint64
        L.fsk_engine_screen_blocks.restype = C.c_uint64
        L.fsk_engine_live_set_fraction.restype = C.c_double
        L.fsk_device_peak_bytes.restype = C.c_int64
        L.fsk_host_alloc.restype = C.c_void_p
        L.fsk_host_alloc.argtypes = [C.c_size_t]
        L.fsk_host_free.argtypes = [C.c_void_p]
        for name in ("fsk_io_count_f_update", "fsk_io_count_g_update",
                     "fsk_io_count_symmetric_update", "fsk_io_count_apply_plan",
                     "fsk_io_count_apply_plan_adjoint", "fsk_io_count_apply_hadamard",
                     "fsk_io_count_induced_marginals"):
            getattr(L, name).restype = C.c_uint64
        _lib = L
    return _lib


class _PinnedBlock:
    """One page-locked host block from the library's pool (fsk_host_alloc); numpy
    arrays made from it keep it alive and hand it back to the pool when collected."""

    def __init__(self, shape, dtype):
        dtype = np.dtype(dtype)
        nbytes = max(int(np.prod(shape, dtype=np.int64)) * dtype.itemsize, 1)
        ptr = lib().fsk_host_alloc(nbytes)
        if not ptr:
            raise DeviceError("fsk_host_alloc: " + lib().fsk_last_error().decode())
        self.ptr = ptr
        self.__array_interface__ = {"shape": tuple(shape), "typestr": dtype.str,
                                    "data": (ptr, False), "version": 3}

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().fsk_host_free(self.ptr)
            self.ptr = None


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """Uninitialised array in page-locked host memory (the library's pinned pool).
    Solve inputs and outputs held in such arrays cross the host link by one DMA."""
    if isinstance(shape, int):
        shape = (shape,)
    return np.asarray(_PinnedBlock(shape, dtype))


def pinned_copy(a) -> np.ndarray:
    """Contiguous copy of `a` in page-locked host memory."""
    a = np.asarray(a)
    out = pinned_empty(a.shape, a.dtype)
    out[...] = a
    return out


def _out_array(shape) -> np.ndarray:
    """Output buffer of a solve: page-locked (pool) from 8 MB up, so the download is
    one DMA; plain numpy when no device / pinned memory is available."""
    if int(np.prod(shape)) * 8 >= (8 << 20):
        try:
            return pinned_empty(shape)
        except (DeviceError, OSError):
            pass
    return np.empty(shape)


def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib().fsk_last_error().decode()
    if status == 1:
        raise ValidationError(msg)
    if status == 2:
        raise NumericalError(msg)
    raise DeviceError(msg)


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


class _Keep:
    """Holds numpy buffers alive for the duration of one C call."""

    def __init__(self):
        self.items = []

    def measure(self, pts, w, labels=None) -> _Measure:
        pts = _f64(pts)
        if pts.ndim == 1:
            pts = pts[:, None]
        w = _f64(w)
        lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
        self.items += [pts, w, lab]
        return _Measure(pts.ctypes.data, w.ctypes.data, None if lab is None else lab.ctypes.data,
                        pts.shape[0], pts.shape[1] if pts.size else 0)

    def cost(self, cost) -> _Cost:
        if cost is None:
            return _Cost(0, 1.0, 0.0, None, 0)
        W = _f64(cost["label_cost"])
        self.items.append(W)
        return _Cost(1, float(cost["lambda1"]), float(cost["lambda2"]), W.ctypes.data,
                     W.shape[0])

    def arr(self, a, dtype=np.float64):
        a = np.ascontiguousarray(a, dtype=dtype)
        self.items.append(a)
        return a


def _tiles(t) -> _Tiles:
    return _Tiles(int(t[0]), int(t[1]))


def _lp(ledger):
    return C.byref(ledger) if ledger is not None else None


# ---- stream ops ---------------------------------------------------------------

def update_f_hat(X, a, Y, b, g_hat, eps, tiles=(64, 64), cost=None, la=None, lb=None,
                 ledger=None):
    k = _Keep()
    src, tgt = k.measure(X, a, la), k.measure(Y, b, lb)
    g = k.arr(g_hat)
    out = np.empty(src.n)
    _check(lib().fsk_update_f_hat(C.byref(src), C.byref(tgt), C.c_void_p(g.ctypes.data),
                                  C.byref(k.cost(cost)), C.c_double(eps), C.byref(_tiles(tiles)),
                                  _lp(ledger), C.c_void_p(out.ctypes.data)))
    return out


def update_g_hat(X, a, Y, b, f_hat, eps, tiles=(64, 64), cost=None, la=None, lb=None,
                 ledger=None):
    k = _Keep()
    src, tgt = k.measure(X, a, la), k.measure(Y, b, lb)
    f = k.arr(f_hat)
    out = np.empty(tgt.n)
    _check(lib().fsk_update_g_hat(C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data),
                                  C.byref(k.cost(cost)), C.c_double(eps), C.byref(_tiles(tiles)),
                                  _lp(ledger), C.c_void_p(out.ctypes.data)))
    return out


def symmetric_update(X, a, Y, b, f_hat, g_hat, eps, tiles=(64, 64), cost=None, la=None, lb=None,
                     ledger=None):
    k = _Keep()
    src, tgt = k.measure(X, a, la), k.measure(Y, b, lb)
    f, g = k.arr(f_hat), k.arr(g_hat)
    of, og = np.empty(src.n), np.empty(tgt.n)
    _check(lib().fsk_symmetric_update(C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data),
                                      C.c_void_p(g.ctypes.data), C.c_double(eps),
                                      C.byref(k.cost(cost)), C.byref(_tiles(tiles)), _lp(ledger),
                                      C.c_void_p(of.ctypes.data), C.c_void_p(og.ctypes.data)))
    return of, og


def _transport(fn, X, a, Y, b, f_hat, g_hat, eps, M, rows, tiles, cost, la, lb, ledger):
    k = _Keep()
    src, tgt = k.measure(X, a, la), k.measure(Y, b, lb)
    f, g = k.arr(f_hat), k.arr(g_hat)
    M = k.arr(M)
    if M.ndim == 1:
        M = k.arr(M[:, None])
    out = np.empty((rows(src, tgt), M.shape[1]))
    _check(fn(C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data), C.c_void_p(g.ctypes.data),
              C.c_double(eps), C.byref(k.cost(cost)), C.c_void_p(M.ctypes.data),
              C.c_int64(M.shape[1]), C.byref(_tiles(tiles)), _lp(ledger),
              C.c_void_p(out.ctypes.data)))
    return out


def apply_plan(X, a, Y, b, f_hat, g_hat, eps, V, tiles=(64, 64), cost=None, la=None, lb=None,
               ledger=None):
    return _transport(lib().fsk_apply_plan, X, a, Y, b, f_hat, g_hat, eps, V,
                      lambda s, t: s.n, tiles, cost, la, lb, ledger)


def apply_plan_adjoint(X, a, Y, b, f_hat, g_hat, eps, U, tiles=(64, 64), cost=None, la=None,
                       lb=None, ledger=None):
    return _transport(lib().fsk_apply_plan_adjoint, X, a, Y, b, f_hat, g_hat, eps, U,
                      lambda s, t: t.n, tiles, cost, la, lb, ledger)


def apply_hadamard_plan(X, a, Y, b, f_hat, g_hat, eps, A, B, V, tiles=(64, 64), cost=None,
                        la=None, lb=None, ledger=None):
    k = _Keep()
    src, tgt = k.measure(X, a, la), k.measure(Y, b, lb)
    f, g = k.arr(f_hat), k.arr(g_hat)
    A, B, V = k.arr(A), k.arr(B), k.arr(V)
    out = np.empty((src.n, V.shape[1]))
    _check(lib().fsk_apply_hadamard_plan(
        C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data), C.c_void_p(g.ctypes.data),
        C.c_double(eps), C.byref(k.cost(cost)), C.c_void_p(A.ctypes.data),
        C.c_void_p(B.ctypes.data), C.c_int64(A.shape[1]), C.c_void_p(V.ctypes.data),
        C.c_int64(V.shape[1]), C.byref(_tiles(tiles)), _lp(ledger), C.c_void_p(out.ctypes.data)))
    return out


def induced_marginals(X, a, Y, b, f_hat, g_hat, eps, tiles=(64, 64), cost=None, la=None, lb=None,
                      ledger=None):
    k = _Keep()
    src, tgt = k.measure(X, a, la), k.measure(Y, b, lb)
    f, g = k.arr(f_hat), k.arr(g_hat)
    r, c = np.empty(src.n), np.empty(tgt.n)
    _check(lib().fsk_induced_marginals(C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data),
                                       C.c_void_p(g.ctypes.data), C.c_double(eps),
                                       C.byref(k.cost(cost)), C.byref(_tiles(tiles)),
                                       _lp(ledger), C.c_void_p(r.ctypes.data),
                                       C.c_void_p(c.ctypes.data)))
    return r, c


def _check_clouds(X, a, Y, b, pots=()):
    """Shape checks a raw-pointer entry cannot make itself (d is passed once for both
    clouds): 2-D clouds of equal width, weights and potentials of matching length."""
    if X.ndim != 2 or Y.ndim != 2:
        raise ValidationError("point clouds must be 2-D (n x d) arrays")
    if X.shape[1] != Y.shape[1]:
        raise ValidationError(f"source and target dimensions differ ({X.shape[1]} vs {Y.shape[1]})")
    if a.shape != (X.shape[0],) or b.shape != (Y.shape[0],):
        raise ValidationError("weight vector length does not match the number of points")
    for v, want, name in pots:
        if v.shape != (want,):
            raise ValidationError(f"{name} length {v.shape[0] if v.ndim else 0} != {want}")


def update_f_hat_f32(X, a, Y, b, g_hat, eps, tiles=(64, 64), ledger=None):
    k = _Keep()
    X, a, Y, b = (k.arr(v, np.float32) for v in (X, a, Y, b))
    g = k.arr(g_hat, np.float32)
    _check_clouds(X, a, Y, b, [(g, Y.shape[0], "g_hat")])
    out = np.empty(X.shape[0], dtype=np.float32)
    _check(lib().fsk_update_f_hat_f32(
        C.c_void_p(X.ctypes.data), C.c_void_p(a.ctypes.data), C.c_int64(X.shape[0]),
        C.c_void_p(Y.ctypes.data), C.c_void_p(b.ctypes.data), C.c_int64(Y.shape[0]),
        C.c_int64(X.shape[1]), C.c_void_p(g.ctypes.data), C.c_float(eps),
        C.byref(_tiles(tiles)), _lp(ledger), C.c_void_p(out.ctypes.data)))
    return out


def update_g_hat_f32(X, a, Y, b, f_hat, eps, tiles=(64, 64), ledger=None):
    k = _Keep()
    X, a, Y, b = (k.arr(v, np.float32) for v in (X, a, Y, b))
    f = k.arr(f_hat, np.float32)
    _check_clouds(X, a, Y, b, [(f, X.shape[0], "f_hat")])
    out = np.empty(Y.shape[0], dtype=np.float32)
    _check(lib().fsk_update_g_hat_f32(
        C.c_void_p(X.ctypes.data), C.c_void_p(a.ctypes.data), C.c_int64(X.shape[0]),
        C.c_void_p(Y.ctypes.data), C.c_void_p(b.ctypes.data), C.c_int64(Y.shape[0]),
        C.c_int64(X.shape[1]), C.c_void_p(f.ctypes.data), C.c_float(eps),
        C.byref(_tiles(tiles)), _lp(ledger), C.c_void_p(out.ctypes.data)))
    return out


def io_count(kind: str, *dims, tiles=(64, 64)) -> int:
    """io_count_{f_update,g_update,symmetric_update,apply_plan,apply_plan_adjoint,
    apply_hadamard,induced_marginals} (stream.cpp:459-499)."""
    fn = getattr(lib(), "fsk_io_count_" + kind)
    return int(fn(*[C.c_int64(int(v)) for v in dims], C.byref(_tiles(tiles))))


def tiles_fit_sram(tiles, d, sram_scalars) -> bool:
    return bool(lib().fsk_tiles_fit_sram(C.byref(_tiles(tiles)), C.c_int64(d),
                                         C.c_int64(sram_scalars)))


def debug_break_lse(broken: bool) -> None:
    lib().fsk_debug_break_lse(C.c_int(1 if broken else 0))


# ---- solver -------------------------------------------------------------------

def _config(eps, schedule, max_iters, marginal_tol, eps_scaling_factor, extra_iters_at_final_eps,
            precision):
    return _Config(eps, 1 if schedule == "symmetric" else 0, max_iters, marginal_tol,
                   eps_scaling_factor, extra_iters_at_final_eps,
                   1 if precision == "double" else 0)


def sinkhorn_solve(X, a, Y, b, eps=0.1, schedule="alternating", max_iters=100, marginal_tol=0.0,
                   eps_scaling_factor=1.0, extra_iters_at_final_eps=0, precision="double",
                   tiles=(64, 64), cost=None, la=None, lb=None, ledger=None, grad=False,
                   f_init=None, g_init=None):
    """fsk::solver::sinkhorn_solve; with grad=True also returns grad_X (fwd+grad).
    f_init / g_init (shifted potentials): warm start (fsk_sinkhorn_solve_warm)."""
    k = _Keep()
    src, tgt = k.measure(X, a, la), k.measure(Y, b, lb)
    cfg = _config(eps, schedule, max_iters, marginal_tol, eps_scaling_factor,
                  extra_iters_at_final_eps, precision)
    f, g = _out_array(src.n), _out_array(tgt.n)
    hist = np.zeros(max(max_iters, 1))
    rep = _Report(f.ctypes.data, g.ctypes.data, hist.ctypes.data, len(hist), 0, 0.0, 0.0, 0.0)
    if f_init is not None or g_init is not None:
        if f_init is None or g_init is None:
            raise ValidationError("warm start needs both f_init and g_init")
        fi, gi = k.arr(f_init), k.arr(g_init)
        if fi.shape != (src.n,) or gi.shape != (tgt.n,):
            raise ValidationError("warm-start potentials do not match the measures")
        G = _out_array((src.n, src.d)) if grad else None
        _check(lib().fsk_sinkhorn_solve_warm(
            C.byref(src), C.byref(tgt), C.byref(k.cost(cost)), C.byref(cfg),
            C.byref(_tiles(tiles)), _lp(ledger), C.c_void_p(fi.ctypes.data),
            C.c_void_p(gi.ctypes.data), C.byref(rep),
            C.c_void_p(G.ctypes.data) if grad else None))
    elif grad:
        G = _out_array((src.n, src.d))
        _check(lib().fsk_sinkhorn_solve_grad(C.byref(src), C.byref(tgt), C.byref(k.cost(cost)),
                                             C.byref(cfg), C.byref(_tiles(tiles)), _lp(ledger),
                                             C.byref(rep), C.c_void_p(G.ctypes.data)))
    else:
        _check(lib().fsk_sinkhorn_solve(C.byref(src), C.byref(tgt), C.byref(k.cost(cost)),
                                        C.byref(cfg), C.byref(_tiles(tiles)), _lp(ledger),
                                        C.byref(rep)))
    out = dict(f_hat=f, g_hat=g, iterations=rep.iterations,
               marginal_violation=rep.marginal_violation, dual_cost=rep.dual_cost, eps=rep.eps,
               eps_history=hist[:rep.iterations].copy())
    if grad:
        out["grad"] = G
    return out


def dual_cost(X, a, Y, b, f_hat, g_hat, eps, tiles=(64, 64), cost=None, la=None, lb=None,
              ledger=None):
    k = _Keep()
    src, tgt = k.measure(X, a, la), k.measure(Y, b, lb)
    f, g = k.arr(f_hat), k.arr(g_hat)
    out = C.c_double(0.0)
    _check(lib().fsk_dual_cost(C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data),
                               C.c_void_p(g.ctypes.data), C.c_double(eps), C.byref(k.cost(cost)),
                               C.byref(_tiles(tiles)), _lp(ledger), C.byref(out)))
    return out.value


def sinkhorn_divergence(X, a, Y, b, eps=0.1, schedule="alternating", max_iters=100,
                        marginal_tol=0.0, eps_scaling_factor=1.0, extra_iters_at_final_eps=0,
                        precision="double", tiles=(64, 64), cost=None, ledger=None):
    k = _Keep()
    mu, nu = k.measure(X, a), k.measure(Y, b)
    cfg = _config(eps, schedule, max_iters, marginal_tol, eps_scaling_factor,
                  extra_iters_at_final_eps, precision)
    c = k.cost(cost)
    out = C.c_double(0.0)
    _check(lib().fsk_sinkhorn_divergence_mixed(C.byref(mu), C.byref(nu), C.byref(c), C.byref(c),
                                               C.byref(c), C.byref(cfg), C.byref(_tiles(tiles)),
                                               _lp(ledger), C.byref(out)))
    return out.value


def sinkhorn_divergence_batch(pairs, eps=0.1, max_iters=10, precision="single", tiles=(64, 64),
                              schedule="alternating", ledger=None):
    """pairs: list of (X, a, Y, b); one call, all 3 solves per pair on device."""
    k = _Keep()
    mus = (_Measure * len(pairs))(*[k.measure(X, a) for (X, a, _, _) in pairs])
    nus = (_Measure * len(pairs))(*[k.measure(Y, b) for (_, _, Y, b) in pairs])
    cfg = _config(eps, schedule, max_iters, 0.0, 1.0, 0, precision)
    out = np.empty(len(pairs))
    _check(lib().fsk_sinkhorn_divergence_batch(mus, nus, C.c_int64(len(pairs)),
                                               C.byref(k.cost(None)), C.byref(cfg),
                                               C.byref(_tiles(tiles)), _lp(ledger),
                                               C.c_void_p(out.ctypes.data)))
    return out


# ---- SPEC autodiff / hvp ---------------------------------------------------------

def _autodiff(fn, rows, X, a, Y, b, f_hat, g_hat, eps, tiles, cost, ledger):
    k = _Keep()
    src, tgt = k.measure(X, a), k.measure(Y, b)
    f, g = k.arr(f_hat), k.arr(g_hat)
    out = np.empty((rows(src, tgt), src.d))
    _check(fn(C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data), C.c_void_p(g.ctypes.data),
              C.c_double(eps), C.byref(k.cost(cost)), C.byref(_tiles(tiles)), _lp(ledger),
              C.c_void_p(out.ctypes.data)))
    return out


def grad_source(X, a, Y, b, f_hat, g_hat, eps, tiles=(64, 64), cost=None, ledger=None):
    return _autodiff(lib().fsk_grad_source, lambda s, t: s.n, X, a, Y, b, f_hat, g_hat, eps,
                     tiles, cost, ledger)


def grad_target(X, a, Y, b, f_hat, g_hat, eps, tiles=(64, 64), cost=None, ledger=None):
    return _autodiff(lib().fsk_grad_target, lambda s, t: t.n, X, a, Y, b, f_hat, g_hat, eps,
                     tiles, cost, ledger)


def barycentric_projection(X, a, Y, b, f_hat, g_hat, eps, tiles=(64, 64), cost=None, ledger=None):
    return _autodiff(lib().fsk_barycentric_projection, lambda s, t: s.n, X, a, Y, b, f_hat, g_hat,
                     eps, tiles, cost, ledger)


def hvp_apply(X, a, Y, b, f_hat, g_hat, eps, A, tau=1e-5, cg_tol=1e-6, cg_max_iters=50,
              tiles=(64, 64), cost=None, ledger=None, precision="double"):
    """SPEC hvp_apply. precision="single" runs the fp32 engine
    (tcgen05 transport-vector applications when the tensor path is enabled)."""
    k = _Keep()
    src, tgt = k.measure(X, a), k.measure(Y, b)
    f, g, A = k.arr(f_hat), k.arr(g_hat), k.arr(A)
    out = _out_array((src.n, src.d))
    h = _HvpConfig(tau, cg_tol, cg_max_iters)
    rep = _HvpReport()
    fn = lib().fsk_hvp_apply_single if precision == "single" else lib().fsk_hvp_apply
    _check(fn(C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data), C.c_void_p(g.ctypes.data),
              C.c_double(eps), C.byref(k.cost(cost)), C.c_void_p(A.ctypes.data), C.byref(h),
              C.byref(_tiles(tiles)), _lp(ledger), C.c_void_p(out.ctypes.data), C.byref(rep)))
    return out, dict(cg_iters=rep.cg_iters, cg_rel_residual=rep.cg_rel_residual,
                     converged=bool(rep.converged))


def rng_normal(seed: int, count: int) -> np.ndarray:
    """fsk::Rng(seed).normal() x count (bit-identical to the reference generator)."""
    out = np.empty(count)
    lib().fsk_rng_normal_fill(C.c_uint64(seed), C.c_void_p(out.ctypes.data), C.c_int64(count))
    return out


def set_num_devices(n: int) -> None:
    """fsk_set_num_devices: 0 (default) = the single-device path; n >= 1 = sinkhorn_solve
    (and _grad / warm starts) shard rows over devices 0..n-1 with in-library NCCL
    all-gathers."""
    _check(lib().fsk_set_num_devices(C.c_int(n)))


def num_devices() -> int:
    return int(lib().fsk_num_devices())


def device_peak_bytes(device: int = 0, reset: bool = False) -> int:
    """High-water mark of the device memory pool every library allocation comes from
    (fsk_device_peak_bytes); reset=True restarts it at the current usage."""
    return int(lib().fsk_device_peak_bytes(C.c_int(device), C.c_int(1 if reset else 0)))


def version() -> str:
    return lib().fsk_version().decode()


# ---- device engine ------------------------------------------------------------------

def _dp(x) -> int:
    """Device pointer of a torch tensor, or the int itself."""
    return x.data_ptr() if hasattr(x, "data_ptr") else int(x)


class Engine:
    """Device-resident problem (fsk_engine_*). Potentials are caller-owned float32
    device buffers (e.g. torch tensors) so a collective library can all-gather them
    in place; half-steps run over row ranges."""

    MODES = {"auto": 0, "fma": 1, "tensor": 2}

    def __init__(self, device, X, a, Y, b, mode="auto", cost=None, la=None, lb=None):
        """cost (dict lambda1, lambda2, label_cost V x V) with labels la, lb: the
        label-augmented cost (fsk_engine_create_labeled)."""
        k = _Keep()
        X, a, Y, b = k.arr(X), k.arr(a), k.arr(Y), k.arr(b)
        _check_clouds(X, a, Y, b)
        h = C.c_void_p()
        if cost is not None:
            la = k.arr(la, np.int32)
            lb = k.arr(lb, np.int32)
            W = k.arr(cost["label_cost"])
            _check(lib().fsk_engine_create_labeled(
                C.c_int(device), C.c_void_p(X.ctypes.data), C.c_void_p(a.ctypes.data),
                C.c_void_p(la.ctypes.data), C.c_int64(X.shape[0]), C.c_void_p(Y.ctypes.data),
                C.c_void_p(b.ctypes.data), C.c_void_p(lb.ctypes.data), C.c_int64(Y.shape[0]),
                C.c_int64(X.shape[1]), C.c_double(cost["lambda1"]), C.c_double(cost["lambda2"]),
                C.c_void_p(W.ctypes.data), C.c_int64(W.shape[0]), C.c_int(self.MODES[mode]),
                C.byref(h)))
        else:
            _check(lib().fsk_engine_create(C.c_int(device), C.c_void_p(X.ctypes.data),
                                           C.c_void_p(a.ctypes.data), C.c_int64(X.shape[0]),
                                           C.c_void_p(Y.ctypes.data), C.c_void_p(b.ctypes.data),
                                           C.c_int64(Y.shape[0]), C.c_int64(X.shape[1]),
                                           C.c_int(self.MODES[mode]), C.byref(h)))
        self.h = h
        self.n, self.m, self.d = X.shape[0], Y.shape[0], X.shape[1]

    def close(self):
        if self.h:
            lib().fsk_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def path(self) -> str:
        return lib().fsk_engine_path(self.h).decode()

    def live_tiles(self) -> int:
        """(query tile, key tile) blocks scored in full by tracked LSE passes so far."""
        return int(lib().fsk_engine_screen_live_tiles(self.h))

    def live_set_fraction(self, side: int) -> float:
        """Live-tile fraction recorded by the last LSE pass of `side` (-1: none)."""
        return float(lib().fsk_engine_live_set_fraction(self.h, C.c_int(side)))

    def screened_blocks(self) -> int:
        """(query tile, key tile) blocks covered by tracked LSE passes so far."""
        return int(lib().fsk_engine_screen_blocks(self.h))

    def pass_counts(self) -> dict:
        """LSE passes of the tensor path so far by kind (screened / warm / plain)."""
        out = (C.c_uint64 * 3)()
        lib().fsk_engine_pass_counts(self.h, out)
        return {"screened": int(out[0]), "warm": int(out[1]), "plain": int(out[2])}

    @staticmethod
    def launches() -> int:
        return int(lib().fsk_engine_kernel_launches(None))

    def set_eps(self, eps: float):
        _check(lib().fsk_engine_set_eps(self.h, C.c_double(eps)))

    def bind(self, f_ptr: int, g_ptr: int):
        _check(lib().fsk_engine_bind_potentials(self.h, C.c_void_p(f_ptr), C.c_void_p(g_ptr)))

    def init_potentials(self, stream: int = 0):
        _check(lib().fsk_engine_init_potentials(self.h, C.c_void_p(stream)))

    def half_step(self, side: int, row_begin: int, row_end: int, viol_ptr: int = 0,
                  stream: int = 0):
        _check(lib().fsk_engine_half_step(self.h, C.c_int(side), C.c_int64(row_begin),
                                          C.c_int64(row_end),
                                          C.c_void_p(viol_ptr) if viol_ptr else None,
                                          C.c_void_p(stream)))

    def iterate(self, iters: int, stream: int = 0):
        """`iters` alternating iterations over all rows (CUDA graph on the CUDA-core path)."""
        _check(lib().fsk_engine_iterate(self.h, C.c_int(iters), C.c_void_p(stream)))

    def transport_vec(self, side: int, v_ptr: int, out_ptr: int, stream: int = 0):
        """out (double, device) = P v (side 0) or P^T v (side 1) at the bound potentials."""
        _check(lib().fsk_engine_transport_vec(self.h, C.c_int(side), C.c_void_p(v_ptr),
                                              C.c_void_p(out_ptr), C.c_void_p(stream)))

    def transport_mat(self, side: int, v_ptr: int, p: int, out_ptr: int, stream: int = 0):
        """out (float, device, rows x p) = P V (side 0) or P^T V (side 1)."""
        _check(lib().fsk_engine_transport_mat(self.h, C.c_int(side), C.c_void_p(v_ptr),
                                              C.c_int64(p), C.c_void_p(out_ptr),
                                              C.c_void_p(stream)))

    def transport_hadamard(self, a_ptr: int, v_ptr: int, p: int, out_ptr: int, stream: int = 0):
        """out (float, device, n x p) = (P (.) A Y^T) V."""
        _check(lib().fsk_engine_transport_hadamard(self.h, C.c_void_p(a_ptr), C.c_void_p(v_ptr),
                                                   C.c_int64(p), C.c_void_p(out_ptr),
                                                   C.c_void_p(stream)))

    def transport_prepare(self, f_rows, g_rows, stream: int = 0):
        """LSE / marginals of both orientations over row shards at the bound potentials
        (fsk_engine_transport_prepare); f_rows, g_rows = (begin, end)."""
        _check(lib().fsk_engine_transport_prepare(self.h, C.c_int64(f_rows[0]),
                                                  C.c_int64(f_rows[1]), C.c_int64(g_rows[0]),
                                                  C.c_int64(g_rows[1]), C.c_void_p(stream)))

    def marginal(self, side: int, out_ptr: int, stream: int = 0):
        _check(lib().fsk_engine_marginal(self.h, C.c_int(side), C.c_void_p(_dp(out_ptr)),
                                         C.c_void_p(stream)))

    def transport_vec_rows(self, side: int, lo: int, hi: int, v_ptr: int, out_ptr: int,
                           stream: int = 0):
        _check(lib().fsk_engine_transport_vec_rows(self.h, C.c_int(side), C.c_int64(lo),
                                                   C.c_int64(hi), C.c_void_p(_dp(v_ptr)),
                                                   C.c_void_p(_dp(out_ptr)), C.c_void_p(stream)))

    def transport_mat_rows(self, side: int, lo: int, hi: int, v_ptr, p: int, out_ptr,
                           a_ptr=None, stream: int = 0):
        _check(lib().fsk_engine_transport_mat_rows(self.h, C.c_int(side), C.c_int64(lo),
                                                   C.c_int64(hi), C.c_void_p(_dp(v_ptr)),
                                                   C.c_int64(p),
                                                   C.c_void_p(_dp(a_ptr)) if a_ptr is not None
                                                   and not (isinstance(a_ptr, int) and a_ptr == 0)
                                                   else None,
                                                   C.c_void_p(_dp(out_ptr)), C.c_void_p(stream)))

    def grad(self, row_begin: int, row_end: int, grad_ptr: int, stream: int = 0):
        _check(lib().fsk_engine_grad(self.h, C.c_int64(row_begin), C.c_int64(row_end),
                                     C.c_void_p(grad_ptr), C.c_void_p(stream)))
