"""Parity oracle for the FlashSinkhorn hot path.

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this package, and only as the
checker or as the timed CPU reference - never as the thing measured or shipped.
The product (paper_2602_03067_b200) has no dependency on it.

Two backends with one numpy-level interface:

* ``Oracle("port")``  - oracle/fsk_oracle.c, a plain-C restatement of the
  reference algorithm (file:line citations in that file), built here and on the
  GPU box by ``build()`` (gcc only).
* ``Oracle("ref")``   - oracle/_ref/libfsk_ref_check.so: the reference's own
  C++ sources compiled by oracle/build_ref.py (two documented patches). Present
  only where it was built (this container, and the GPU box via the snapshot).

Status codes mirror the reference exceptions: ValidationError / NumericalError.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD = HERE / "_build"
PORT_SO = BUILD / "libfsk_oracle.so"
REF_DIR = HERE / "_ref"
REF_CHECK_SO = REF_DIR / "libfsk_ref_check.so"


class ValidationError(RuntimeError):
    pass


class NumericalError(RuntimeError):
    pass


def build(force: bool = False) -> Path:
    """Compile the C restatement (strict IEEE order, OpenMP over row blocks)."""
    BUILD.mkdir(exist_ok=True)
    src = HERE / "fsk_oracle.c"
    if force or not PORT_SO.exists() or PORT_SO.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(
            ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-march=x86-64-v3", "-fopenmp",
             "-fPIC", "-shared", "-Wno-unknown-pragmas", "-Wno-format-truncation", str(src),
             "-o", str(PORT_SO), "-lm"],
            check=True,
        )
    return PORT_SO


class _Measure(C.Structure):
    _fields_ = [("pts", C.c_void_p), ("w", C.c_void_p), ("labels", C.c_void_p),
                ("n", C.c_int64), ("d", C.c_int64)]


class _Cost(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lambda1", C.c_double), ("lambda2", C.c_double),
                ("label_cost", C.c_void_p), ("num_labels", C.c_int64)]


class _Config(C.Structure):
    _fields_ = [("eps", C.c_double), ("schedule", C.c_int32), ("max_iters", C.c_int32),
                ("marginal_tol", C.c_double), ("eps_scaling_factor", C.c_double),
                ("extra_iters_at_final_eps", C.c_int32), ("precision", C.c_int32)]


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a):
    return None if a is None else a.ctypes.data


class Oracle:
    """Numpy-level access to one backend ("port" or "ref")."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        if kind == "port":
            self.lib = C.CDLL(str(build()))
            self.p = "fo_"
            self.lib.fo_fast_exp_d.restype = C.c_double
            self.lib.fo_fast_exp_d.argtypes = [C.c_double]
            self.lib.fo_fast_exp_f.restype = C.c_float
            self.lib.fo_fast_exp_f.argtypes = [C.c_float]
            self.lib.fo_joint_sq_diameter.restype = C.c_double
            self.lib.fo_eps_schedule.restype = C.c_int64
        elif kind == "ref":
            if not REF_CHECK_SO.exists():
                raise FileNotFoundError(f"{REF_CHECK_SO} not built (run oracle/build_ref.py)")
            self.lib = C.CDLL(str(REF_CHECK_SO))
            self.p = "ref_"
        elif kind == "ref_fast":
            # the reference's CMake flavour (-O3, FMA contraction), widest ISA the host has
            so = REF_DIR / ("libfsk_ref_fast_v4.so" if _has_avx512() else "libfsk_ref_fast_v3.so")
            if not so.exists():
                raise FileNotFoundError(f"{so} not built (run oracle/build_ref.py)")
            self.lib = C.CDLL(str(so))
            self.p = "ref_"
            self.so_path = so
            self.lib.ref_num_threads.restype = C.c_int64
        else:
            raise ValueError(kind)
        getattr(self.lib, self.p + "last_error").restype = C.c_char_p
        self._keep = []

    # ---- helpers -----------------------------------------------------------
    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, st):
        if st == 0:
            return
        msg = self._fn("last_error")().decode()
        if st == 1:
            raise ValidationError(msg)
        if st == 2:
            raise NumericalError(msg)
        raise RuntimeError(msg)

    def _measure(self, pts, w, labels=None):
        pts = _f64(pts)
        if pts.ndim == 1:
            pts = pts[:, None]
        w = _f64(w)
        lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
        self._keep += [pts, w, lab]
        return _Measure(pts.ctypes.data, w.ctypes.data, _ptr(lab), pts.shape[0], pts.shape[1])

    def _cost(self, cost):
        if cost is None:
            return _Cost(0, 1.0, 0.0, None, 0)
        W = _f64(cost["label_cost"])
        self._keep.append(W)
        return _Cost(1, float(cost["lambda1"]), float(cost["lambda2"]), W.ctypes.data,
                     W.shape[0])

    def _ledger(self):
        return np.zeros(6, dtype=np.uint64)

    # ---- stream ops (stream.hpp:20-75) -------------------------------------
    def update_f_hat(self, X, a, Y, b, g_hat, eps, tiles=(64, 64), cost=None, la=None, lb=None):
        src, tgt = self._measure(X, a, la), self._measure(Y, b, lb)
        out = np.empty(src.n, dtype=np.float64)
        g = _f64(g_hat)
        args = [C.byref(src), C.byref(tgt), C.c_void_p(g.ctypes.data), C.byref(self._cost(cost)),
                C.c_double(eps), C.c_int64(tiles[0]), C.c_int64(tiles[1]),
                C.c_void_p(out.ctypes.data)]
        if self.kind != "port":
            args.append(C.c_void_p(self._ledger().ctypes.data))
        self._check(self._fn("update_f_hat")(*args))
        self._keep.clear()
        return out

    def update_g_hat(self, X, a, Y, b, f_hat, eps, tiles=(64, 64), cost=None, la=None, lb=None):
        src, tgt = self._measure(X, a, la), self._measure(Y, b, lb)
        out = np.empty(tgt.n, dtype=np.float64)
        f = _f64(f_hat)
        args = [C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data), C.byref(self._cost(cost)),
                C.c_double(eps), C.c_int64(tiles[0]), C.c_int64(tiles[1]),
                C.c_void_p(out.ctypes.data)]
        if self.kind != "port":
            args.append(C.c_void_p(self._ledger().ctypes.data))
        self._check(self._fn("update_g_hat")(*args))
        self._keep.clear()
        return out

    def symmetric_update(self, X, a, Y, b, f_hat, g_hat, eps, tiles=(64, 64), cost=None, la=None,
                         lb=None):
        src, tgt = self._measure(X, a, la), self._measure(Y, b, lb)
        f, g = _f64(f_hat), _f64(g_hat)
        of, og = np.empty(src.n), np.empty(tgt.n)
        args = [C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data), C.c_void_p(g.ctypes.data),
                C.c_double(eps), C.byref(self._cost(cost)), C.c_int64(tiles[0]),
                C.c_int64(tiles[1]), C.c_void_p(of.ctypes.data), C.c_void_p(og.ctypes.data)]
        if self.kind != "port":
            args.append(C.c_void_p(self._ledger().ctypes.data))
        self._check(self._fn("symmetric_update")(*args))
        self._keep.clear()
        return of, og

    def _apply(self, name, X, a, Y, b, f_hat, g_hat, eps, M, rows_out, tiles, cost, la, lb):
        src, tgt = self._measure(X, a, la), self._measure(Y, b, lb)
        f, g = _f64(f_hat), _f64(g_hat)
        M = _f64(M)
        if M.ndim == 1:
            M = M[:, None]
        p = M.shape[1]
        out = np.empty((rows_out(src, tgt), p))
        args = [C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data), C.c_void_p(g.ctypes.data),
                C.c_double(eps), C.byref(self._cost(cost)), C.c_void_p(M.ctypes.data),
                C.c_int64(p), C.c_int64(tiles[0]), C.c_int64(tiles[1]),
                C.c_void_p(out.ctypes.data)]
        if self.kind != "port":
            args.append(C.c_void_p(self._ledger().ctypes.data))
        self._check(self._fn(name)(*args))
        self._keep.clear()
        return out

    def apply_plan(self, X, a, Y, b, f_hat, g_hat, eps, V, tiles=(64, 64), cost=None, la=None,
                   lb=None):
        return self._apply("apply_plan", X, a, Y, b, f_hat, g_hat, eps, V, lambda s, t: s.n,
                           tiles, cost, la, lb)

    def apply_plan_adjoint(self, X, a, Y, b, f_hat, g_hat, eps, U, tiles=(64, 64), cost=None,
                           la=None, lb=None):
        return self._apply("apply_plan_adjoint", X, a, Y, b, f_hat, g_hat, eps, U,
                           lambda s, t: t.n, tiles, cost, la, lb)

    def apply_hadamard_plan(self, X, a, Y, b, f_hat, g_hat, eps, A, B, V, tiles=(64, 64),
                            cost=None, la=None, lb=None):
        src, tgt = self._measure(X, a, la), self._measure(Y, b, lb)
        f, g = _f64(f_hat), _f64(g_hat)
        A, B, V = _f64(A), _f64(B), _f64(V)
        r, p = A.shape[1], V.shape[1]
        out = np.empty((src.n, p))
        args = [C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data), C.c_void_p(g.ctypes.data),
                C.c_double(eps), C.byref(self._cost(cost)), C.c_void_p(A.ctypes.data),
                C.c_void_p(B.ctypes.data), C.c_int64(r), C.c_void_p(V.ctypes.data),
                C.c_int64(p), C.c_int64(tiles[0]), C.c_int64(tiles[1]),
                C.c_void_p(out.ctypes.data)]
        if self.kind != "port":
            args.append(C.c_void_p(self._ledger().ctypes.data))
        self._check(self._fn("apply_hadamard_plan")(*args))
        self._keep.clear()
        return out

    def induced_marginals(self, X, a, Y, b, f_hat, g_hat, eps, tiles=(64, 64), cost=None,
                          la=None, lb=None):
        src, tgt = self._measure(X, a, la), self._measure(Y, b, lb)
        f, g = _f64(f_hat), _f64(g_hat)
        r, c = np.empty(src.n), np.empty(tgt.n)
        args = [C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data), C.c_void_p(g.ctypes.data),
                C.c_double(eps), C.byref(self._cost(cost)), C.c_int64(tiles[0]),
                C.c_int64(tiles[1]), C.c_void_p(r.ctypes.data), C.c_void_p(c.ctypes.data)]
        if self.kind != "port":
            args.append(C.c_void_p(self._ledger().ctypes.data))
        self._check(self._fn("induced_marginals")(*args))
        self._keep.clear()
        return r, c

    # ---- fp32 half-steps (stream.cpp:437-451) --------------------------------
    def update_f_hat_f32(self, X, a, Y, b, g_hat, eps, tiles=(64, 64)):
        X, a, Y, b, g = _f32(X), _f32(a), _f32(Y), _f32(b), _f32(g_hat)
        n, d = X.shape
        m = Y.shape[0]
        out = np.empty(n, dtype=np.float32)
        if self.kind != "port":
            st = self.lib.ref_update_f_hat_f32(
                C.c_void_p(X.ctypes.data), C.c_void_p(a.ctypes.data), C.c_int64(n),
                C.c_void_p(Y.ctypes.data), C.c_void_p(b.ctypes.data), C.c_int64(m),
                C.c_int64(d), C.c_void_p(g.ctypes.data), C.c_float(eps), C.c_int64(tiles[0]),
                C.c_int64(tiles[1]), C.c_void_p(out.ctypes.data),
                C.c_void_p(self._ledger().ctypes.data))
        else:
            st = self.lib.fo_update_f_hat_f32(
                C.c_void_p(X.ctypes.data), C.c_int64(n), C.c_void_p(Y.ctypes.data),
                C.c_void_p(b.ctypes.data), C.c_int64(m), C.c_int64(d),
                C.c_void_p(g.ctypes.data), C.c_float(eps), C.c_int64(tiles[0]),
                C.c_int64(tiles[1]), C.c_void_p(out.ctypes.data))
        self._check(st)
        return out

    def update_g_hat_f32(self, X, a, Y, b, f_hat, eps, tiles=(64, 64)):
        X, a, Y, b, f = _f32(X), _f32(a), _f32(Y), _f32(b), _f32(f_hat)
        n, d = X.shape
        m = Y.shape[0]
        out = np.empty(m, dtype=np.float32)
        if self.kind != "port":
            st = self.lib.ref_update_g_hat_f32(
                C.c_void_p(X.ctypes.data), C.c_void_p(a.ctypes.data), C.c_int64(n),
                C.c_void_p(Y.ctypes.data), C.c_void_p(b.ctypes.data), C.c_int64(m),
                C.c_int64(d), C.c_void_p(f.ctypes.data), C.c_float(eps), C.c_int64(tiles[0]),
                C.c_int64(tiles[1]), C.c_void_p(out.ctypes.data),
                C.c_void_p(self._ledger().ctypes.data))
        else:
            st = self.lib.fo_update_g_hat_f32(
                C.c_void_p(X.ctypes.data), C.c_void_p(a.ctypes.data), C.c_int64(n),
                C.c_void_p(Y.ctypes.data), C.c_int64(m), C.c_int64(d),
                C.c_void_p(f.ctypes.data), C.c_float(eps), C.c_int64(tiles[0]),
                C.c_int64(tiles[1]), C.c_void_p(out.ctypes.data))
        self._check(st)
        return out

    # ---- solver (solver.hpp:17-40) -------------------------------------------
    def sinkhorn_solve(self, X, a, Y, b, eps=0.1, schedule="alternating", max_iters=100,
                       marginal_tol=0.0, eps_scaling_factor=1.0, extra_iters_at_final_eps=0,
                       precision="double", tiles=(64, 64), cost=None, la=None, lb=None):
        src, tgt = self._measure(X, a, la), self._measure(Y, b, lb)
        cfg = _Config(eps, 1 if schedule == "symmetric" else 0, max_iters, marginal_tol,
                      eps_scaling_factor, extra_iters_at_final_eps,
                      1 if precision == "double" else 0)
        f, g = np.empty(src.n), np.empty(tgt.n)
        sc = np.zeros(4)
        hist = np.zeros(max(max_iters, 1))
        args = [C.byref(src), C.byref(tgt), C.byref(self._cost(cost)), C.byref(cfg),
                C.c_int64(tiles[0]), C.c_int64(tiles[1]), C.c_void_p(f.ctypes.data),
                C.c_void_p(g.ctypes.data), C.c_void_p(sc.ctypes.data),
                C.c_void_p(hist.ctypes.data)]
        if self.kind != "port":
            args += [C.c_int64(len(hist)), C.c_void_p(self._ledger().ctypes.data)]
        self._check(self._fn("sinkhorn_solve")(*args))
        self._keep.clear()
        it = int(sc[0])
        return dict(f_hat=f, g_hat=g, iterations=it, marginal_violation=sc[1], dual_cost=sc[2],
                    eps=sc[3], eps_history=hist[:it].copy())

    def dual_cost(self, X, a, Y, b, f_hat, g_hat, eps, tiles=(64, 64), cost=None, la=None,
                  lb=None):
        src, tgt = self._measure(X, a, la), self._measure(Y, b, lb)
        f, g = _f64(f_hat), _f64(g_hat)
        out = np.zeros(1)
        args = [C.byref(src), C.byref(tgt), C.c_void_p(f.ctypes.data), C.c_void_p(g.ctypes.data),
                C.c_double(eps), C.byref(self._cost(cost)), C.c_int64(tiles[0]),
                C.c_int64(tiles[1]), C.c_void_p(out.ctypes.data)]
        if self.kind != "port":
            args.append(C.c_void_p(self._ledger().ctypes.data))
        self._check(self._fn("dual_cost")(*args))
        self._keep.clear()
        return float(out[0])

    def sinkhorn_divergence(self, X, a, Y, b, **kw):
        """S = OT(mu,nu) - OT(mu,mu)/2 - OT(nu,nu)/2 (solver.cpp:145-159)."""
        cross = self.sinkhorn_solve(X, a, Y, b, **kw)["dual_cost"]
        smu = self.sinkhorn_solve(X, a, X, a, **kw)["dual_cost"]
        snu = self.sinkhorn_solve(Y, b, Y, b, **kw)["dual_cost"]
        return cross - 0.5 * smu - 0.5 * snu

    # ---- misc ----------------------------------------------------------------
    def set_num_threads(self, n: int):
        if self.kind != "port":
            self.lib.ref_set_num_threads(C.c_int64(n))
        else:
            os.environ["OMP_NUM_THREADS"] = str(n)


    def num_threads(self) -> int:
        if self.kind.startswith("ref"):
            self.lib.ref_num_threads.restype = C.c_int64
            return int(self.lib.ref_num_threads())
        return os.cpu_count() or 1


def uniform(n: int) -> np.ndarray:
    return np.full(n, 1.0 / n)


def _has_avx512() -> bool:
    try:
        return " avx512f" in Path("/proc/cpuinfo").read_text()
    except OSError:
        return False


def rng_normal(seed: int, count: int) -> np.ndarray:
    """fsk::Rng(seed).normal() x count via the C restatement (rng.hpp:44-57)."""
    lib = C.CDLL(str(build()))
    out = np.empty(count)
    lib.fo_rng_normal_fill(C.c_uint64(seed), C.c_void_p(out.ctypes.data), C.c_int64(count))
    return out
