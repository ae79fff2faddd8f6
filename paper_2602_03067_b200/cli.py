"""Command-line surface (SPEC.md:607-693 `cli`).

    python -m paper_2602_03067_b200.cli gen    out.fsk --n 4096 --d 3 --seed 1
    python -m paper_2602_03067_b200.cli solve  X.fsk Y.fsk --eps 0.1 --iters 100 --precision f32
    python -m paper_2602_03067_b200.cli bench  --n 4096,16384 --d 3,64 --precision f32

FSK1 point-cloud files (SPEC PointCloudFile): magic "FSK1", u16 version (1),
u64 n, u64 d, u8 dtype (0 single, 1 double), u8 has_labels, then the row-major
little-endian payload and, if labelled, n u32 labels. Exit codes follow SPEC:
0 success, 1 validation error, 2 numerical failure. (The SPEC `parity` command is
the test suite, tests/, which checks the kernels against the oracle.)
`bench` prints the SPEC BenchRecord CSV; peak_bytes is the device high-water
mark of the stream-ordered allocator pool during the solve (the GPU analogue of
the reference's heap hook, alloc_hook.cpp) and io_scalars the IoLedger total.
"""
from __future__ import annotations

import argparse
import csv
import struct
import sys
import time
from pathlib import Path

import numpy as np

MAGIC = b"FSK1"
VERSION = 1
_HDR = struct.Struct("<4sHQQBB")
BENCH_HEADER = ["method", "schedule", "n", "m", "d", "eps", "iters", "time_ms", "peak_bytes",
                "io_scalars", "precision"]


class FormatError(ValueError):
    pass


def write_point_cloud(path, points, labels=None, dtype="double") -> None:
    pts = np.ascontiguousarray(points, dtype="<f8" if dtype == "double" else "<f4")
    if pts.ndim != 2:
        raise FormatError("points must be n x d")
    n, d = pts.shape
    with open(path, "wb") as fh:
        fh.write(_HDR.pack(MAGIC, VERSION, n, d, 1 if dtype == "double" else 0,
                           0 if labels is None else 1))
        fh.write(pts.tobytes())
        if labels is not None:
            lab = np.ascontiguousarray(labels, dtype="<u4")
            if lab.shape != (n,):
                raise FormatError("labels must have length n")
            fh.write(lab.tobytes())


def read_point_cloud(path):
    """-> (points float64 n x d, labels uint32 or None)."""
    raw = Path(path).read_bytes()
    if len(raw) < _HDR.size:
        raise FormatError(f"{path}: truncated header ({len(raw)} of {_HDR.size} bytes)")
    magic, ver, n, d, dt, has_lab = _HDR.unpack_from(raw)
    if magic != MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r} (expected {MAGIC!r})")
    if ver != VERSION:
        raise FormatError(f"{path}: unsupported version {ver}")
    if dt not in (0, 1) or has_lab not in (0, 1):
        raise FormatError(f"{path}: bad dtype/label flags")
    width = 8 if dt == 1 else 4
    expect = _HDR.size + n * d * width + (4 * n if has_lab else 0)
    if len(raw) != expect:
        raise FormatError(f"{path}: payload is {len(raw) - _HDR.size} bytes, expected "
                          f"{expect - _HDR.size} (n={n}, d={d}, width={width}, "
                          f"labels={bool(has_lab)})")
    pts = np.frombuffer(raw, dtype="<f8" if dt == 1 else "<f4", count=n * d,
                        offset=_HDR.size).astype(np.float64).reshape(n, d)
    labels = None
    if has_lab:
        labels = np.frombuffer(raw, dtype="<u4", count=n, offset=_HDR.size + n * d * width).copy()
    return pts, labels


def read_csv_cloud(path):
    """CSV with header x0,...,x{d-1}[,label]; uniform weights are implied."""
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    head, body = rows[0], rows[1:]
    has_lab = head[-1] == "label"
    d = len(head) - (1 if has_lab else 0)
    pts = np.array([[float(v) for v in r[:d]] for r in body])
    labels = np.array([int(r[d]) for r in body], dtype=np.uint32) if has_lab else None
    return pts, labels


def load_cloud(path):
    return read_csv_cloud(path) if str(path).endswith(".csv") else read_point_cloud(path)


def uniform(n):
    w = np.full(n, 1.0 / n)
    if n > 1:
        w[-1] = 1.0 - np.cumsum(w[:-1])[-1]  # passes the naive-sum check (core.cpp:27-33)
    return w


def _device_pool_peak_reset():
    try:
        import torch
        if not torch.cuda.is_available():
            return None
        from cuda.bindings import driver, runtime as rt  # cuda-python
        err, pool = rt.cudaDeviceGetDefaultMemPool(torch.cuda.current_device())
        rt.cudaMemPoolSetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemHigh,
                                   driver.cuuint64_t(0))
        return pool
    except Exception:
        return None


def _device_pool_peak(pool):
    if pool is None:
        return -1
    try:
        from cuda.bindings import runtime as rt
        err, v = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemHigh)
        return int(v)
    except Exception:
        return -1


def cmd_gen(a) -> int:
    import paper_2602_03067_b200 as fsk
    pts = fsk.rng_normal(a.seed, a.n * a.d).reshape(a.n, a.d)  # fsk::Rng(seed).normal()
    write_point_cloud(a.out, pts, dtype="single" if a.single else "double")
    return 0


def cmd_solve(a) -> int:
    import paper_2602_03067_b200 as fsk
    X, _ = load_cloud(a.X)
    Y, _ = load_cloud(a.Y)
    led = fsk.Ledger()
    out = fsk.sinkhorn_solve(X, uniform(len(X)), Y, uniform(len(Y)), eps=a.eps,
                             schedule="symmetric" if a.schedule == "sym" else "alternating",
                             max_iters=a.iters, marginal_tol=a.tol,
                             eps_scaling_factor=a.eps_scale,
                             precision="single" if a.precision == "f32" else "double",
                             tiles=(a.tile_bn, a.tile_bm), ledger=led)
    print(f"dual_cost {out['dual_cost']:.17g}")
    print(f"iterations {out['iterations']}")
    print(f"marginal_violation {out['marginal_violation']:.6e}")
    print(f"io_scalars {led.total_scalars()}")
    if a.potentials:
        np.savez(a.potentials, f_hat=out["f_hat"], g_hat=out["g_hat"])
    return 0


def cmd_bench(a) -> int:
    import paper_2602_03067_b200 as fsk
    w = csv.writer(sys.stdout, lineterminator="\n")
    w.writerow(BENCH_HEADER)
    for n in [int(v) for v in a.n.split(",")]:
        for d in [int(v) for v in a.d.split(",")]:
            z = fsk.rng_normal(a.seed, 2 * n * d)
            X, Y = z[: n * d].reshape(n, d), z[n * d:].reshape(n, d)
            wts = uniform(n)
            for sched in a.schedule.split(","):
                prec = "single" if a.precision == "f32" else "double"
                kw = dict(eps=a.eps, max_iters=a.iters, precision=prec,
                          schedule="symmetric" if sched == "sym" else "alternating")
                fsk.sinkhorn_solve(X, wts, Y, wts, **kw)  # warm-up (module load, pools)
                led = fsk.Ledger()
                pool = _device_pool_peak_reset()
                t0 = time.perf_counter()
                fsk.sinkhorn_solve(X, wts, Y, wts, ledger=led, **kw)
                ms = (time.perf_counter() - t0) * 1e3
                w.writerow(["stream", sched, n, n, d, a.eps, a.iters,
                            0 if a.deterministic else f"{ms:.3f}", _device_pool_peak(pool),
                            led.total_scalars(), a.precision])
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="fsk")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen")
    g.add_argument("out")
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--d", type=int, required=True)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--single", action="store_true")
    s = sub.add_parser("solve")
    s.add_argument("X")
    s.add_argument("Y")
    s.add_argument("--eps", type=float, default=0.1)
    s.add_argument("--iters", type=int, default=100)
    s.add_argument("--tol", type=float, default=0.0)
    s.add_argument("--schedule", choices=["alt", "sym"], default="alt")
    s.add_argument("--eps-scale", type=float, default=1.0)
    s.add_argument("--tile-bn", type=int, default=64)
    s.add_argument("--tile-bm", type=int, default=64)
    s.add_argument("--precision", choices=["f32", "f64"], default="f64")
    s.add_argument("--potentials")
    b = sub.add_parser("bench")
    b.add_argument("--n", default="4096")
    b.add_argument("--d", default="3")
    b.add_argument("--eps", type=float, default=0.1)
    b.add_argument("--iters", type=int, default=10)
    b.add_argument("--schedule", default="alt")
    b.add_argument("--precision", choices=["f32", "f64"], default="f32")
    b.add_argument("--seed", type=int, default=1000)
    b.add_argument("--deterministic", action="store_true")
    a = ap.parse_args(argv)
    import paper_2602_03067_b200 as fsk
    try:
        return {"gen": cmd_gen, "solve": cmd_solve, "bench": cmd_bench}[a.cmd](a)
    except (FormatError, fsk.ValidationError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except fsk.NumericalError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
