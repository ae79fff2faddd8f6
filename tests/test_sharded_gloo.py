"""Multi-rank path on CPU: world_size 2 over gloo.

The sharded driver (paper_2602_03067_b200.sharded) is engine-agnostic; here it
drives an oracle-backed stand-in engine, so the shard plan, the in-place
potential all-gathers and the lagged-violation reduction are checked against a
single-process oracle solve without a GPU. The GPU engine itself is checked
row-range by row-range in tests/test_tensor_gpu.py.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2602_03067_b200.sharded import ShardPlan, ShardedSinkhorn, shard_bounds  # noqa: E402


class OracleEngine:
    """Stand-in for fsk.Engine: half-steps over row ranges via the C oracle."""

    def __init__(self, X, a, Y, b, eps):
        from oracle import Oracle
        self.port = Oracle("port")
        self.X, self.a, self.Y, self.b, self.eps = X, a, Y, b, eps
        self.f = self.g = None

    def bind(self, f_ptr, g_ptr):
        pass

    def attach(self, f, g, viol=None):
        self.f, self.g, self.viol = f, g, viol

    def init_potentials(self, stream=0):
        n, m = len(self.a), len(self.b)
        self.f[:n] = torch.from_numpy(-(self.X ** 2).sum(1)).float()
        self.g[:m] = torch.from_numpy(-(self.Y ** 2).sum(1)).float()

    def half_step(self, side, lo, hi, viol_ptr=0, stream=0):
        n, m = len(self.a), len(self.b)
        f = self.f[:n].double().numpy()
        g = self.g[:m].double().numpy()
        if side == 0:
            new = self.port.update_f_hat(self.X[lo:hi], np.full(hi - lo, 1.0 / (hi - lo)),
                                         self.Y, self.b, g, self.eps)
            if viol_ptr:
                r = self.a[lo:hi] * np.exp((f[lo:hi] - new) / self.eps)
                self.viol += float(np.abs(r - self.a[lo:hi]).sum())
            self.f[lo:hi] = torch.from_numpy(new).float()
        else:
            new = self.port.update_g_hat(self.X, self.a, self.Y[lo:hi],
                                         np.full(hi - lo, 1.0 / (hi - lo)), f, self.eps)
            self.g[lo:hi] = torch.from_numpy(new).float()


class OracleTransportEngine(OracleEngine):
    """OracleEngine plus the fixed-potential row-shard transport calls the sharded
    HVP makes (fsk_engine_transport_*), through the C port on row slices (rows are
    independent given the potentials; slice weights renormalised, outputs rescaled
    by the true row weight)."""

    def set_potentials(self, f, g):
        self.fh, self.gh = np.asarray(f, dtype=np.float64), np.asarray(g, dtype=np.float64)

    def transport_prepare(self, f_rows, g_rows, stream=0):
        from oracle import rows as orows
        X, Y, a, b, eps = self.X, self.Y, self.a, self.b, self.eps
        self.marg = [np.zeros(len(a)), np.zeros(len(b))]
        lo, hi = f_rows
        if hi > lo:
            fp = orows.half_step_rows(self.port, 0, X, a, Y, b, self.gh, eps, np.arange(lo, hi))
            self.marg[0][lo:hi] = a[lo:hi] * np.exp((self.fh[lo:hi] - fp) / eps)
        lo, hi = g_rows
        if hi > lo:
            gp = orows.half_step_rows(self.port, 1, X, a, Y, b, self.fh, eps, np.arange(lo, hi))
            self.marg[1][lo:hi] = b[lo:hi] * np.exp((self.gh[lo:hi] - gp) / eps)

    def marginal(self, side, out, stream=0):
        out.copy_(torch.from_numpy(self.marg[side]).float())

    def _rows(self, side, lo, hi, V, A=None):
        from oracle import rows as orows
        X, Y, a, b, eps, f, g = self.X, self.Y, self.a, self.b, self.eps, self.fh, self.gh
        w = orows.slice_weights(hi - lo)
        if side == 0:
            if A is None:
                o = self.port.apply_plan(X[lo:hi], w, Y, b, f[lo:hi], g, eps, V)
            else:
                o = self.port.apply_hadamard_plan(X[lo:hi], w, Y, b, f[lo:hi], g, eps,
                                                  A[lo:hi], Y, V)
            return o * (a[lo:hi] / w)[:, None]
        o = self.port.apply_plan_adjoint(X, a, Y[lo:hi], w, f, g[lo:hi], eps, V)
        return o * (b[lo:hi] / w)[:, None]

    def transport_vec_rows(self, side, lo, hi, v, out, stream=0):
        o = self._rows(side, lo, hi, v.double().numpy()[:, None])[:, 0]
        out[:hi - lo] = torch.from_numpy(o)

    def transport_mat_rows(self, side, lo, hi, V, q, out, A=None, stream=0):
        o = self._rows(side, lo, hi, V.double().numpy(),
                       None if A is None else A.double().numpy())
        out[:hi - lo] = torch.from_numpy(o).float()


def _hvp_worker(rank, world, port, out):
    from paper_2602_03067_b200.sharded import ShardedHvp
    from oracle import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(4)
    n, m, d, eps = 300, 260, 4, 0.5
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d)) * 0.7 + 0.2
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    s = Oracle("port").sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=200)
    A = rng.normal(size=(n, d))
    eng = OracleTransportEngine(X, a, Y, b, eps)
    eng.set_potentials(s["f_hat"], s["g_hat"])
    plan = ShardPlan(rank, world, n, m, align=64)
    h = ShardedHvp(eng, plan, torch.device("cpu"), dist)
    T = lambda z: torch.from_numpy(z)  # noqa: E731
    H, info = h.apply(T(X), T(Y), T(A), eps, tau=1e-5, cg_tol=1e-30, cg_max_iters=25)
    lo, hi = plan.f_bounds[rank]
    out.put((rank, lo, hi, H.numpy(), info, dict(h.counts)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_hvp_matches_composition():
    """ShardedHvp over 2 gloo ranks (2 all-gathers per CG iteration, row-local
    assembly) equals the single-process SPEC composition (oracle/compose.py) to
    the fp32 narrowing of the transport inputs; each rank issues 2 K + 3 vector,
    3 matrix and 1 Hadamard transport calls on its shards (Thm. 3.5 count)."""
    from oracle import Oracle, compose
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_hvp_worker, args=(r, 2, _free_port_once(), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(4)
    n, m, d, eps = 300, 260, 4, 0.5
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d)) * 0.7 + 0.2
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    port = Oracle("port")
    s = port.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=200)
    A = rng.normal(size=(n, d))
    ws = compose.Workspace(port, X, a, Y, b, s["f_hat"], s["g_hat"], eps)
    want, iters, _ = compose.hvp_apply(ws, A, tau=1e-5, tol=1e-30, max_iters=25)
    got = np.zeros_like(want)
    for rank, lo, hi, H, info, counts in res:
        got[lo:hi] = H
        assert info["cg_iters"] == iters == 25
        assert counts == dict(vector=2 * 25 + 3, matrix=3, hadamard=1)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel <= 1e-5, rel


_PORTS = []


def _free_port_once():
    if not _PORTS:
        _PORTS.append(_free_port())
    return _PORTS[0]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    n, m, d, eps = 700, 530, 5, 0.3
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d))
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    eng = OracleEngine(X, a, Y, b, eps)
    plan = ShardPlan(rank, world, n, m, align=64)
    s = ShardedSinkhorn(eng, plan, torch.device("cpu"), dist)
    eng.attach(s.f, s.g, s.viol)
    s.init()
    s.iterate(4)
    # lagged violation: per-rank partials from the next f-update, riding in the payload
    # of that half-step's all-gather (ShardedSinkhorn._gather_with_violation)
    f4 = s.f.clone()
    v = s.iterate(0, track_violation=True)
    assert torch.equal(s.f, f4)   # the extra f-update is discarded
    if rank == 0:
        out.put((s.f[:n].double().numpy(), s.g[:m].double().numpy(), v))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_shard_bounds_cover_rows():
    for rows, world in [(1 << 20, 8), (1000, 3), (5, 4), (256, 2)]:
        b = shard_bounds(rows, world)
        assert b[0][0] == 0 and b[-1][1] == rows
        assert all(b[k][1] == b[k + 1][0] for k in range(world - 1))
        per = b[0][1] - b[0][0]
        assert per % 256 == 0 or per == rows


def test_two_rank_gloo_matches_single_process():
    from oracle import Oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    f, g, viol = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(0)
    n, m, d, eps = 700, 530, 5, 0.3
    X, Y = rng.normal(size=(n, d)), rng.normal(size=(m, d))
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    port_ = Oracle("port")
    fr, gr = -(X ** 2).sum(1), -(Y ** 2).sum(1)
    for _ in range(4):
        fr = port_.update_f_hat(X, a, Y, b, gr, eps)
        gr = port_.update_g_hat(X, a, Y, b, fr, eps)
    assert np.abs(f - fr).max() <= 1e-5 * np.abs(fr).max()
    assert np.abs(g - gr).max() <= 1e-5 * np.abs(gr).max()
    r, _ = port_.induced_marginals(X, a, Y, b, fr, gr, eps)
    want = np.abs(r - a).sum()
    assert abs(viol - want) <= 1e-3 * want + 1e-7
