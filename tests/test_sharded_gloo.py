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

    def attach(self, f, g):
        self.f, self.g = f, g

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
                self.viol_acc += np.abs(r - self.a[lo:hi]).sum()
            self.f[lo:hi] = torch.from_numpy(new).float()
        else:
            new = self.port.update_g_hat(self.X, self.a, self.Y[lo:hi],
                                         np.full(hi - lo, 1.0 / (hi - lo)), f, self.eps)
            self.g[lo:hi] = torch.from_numpy(new).float()


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
    eng.attach(s.f, s.g)
    s.init()
    s.iterate(4)
    # lagged violation: per-rank partial via the engine, summed across ranks
    eng.viol_acc = 0.0
    flo, fhi = plan.f_bounds[rank]
    f_save = s.f.clone()
    eng.half_step(0, flo, fhi, viol_ptr=1)
    s.f.copy_(f_save)
    v = torch.tensor([eng.viol_acc], dtype=torch.float64)
    dist.all_reduce(v)
    if rank == 0:
        out.put((s.f[:n].double().numpy(), s.g[:m].double().numpy(), float(v.item())))
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
