"""Multi-GPU driver paths on the one reachable B200.

* ShardedHvp (2 all-gathers per CG iteration) on the real engine, world 1 and two
  gloo ranks sharing the device, against the single-process fsk_hvp_apply_single;
* the NCCL branch of the shard all-gather (all_gather_into_tensor, in place) and
  the violation payload, through a world-size-1 NCCL process group;
* two gloo ranks sharing the device: the sharded Sinkhorn and its piggybacked
  lagged violation against one engine.
The multi-rank logic itself is also covered on CPU (tests/test_sharded_gloo.py).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _problem(n=1300, m=1100, d=64, eps=0.2, seed=3):
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(n, d)) * 0.5
    Y = rng.normal(size=(m, d)) * 0.5 + 0.05
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    return X, a, Y, b, eps


def _sharded_hvp(fsk, rank, world, dist_mod, X, a, Y, b, eps, f, g, A, K):
    from paper_2602_03067_b200.sharded import ShardedHvp, ShardPlan
    n, m = len(X), len(Y)
    dev = torch.device("cuda", 0)
    eng = fsk.Engine(0, X, a, Y, b, mode="tensor")
    eng.set_eps(eps)
    ft = torch.tensor(f, dtype=torch.float32, device=dev)
    gt = torch.tensor(g, dtype=torch.float32, device=dev)
    eng.bind(ft.data_ptr(), gt.data_ptr())
    plan = ShardPlan(rank, world, n, m)
    h = ShardedHvp(eng, plan, dev, dist_mod)
    T = lambda z: torch.tensor(z, dtype=torch.float64, device=dev)  # noqa: E731
    H, info = h.apply(T(X), T(Y), T(A), eps, tau=1e-5, cg_tol=1e-30, cg_max_iters=K)
    torch.cuda.synchronize()
    lo, hi = plan.f_bounds[rank]
    out = (lo, hi, H.cpu().numpy(), info, dict(h.counts))
    eng.close()
    return out


def _reference_hvp(fsk, X, a, Y, b, eps, K):
    s = fsk.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=30, precision="single")
    f, g = s["f_hat"].astype(np.float32).astype(np.float64), \
        s["g_hat"].astype(np.float32).astype(np.float64)
    A = np.random.default_rng(9).standard_normal(X.shape)
    os.environ["FSK_TENSOR_MODE"] = "tensor"
    try:
        H, info = fsk.hvp_apply(X, a, Y, b, f, g, eps, A, tau=1e-5, cg_tol=1e-30,
                                cg_max_iters=K, precision="single")
    finally:
        os.environ.pop("FSK_TENSOR_MODE", None)
    return f, g, A, H, info


def test_sharded_hvp_world1_matches_single_process_hvp(fsk):
    X, a, Y, b, eps = _problem()
    f, g, A, want, info = _reference_hvp(fsk, X, a, Y, b, eps, 20)
    lo, hi, H, sinfo, counts = _sharded_hvp(fsk, 0, 1, None, X, a, Y, b, eps, f, g, A, 20)
    rel = np.linalg.norm(H - want) / np.linalg.norm(want)
    print(f"sharded HVP (world 1) vs fsk_hvp_apply_single: rel {rel:.2e}")
    assert (lo, hi) == (0, len(X)) and sinfo["cg_iters"] == info["cg_iters"] == 20
    assert counts == dict(vector=2 * 20 + 3, matrix=3, hadamard=1)
    assert rel <= 1e-5


def _hvp_worker(rank, world, port, q, K):
    import paper_2602_03067_b200 as fsk
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    X, a, Y, b, eps = _problem()
    z = np.load(os.environ["FSK_TEST_FGA"] + ".npz")
    f, g, A = z["f"], z["g"], z["A"]
    q.put((rank,) + _sharded_hvp(fsk, rank, world, dist, X, a, Y, b, eps, f, g, A, K))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_hvp_two_gloo_ranks_on_one_gpu(fsk, tmp_path):
    """Two ranks (gloo, CUDA tensors) each updating their 256-aligned shards: the
    gathered HVP equals the single-process one."""
    X, a, Y, b, eps = _problem()
    f, g, A, want, _ = _reference_hvp(fsk, X, a, Y, b, eps, 15)
    base = str(tmp_path / "fga")
    np.savez(base + ".npz", f=f, g=g, A=A)
    os.environ["FSK_TEST_FGA"] = base
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hvp_worker, args=(r, 2, port, q, 15)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = np.zeros_like(want)
    for rank, lo, hi, H, info, counts in res:
        got[lo:hi] = H
        assert counts == dict(vector=2 * 15 + 3, matrix=3, hadamard=1)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    print(f"sharded HVP (2 gloo ranks, one B200) vs fsk_hvp_apply_single: rel {rel:.2e}")
    assert rel <= 1e-5


def test_nccl_world1_gather_and_violation_payload(fsk):
    """The NCCL branch (in-place all_gather_into_tensor) and the violation payload
    path, through a world-size-1 NCCL group: the sharded loop equals the engine's
    own iterate, and the piggybacked lagged violation equals the fused one."""
    from paper_2602_03067_b200.sharded import ShardPlan, ShardedSinkhorn
    X, a, Y, b, eps = _problem(n=2000, m=1800)
    n, m = len(X), len(Y)
    store = dist.TCPStore("127.0.0.1", _free_port(), 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        dev = torch.device("cuda", 0)
        eng = fsk.Engine(0, X, a, Y, b)
        eng.set_eps(eps)
        plan = ShardPlan(0, 1, n, m)
        s = ShardedSinkhorn(eng, plan, dev, dist)
        assert dist.get_backend() == "nccl"
        s.init()
        s.iterate(6)
        buf = s.f.clone()
        s._gather(buf, plan.f_per)     # NCCL all_gather_into_tensor, in place
        assert torch.equal(buf, s.f)
        v = s.iterate(0, track_violation=True)
        f1, g1 = s.f.clone(), s.g.clone()
        eng.close()
        eng2 = fsk.Engine(0, X, a, Y, b)
        eng2.set_eps(eps)
        f2 = torch.empty(n, dtype=torch.float32, device=dev)
        g2 = torch.empty(m, dtype=torch.float32, device=dev)
        eng2.bind(f2.data_ptr(), g2.data_ptr())
        eng2.init_potentials()
        eng2.iterate(6)
        torch.cuda.synchronize()
        f6 = f2.clone()
        vv = torch.zeros(1, dtype=torch.float64, device=dev)
        eng2.half_step(0, 0, n, vv.data_ptr())
        torch.cuda.synchronize()
        # same kernels, same deterministic skip decisions: identical bits
        assert torch.equal(f1[:n], f6) and torch.equal(g1[:m], g2)
        assert abs(v - float(vv.item())) <= 1e-7 * float(vv.item())
        eng2.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("precision,tol", [("single", 0.0), ("double", 0.0), ("double", 1e-7)])
def test_in_library_multi_device_solve_matches_single_device(fsk, port, precision, tol):
    """fsk_set_num_devices(1): sinkhorn_solve(_grad) through the in-library NCCL path
    (one host thread + stream per device, ncclCommInitAll, all-gather of the potential
    shards after every half-step, fused early stop with the violation all-reduce in
    the same NCCL group) returns what the single-device path returns: same iterate
    count, potentials, loss, violation, gradient, ledger."""
    X, a, Y, b, eps = _problem(n=3000, m=2600, d=64, eps=0.2)
    kw = dict(eps=eps, max_iters=300 if tol else 12, marginal_tol=tol, precision=precision,
              grad=True)
    l0, l1 = fsk.Ledger(), fsk.Ledger()
    want = fsk.sinkhorn_solve(X, a, Y, b, ledger=l0, **kw)
    fsk.set_num_devices(1)
    try:
        got = fsk.sinkhorn_solve(X, a, Y, b, ledger=l1, **kw)
    finally:
        fsk.set_num_devices(0)
    print(f"{precision} tol={tol}: iterations {got['iterations']} vs {want['iterations']}, "
          f"loss {got['dual_cost']!r} vs {want['dual_cost']!r}")
    assert got["iterations"] == want["iterations"]
    for key in ("f_hat", "g_hat", "grad"):
        ref = want[key]
        err = np.abs(got[key] - ref).max() / max(1.0, np.abs(ref).max())
        assert err <= (1e-12 if precision == "double" else 1e-6), (key, err)
    assert abs(got["dual_cost"] - want["dual_cost"]) <= 1e-12 * abs(want["dual_cost"]) + (
        0.0 if precision == "double" else 1e-7 * abs(want["dual_cost"]))
    assert abs(got["marginal_violation"] - want["marginal_violation"]) <= \
        1e-9 * want["marginal_violation"] + (0.0 if precision == "double" else 1e-6)
    assert l0.total_scalars() == l1.total_scalars()


def test_in_library_multi_device_rejects_missing_devices(fsk):
    X, a, Y, b, eps = _problem(n=300, m=260, d=8)
    fsk.set_num_devices(fsk.lib().fsk_device_count() + 1)
    try:
        with pytest.raises(fsk.ValidationError):
            fsk.sinkhorn_solve(X, a, Y, b, eps=eps, max_iters=3)
    finally:
        fsk.set_num_devices(0)
