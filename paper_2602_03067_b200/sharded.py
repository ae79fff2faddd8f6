"""Row-sharded Sinkhorn over N GPUs of one box.

Each rank holds both clouds resident (an ``Engine``), updates only its shard of
rows of f (rows of X) and of g (rows of Y) per half-step, and the only
communication is an in-place all-gather of the length-n / length-m fp32
potential vector after each half-iteration (NCCL over NVLink when the process
group is NCCL). The lagged marginal violation of the previous iterate is a
fused by-product of the f-update epilogue; its per-rank partials ride in the
payload of that half-step's all-gather (no separate collective).

The driver is engine-agnostic: ``half_step(side, lo, hi, viol_ptr)`` and
``grad(lo, hi, out)`` are the only calls it makes, so the same logic is
exercised on CPU with gloo and an oracle-backed engine in the tests.

``ShardedHvp`` is the HVP over the same shards: every Schur
product S v = c v - P^T diag(r)^-1 P v + tau v is one transport-vector pass on the
rank's rows of X, an all-gather (n), one pass on its rows of Y and an all-gather
(m) - the 2 all-gathers per CG iteration of SURVEY §8e; the CG vectors (length m)
are replicated and their algebra is redundant on every rank.
"""
from __future__ import annotations

from dataclasses import dataclass


def all_gather_shards(dist, group, buf, per, rank, world):
    """In-place all-gather of `buf` (world * per), rank k owning [k per, (k+1) per).
    (A world-size-1 group still runs the collective: that is how the NCCL branch is
    exercised on a single device.)"""
    if dist is None:
        return
    if dist.get_backend(group) == "nccl":
        # in place: rank k's slice is the send buffer (NVLink / NVSwitch)
        dist.all_gather_into_tensor(buf, buf[rank * per:(rank + 1) * per], group=group)
    else:
        import torch
        parts = list(buf.split(per))
        dist.all_gather(parts, parts[rank].clone(), group=group)
        buf.copy_(torch.cat(parts))


def shard_bounds(rows: int, world: int, align: int = 256) -> list[tuple[int, int]]:
    """Contiguous equal shards of `align`-multiple size (the last one ragged):
    shard k is [k S, min((k+1) S, rows)) with S = ceil(rows / world / align) align."""
    per = -(-rows // world)
    per = -(-per // align) * align
    return [(min(k * per, rows), min((k + 1) * per, rows)) for k in range(world)]


@dataclass
class ShardPlan:
    rank: int
    world: int
    n: int
    m: int
    align: int = 256

    def __post_init__(self):
        self.f_bounds = shard_bounds(self.n, self.world, self.align)
        self.g_bounds = shard_bounds(self.m, self.world, self.align)
        self.f_per = self.f_bounds[0][1] - self.f_bounds[0][0] if self.n else 0
        self.g_per = self.g_bounds[0][1] - self.g_bounds[0][0] if self.m else 0
        # gather buffers are world * per long; the first n (m) entries are the potential
        self.f_len = self.world * self.f_per
        self.g_len = self.world * self.g_per


class ShardedSinkhorn:
    """Alternating Sinkhorn with sharded rows and potential all-gathers.

    torch is used for device buffers, streams and torch.distributed only.
    """

    def __init__(self, engine, plan: ShardPlan, device, dist=None, group=None,
                 dtype=None):
        import torch

        self.torch = torch
        self.engine = engine
        self.plan = plan
        self.dist = dist
        self.group = group
        dt = dtype or torch.float32
        self.f = torch.zeros(plan.f_len, dtype=dt, device=device)
        self.g = torch.zeros(plan.g_len, dtype=dt, device=device)
        self.viol = torch.zeros(1, dtype=torch.float64, device=device)
        engine.bind(self.f.data_ptr(), self.g.data_ptr())

    def _stream(self):
        # the engine launches on torch's current stream so its kernels are
        # ordered with the collectives torch issues on that stream
        if self.torch.cuda.is_available() and self.f.is_cuda:
            return self.torch.cuda.current_stream(self.f.device).cuda_stream
        return 0

    def _gather(self, buf, per):
        all_gather_shards(self.dist, self.group, buf, per, self.plan.rank, self.plan.world)

    def _gather_with_violation(self, buf, per, viol_partial):
        """All-gather of the potential shards with each rank's violation partial riding
        in the same payload (2 extra fp32 words per rank: the fp64 partial as hi + lo):
        one collective per half-step; returns the summed violation (fp64)."""
        torch = self.torch
        k, world = self.plan.rank, self.plan.world
        if self.dist is None:
            return float(viol_partial.item())
        stride = per + 2
        pay = self._pay if getattr(self, "_pay", None) is not None and \
            self._pay.numel() == world * stride else torch.empty(world * stride, dtype=buf.dtype,
                                                                 device=buf.device)
        self._pay = pay
        mine = pay[k * stride:(k + 1) * stride]
        mine[:per].copy_(buf[k * per:(k + 1) * per])
        hi = viol_partial.to(torch.float32)
        mine[per:per + 1].copy_(hi)
        mine[per + 1:per + 2].copy_((viol_partial - hi.double()).to(torch.float32))
        all_gather_shards(self.dist, self.group, pay, stride, k, world)
        grid = pay.view(world, stride)
        buf[:world * per].view(world, per).copy_(grid[:, :per])
        return float(grid[:, per].double().sum().item() + grid[:, per + 1].double().sum().item())

    def init(self):
        self.engine.init_potentials(self._stream())

    def iterate(self, iters: int, track_violation: bool = False):
        """`iters` alternating iterations; returns the lagged violation of the
        last completed iterate when track_violation (needs one extra f pass)."""
        p = self.plan
        flo, fhi = p.f_bounds[p.rank]
        glo, ghi = p.g_bounds[p.rank]
        st = self._stream()
        for _ in range(iters):
            self.engine.half_step(0, flo, fhi, 0, st)
            self._gather(self.f, p.f_per)
            self.engine.half_step(1, glo, ghi, 0, st)
            self._gather(self.g, p.g_per)
        if track_violation:
            # the next f-update's epilogue yields sum |r - a| of the current iterate
            # (SURVEY §8a); the partials ride in the potential all-gather's payload
            self.viol.zero_()
            f_save = self.f.clone()
            self.engine.half_step(0, flo, fhi, self.viol.data_ptr(), st)
            v = self._gather_with_violation(self.f, p.f_per, self.viol)
            self.f.copy_(f_save)
            return v
        return None

    def grad_shard(self, out):
        """Gradient rows of this rank's shard of X into `out` ((hi-lo) x d)."""
        lo, hi = self.plan.f_bounds[self.plan.rank]
        self.engine.grad(lo, hi, out.data_ptr(), self._stream())
        return lo, hi


class ShardedHvp:
    """Hessian-vector product of OT_eps w.r.t. X (Thm. 3.5) at the
    engine's bound potentials, rows of X and Y sharded as in ``ShardPlan``.

    Same composition as oracle/compose.py hvp_apply and csrc/hvp.cpp: build_rhs
    (SPEC.md:458-466), damped Schur CG (:468-486), R^T w + E.A (:448-456, :488-496).
    Row-local terms (P Y, u_P, w1, P (w2 Y), the Hadamard term) stay on the rank; the
    length-n / length-m vectors that feed a transpose pass are all-gathered. Vector
    algebra in fp64 torch tensors on the engine's device; transport inputs narrow to
    fp32 as in fsk_hvp_apply_single.
    """

    def __init__(self, engine, plan: ShardPlan, device, dist=None, group=None):
        import torch

        self.torch = torch
        self.engine = engine
        self.plan = plan
        self.device = device
        self.dist = dist
        self.group = group
        self.counts = dict(vector=0, matrix=0, hadamard=0)

    def _stream(self):
        t = self.torch
        if t.cuda.is_available() and self.device.type == "cuda":
            return t.cuda.current_stream(self.device).cuda_stream
        return 0

    def _full(self, shard, which):
        """All-gather a row-shard vector (fp64) to its full length (which: 'f' n, 'g' m)."""
        p = self.plan
        per, total = (p.f_per, p.n) if which == "f" else (p.g_per, p.m)
        lo, hi = (p.f_bounds if which == "f" else p.g_bounds)[p.rank]
        buf = self.torch.zeros(p.world * per, dtype=self.torch.float64, device=self.device)
        buf[p.rank * per:p.rank * per + (hi - lo)] = shard
        all_gather_shards(self.dist, self.group, buf, per, p.rank, p.world)
        return buf[:total]

    def _vec(self, side, v):
        p, t = self.plan, self.torch
        lo, hi = (p.f_bounds if side == 0 else p.g_bounds)[p.rank]
        out = t.empty(max(hi - lo, 1), dtype=t.float64, device=self.device)
        if hi > lo:
            self.engine.transport_vec_rows(side, lo, hi, v.to(t.float32).contiguous(), out,
                                           self._stream())
        self.counts["vector"] += 1
        return out[:hi - lo]

    def _mat(self, side, V, A=None):
        p, t = self.plan, self.torch
        lo, hi = (p.f_bounds if side == 0 else p.g_bounds)[p.rank]
        q = V.shape[1]
        out = t.empty((max(hi - lo, 1), q), dtype=t.float32, device=self.device)
        if hi > lo:
            self.engine.transport_mat_rows(side, lo, hi, V.to(t.float32).contiguous(), q, out,
                                           None if A is None else A.to(t.float32).contiguous(),
                                           self._stream())
        self.counts["hadamard" if A is not None else "matrix"] += 1
        return out[:hi - lo].double()

    def apply(self, X, Y, A, eps, tau=1e-5, cg_tol=1e-6, cg_max_iters=50):
        """HVP rows of this rank's shard of X ((hi - lo) x d, fp64) along A (n x d) at
        the engine's potentials and eps. X, Y, A: fp64 tensors on the device,
        replicated on every rank."""
        t = self.torch
        p = self.plan
        flo, fhi = p.f_bounds[p.rank]
        glo, ghi = p.g_bounds[p.rank]
        eng, st = self.engine, self._stream()
        eng.transport_prepare((flo, fhi), (glo, ghi), st)
        rs_ = t.zeros(p.n, dtype=t.float32, device=self.device)
        cs_ = t.zeros(p.m, dtype=t.float32, device=self.device)
        eng.marginal(0, rs_, st)
        eng.marginal(1, cs_, st)
        r = self._full(rs_[flo:fhi].double(), "f")
        c = self._full(cs_[glo:ghi].double(), "g")
        eps = float(eps)
        # build_rhs
        PY = self._mat(0, Y)                                   # rows [flo, fhi)
        u = (X * A).sum(1)
        uP = (PY * A[flo:fhi]).sum(1)
        r1 = self._full(2.0 * (r[flo:fhi] * u[flo:fhi] - uP), "f")
        Ptu = self._vec(1, u)
        PtA = self._mat(1, A)
        r2 = 2.0 * (Ptu - (PtA * Y[glo:ghi]).sum(1))
        rhs = self._full(r2 - self._vec(1, r1 / r), "g")
        # damped Schur CG from 0, replicated vectors

        def schur(v):
            q = self._full(self._vec(0, v), "f")
            z = self._full(self._vec(1, q / r), "g")
            return c * v - z + tau * v

        w2 = t.zeros_like(rhs)
        rn0 = float(t.linalg.norm(rhs))
        iters, relres, converged = 0, 0.0, True
        if rn0 > 0.0:
            res = rhs.clone()
            pdir = rhs.clone()
            rs = float(res @ res)
            converged = False
            while iters < cg_max_iters:
                Ap = schur(pdir)
                alpha = rs / float(pdir @ Ap)
                w2 += alpha * pdir
                res -= alpha * Ap
                iters += 1
                rs_new = float(res @ res)
                if rs_new ** 0.5 <= cg_tol * rn0:
                    converged = True
                    rs = rs_new
                    break
                pdir = res + (rs_new / rs) * pdir
                rs = rs_new
            relres = rs ** 0.5 / rn0
        # R^T w + E.A on this rank's rows
        Pw2 = self._vec(0, w2)
        rl = r[flo:fhi]
        w1 = (r1[flo:fhi] - Pw2) / rl
        Pw2Y = self._mat(0, w2[:, None] * Y)
        B5 = self._mat(0, Y, A=A)
        Xl, Al, ul, uPl = X[flo:fhi], A[flo:fhi], u[flo:fhi], uP
        RTw = 2.0 * ((rl * w1)[:, None] * Xl - w1[:, None] * PY + Pw2[:, None] * Xl - Pw2Y)
        EA = 2.0 * rl[:, None] * Al - (4.0 / eps) * ((rl * ul)[:, None] * Xl - ul[:, None] * PY
                                                     - uPl[:, None] * Xl + B5)
        return RTw / eps + EA, dict(cg_iters=iters, cg_rel_residual=relres, converged=converged)
