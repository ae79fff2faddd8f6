"""Row-sharded Sinkhorn over N GPUs of one box.

Each rank holds both clouds resident (an ``Engine``), updates only its shard of
rows of f (rows of X) and of g (rows of Y) per half-step, and the only
communication is an in-place all-gather of the length-n / length-m fp32
potential vector after each half-iteration (NCCL over NVLink when the process
group is NCCL). The lagged marginal violation of the previous iterate is a
fused by-product of the f-update epilogue; its per-rank partials are summed
with one all-reduce only when early stopping asks for it.

The driver is engine-agnostic: ``half_step(side, lo, hi, viol_ptr)`` and
``grad(lo, hi, out)`` are the only calls it makes, so the same logic is
exercised on CPU with gloo and an oracle-backed engine in the tests.
"""
from __future__ import annotations

from dataclasses import dataclass


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
        if self.dist is None or self.plan.world == 1:
            return
        k = self.plan.rank
        if self.dist.get_backend(self.group) == "nccl":
            # in place: rank k's slice is the send buffer (NVLink / NVSwitch)
            self.dist.all_gather_into_tensor(buf, buf[k * per:(k + 1) * per], group=self.group)
        else:
            parts = list(buf.split(per))
            self.dist.all_gather(parts, parts[k].clone(), group=self.group)
            buf.copy_(self.torch.cat(parts))

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
            self.viol.zero_()
            f_save = self.f.clone()
            self.engine.half_step(0, flo, fhi, self.viol.data_ptr(), st)
            self.f.copy_(f_save)
            if self.dist is not None and p.world > 1:
                self.dist.all_reduce(self.viol, group=self.group)
            return float(self.viol.item())
        return None

    def grad_shard(self, out):
        """Gradient rows of this rank's shard of X into `out` ((hi-lo) x d)."""
        lo, hi = self.plan.f_bounds[self.plan.rank]
        self.engine.grad(lo, hi, out.data_ptr(), self._stream())
        return lo, hi
