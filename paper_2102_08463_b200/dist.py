"""Multi-GPU NUFFT: one process per GPU over torch.distributed (NCCL).

The reference's multi-GPU story is the paper's M-TIP application: one MPI
rank per GPU, independent transforms, mpi4py scatter/reduce on the host
(PAPER.md:1583-1597).  Here the work shards only where it naturally does
(SURVEY.md §8e):

* ``ReplicaPlan``   -- independent transforms per rank, no collective on
                       the hot path (the M-TIP pattern; optional final
                       reduce of per-rank results, as mpi4py.reduce).
* ``ShardedPlan`` type 2 -- the points are split across ranks (contiguous
                       slices of the input order); the root's modes are
                       broadcast, every rank pads + inverse-FFTs the
                       replicated fine grid and interpolates its own points.
* ``ShardedPlan`` type 1 -- the points are split across ranks; each rank
                       spreads its slice into a full fine grid, the grids are
                       summed with an NCCL reduce (or all-reduce) and the
                       root runs FFT + deconvolution.

The compute steps go through a ``StageOps`` object so the collective logic
can be exercised on CPU (gloo) with any implementation of the four steps;
the product ops are ``CudaStageOps`` (libnufft_b200 kernels + cuFFT).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

__all__ = ["shard_bounds", "CudaStageOps", "ShardedPlan", "ReplicaPlan"]


def shard_bounds(M, world, rank):
    """Contiguous near-equal slice [lo, hi) of range(M) owned by ``rank``
    (same split rule as the reference's _parallel.chunk_bounds,
    _parallel.py:32-42, over ranks instead of threads)."""
    step, extra = divmod(int(M), int(world))
    lo = rank * step + min(rank, extra)
    hi = lo + step + (1 if rank < extra else 0)
    return lo, hi


class CudaStageOps:
    """The four NUFFT steps on this rank's GPU, over a TransformPlan."""

    def __init__(self, plan):
        self.plan = plan
        self.fine = plan.new_fine_grid()

    def spread(self, strengths):
        return self.plan.spread_to(strengths, self.fine)

    def fft_deconvolve(self, fine, out):
        return self.plan.fft_deconvolve_to(fine, out)

    def pad_ifft(self, modes):
        self.plan.pad_to(modes, self.fine)
        return self.plan.fft_(self.fine, +1)

    def execute_type2(self, modes, out):
        """The whole type-2 execute on this rank's points (fused pad + FFT +
        interp, CUDA-graph replay on fixed buffers) once the modes are here."""
        return self.plan.execute(modes, out)

    def interp(self, fine, out=None):
        if out is None:
            out = self.new_values(self.plan.num_points)
        return self.plan.interp_to(fine, out)

    def new_modes(self):
        p = self.plan
        return torch.empty(p._batch(p.grid.mode_shape), dtype=self.fine.dtype,
                           device=self.fine.device)

    def new_values(self, n):
        return torch.empty(self.plan._batch((n,)), dtype=self.fine.dtype,
                           device=self.fine.device)


class ShardedPlan:
    """A type-1 or type-2 transform whose points are sharded over the ranks
    of ``group``.  Each rank holds only its own points and strengths (or
    output values); the uniform side lives on ``root`` (type 1 output, type 2
    input), or on every rank with ``all_ranks=True``.

    Args:
        ops: StageOps for this rank (CudaStageOps over a plan whose points are
             this rank's shard).
        nufft_type: 1 or 2.
        root: rank that owns the modes.
        all_ranks: type 1: all-reduce the fine grid so every rank gets the
             modes; type 2: skip the broadcast (every rank already has f).
    """

    def __init__(self, ops, nufft_type, group=None, root=0, all_ranks=False):
        if nufft_type not in (1, 2):
            raise ValueError("nufft_type must be 1 or 2")
        self.ops = ops
        self.type = nufft_type
        self.group = group
        self.root = root
        self.all_ranks = all_ranks
        self.rank = dist.get_rank(group)
        # ``root`` is a rank of ``group``; torch's reduce(dst=) / broadcast(src=)
        # take global ranks
        self.root_global = root if group is None else dist.get_global_rank(group, root)

    def execute(self, inp, out=None):
        """type 1: inp = this rank's strengths -> modes (root / all ranks,
        None elsewhere).  type 2: inp = modes (read on root) -> this rank's
        values."""
        if self.type == 1:
            fine = self.ops.spread(inp)
            if self.all_ranks:
                dist.all_reduce(fine, op=dist.ReduceOp.SUM, group=self.group)
            else:
                dist.reduce(fine, dst=self.root_global, op=dist.ReduceOp.SUM, group=self.group)
                if self.rank != self.root:
                    return None
            out = self.ops.new_modes() if out is None else out
            return self.ops.fft_deconvolve(fine, out)
        if not self.all_ranks:
            dist.broadcast(inp, src=self.root_global, group=self.group)
        if hasattr(self.ops, "execute_type2"):
            if out is None:
                out = self.ops.new_values(self.ops.plan.num_points)
            return self.ops.execute_type2(inp, out)
        fine = self.ops.pad_ifft(inp)
        return self.ops.interp(fine, out)


class ReplicaPlan:
    """Independent per-rank transforms (the paper's one-rank-per-GPU M-TIP
    pattern): execute() runs the rank's own plan with no communication;
    ``reduce_result`` is the optional end-of-iteration merge that the
    application does with mpi4py.reduce."""

    def __init__(self, plan, group=None, root=0):
        self.plan = plan
        self.group = group
        self.root = root

    def execute(self, inp, out=None):
        return self.plan.execute(inp, out)

    def reduce_result(self, t):
        dst = self.root if self.group is None else dist.get_global_rank(self.group, self.root)
        dist.reduce(t, dst=dst, op=dist.ReduceOp.SUM, group=self.group)
        return t
