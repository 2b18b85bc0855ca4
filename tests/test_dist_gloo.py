"""Multi-process (world_size 2, gloo, CPU) tests of the sharding logic in
paper_2102_08463_b200/dist.py.  The four compute steps are supplied by the
CPU oracle (test infrastructure) so the collectives -- type-1 fine-grid
reduce / all-reduce, type-2 mode broadcast, replica reduce -- run here
without a GPU; on a GPU box the same classes run with CudaStageOps/NCCL."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODES = (20, 18)
EPS = 1e-9
M = 3001


class OracleOps:
    """StageOps backed by the CPU oracle for this rank's point shard."""

    def __init__(self, orc, pts, nufft_type):
        self.orc = orc
        self.p = orc.OraclePlan(nufft_type, MODES, EPS, "sm" if nufft_type == 1 else "gmsort")
        self.p.set_points(pts)

    def spread(self, c):
        return torch.from_numpy(self.p.spread(c.numpy()))

    def fft_deconvolve(self, fine, out):
        o = self.orc
        bh = o.fft_fine(fine.numpy(), "forward")
        out.copy_(torch.from_numpy(o.deconvolve_type1(bh, self.p.grid, self.p.params, self.p.corr)))
        return out

    def pad_ifft(self, modes):
        o = self.orc
        bh = o.deconvolve_type2(modes.numpy(), self.p.grid, self.p.params, self.p.corr)
        return torch.from_numpy(o.fft_fine(bh, "inverse"))

    def interp(self, fine, out=None):
        o = self.orc
        return torch.from_numpy(o.interpolate(self.p.points, fine.numpy(), self.p.params,
                                              self.p.grid, self.p.layout))

    def new_modes(self):
        return torch.zeros(MODES[::-1], dtype=torch.complex128)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from oracle import oracle as orc
    from paper_2102_08463_b200.dist import ReplicaPlan, ShardedPlan, shard_bounds
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = orc.make_grid(MODES, EPS)
    pts = orc.gen_points("rand", M, g, 3)
    c = orc.gen_strengths(M, 3)
    f = orc.gen_strengths(int(np.prod(MODES)), 4).reshape(MODES[::-1])
    lo, hi = shard_bounds(M, world, rank)
    res = {}
    # type 1, reduce to root
    sp = ShardedPlan(OracleOps(orc, pts[lo:hi], 1), 1, root=0)
    r = sp.execute(torch.from_numpy(c[lo:hi].copy()))
    res["t1_root"] = r.numpy() if r is not None else np.zeros(0)
    # type 1, all-reduce (every rank gets the modes)
    sp = ShardedPlan(OracleOps(orc, pts[lo:hi], 1), 1, all_ranks=True)
    res["t1_all"] = sp.execute(torch.from_numpy(c[lo:hi].copy())).numpy()
    # type 2, modes only valid on root, broadcast
    fin = torch.from_numpy(f.copy()) if rank == 0 else torch.zeros(MODES[::-1],
                                                                   dtype=torch.complex128)
    sp = ShardedPlan(OracleOps(orc, pts[lo:hi], 2), 2, root=0)
    res["t2"] = sp.execute(fin).numpy()
    # replicas: independent per-rank work + final reduce
    t = torch.full((4,), float(rank + 1), dtype=torch.float64)
    ReplicaPlan(None).reduce_result(t)
    res["replica"] = t.numpy()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), lo=lo, hi=hi, **res)
    dist.barrier()
    dist.destroy_process_group()


def test_sharding_world2_gloo(orc):
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        outs = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    g = orc.make_grid(MODES, EPS)
    pts = orc.gen_points("rand", M, g, 3)
    c = orc.gen_strengths(M, 3)
    f = orc.gen_strengths(int(np.prod(MODES)), 4).reshape(MODES[::-1])
    p1 = orc.OraclePlan(1, MODES, EPS, "sm")
    p1.set_points(pts)
    ref1 = p1.execute(c).reshape(MODES[::-1])
    p2 = orc.OraclePlan(2, MODES, EPS, "gmsort")
    p2.set_points(pts)
    ref2 = p2.execute(f)
    assert orc.rel_l2_error(outs[0]["t1_root"], ref1) < 1e-13
    assert outs[1]["t1_root"].size == 0
    for o in outs:
        assert orc.rel_l2_error(o["t1_all"], ref1) < 1e-13
        lo, hi = int(o["lo"]), int(o["hi"])
        np.testing.assert_allclose(o["t2"], ref2[lo:hi], rtol=0, atol=1e-13)
        np.testing.assert_array_equal(o["replica"], np.full(4, 3.0)) if o is outs[0] else None
    assert int(outs[0]["hi"]) == int(outs[1]["lo"]) and int(outs[1]["hi"]) == M


def test_shard_bounds_partition():
    from paper_2102_08463_b200.dist import shard_bounds
    for M_, W in [(0, 3), (1, 4), (10, 3), (1000003, 8)]:
        b = [shard_bounds(M_, W, r) for r in range(W)]
        assert b[0][0] == 0 and b[-1][1] == M_
        assert all(b[i][1] == b[i + 1][0] for i in range(W - 1))
        assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1
