"""GPU checks of the sharded paths (emulated shards on
one GPU must equal the unsharded transform; NCCL world-size-1 group runs the
real collectives through ShardedPlan + CudaStageOps)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2102_08463_b200 as nk
    from paper_2102_08463_b200 import dist as nkd
    return torch, nk, nkd


@pytest.mark.parametrize("dim,prec,eps", [(2, "single", 1e-5), (3, "double", 1e-9)])
def test_emulated_type1_shards(env, orc, dim, prec, eps):
    torch, nk, nkd = env
    modes = (64, 48) if dim == 2 else (16, 20, 12)
    grid = orc.make_grid(modes, eps, prec)
    rdt = np.float32 if prec == "single" else np.float64
    cdt = np.complex64 if prec == "single" else np.complex128
    M, S = 40000, 3
    pts = orc.gen_points("rand", M, grid, 2, rdt)
    c = torch.from_numpy(orc.gen_strengths(M, 2, cdt)).cuda()
    full = nk.make_plan(1, modes, eps, precision=prec)
    full.set_points(pts)
    ref = full.execute(c)
    acc = None
    for r in range(S):
        lo, hi = nkd.shard_bounds(M, S, r)
        p = nk.make_plan(1, modes, eps, precision=prec)
        p.set_points(pts[lo:hi])
        ops = nkd.CudaStageOps(p)
        g = ops.spread(c[lo:hi].contiguous()).clone()
        acc = g if acc is None else acc + g
    out = ops.new_modes()
    ops.fft_deconvolve(acc, out)
    tol = 1e-5 if prec == "single" else 1e-12
    assert orc.rel_l2_error(out.cpu().numpy(), ref.cpu().numpy()) < tol


def test_sharded_plan_nccl_world1(env, orc):
    torch, nk, nkd = env
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        modes, eps = (40, 44), 1e-6
        grid = orc.make_grid(modes, eps, "single")
        pts = orc.gen_points("rand", 20000, grid, 5, np.float32)
        c = torch.from_numpy(orc.gen_strengths(20000, 5, np.complex64)).cuda()
        f = torch.from_numpy(orc.gen_strengths(int(np.prod(modes)), 6, np.complex64)
                             .reshape(modes[::-1])).cuda()
        for t, inp in ((1, c), (2, f)):
            p = nk.make_plan(t, modes, eps, precision="single")
            p.set_points(pts)
            ref = p.execute(inp).cpu().numpy()
            sp = nkd.ShardedPlan(nkd.CudaStageOps(p), t)
            got = sp.execute(inp).cpu().numpy()
            assert orc.rel_l2_error(got, ref) < 1e-6
    finally:
        dist.destroy_process_group()


def _gpu_worker(rank, world, port, outdir, cfg):
    """One rank of the 2-process CUDA test: this rank's point shard through
    ShardedPlan(CudaStageOps) on cuda:0 (both ranks share the one GPU; gloo
    carries the CUDA-tensor all-reduce / broadcast)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_2102_08463_b200 as nk
    from paper_2102_08463_b200 import dist as nkd
    from oracle import oracle as orc
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        modes, eps, prec, M = cfg
        grid = orc.make_grid(modes, eps, prec)
        rdt = np.float32 if prec == "single" else np.float64
        cdt = np.complex64 if prec == "single" else np.complex128
        pts = orc.gen_points("rand", M, grid, 8, rdt)
        c = torch.from_numpy(orc.gen_strengths(M, 8, cdt)).cuda()
        f = torch.from_numpy(orc.gen_strengths(int(np.prod(modes)), 9, cdt)
                             .reshape(modes[::-1])).cuda()
        lo, hi = nkd.shard_bounds(M, world, rank)
        res = {}
        p1 = nk.make_plan(1, modes, eps, precision=prec)
        p1.set_points(pts[lo:hi])
        res["t1"] = nkd.ShardedPlan(nkd.CudaStageOps(p1), 1, all_ranks=True).execute(
            c[lo:hi].contiguous()).cpu().numpy()
        p2 = nk.make_plan(2, modes, eps, precision=prec)
        p2.set_points(pts[lo:hi])
        fin = f if rank == 0 else torch.zeros_like(f)
        res["t2"] = nkd.ShardedPlan(nkd.CudaStageOps(p2), 2, root=0).execute(fin).cpu().numpy()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), lo=lo, hi=hi, **res)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [((40, 44), 1e-6, "single", 30001),
                                 ((16, 20, 12), 1e-12, "double", 20001)])
def test_sharded_plan_two_processes_cuda(env, orc, cfg):
    """World-size-2 ShardedPlan over the CUDA stage ops (two processes on
    one GPU, gloo): type 1 (per-rank spread + all-reduce of the fine grids +
    FFT / deconvolution) and type 2 (root's modes broadcast, per-rank
    interpolation) must equal the unsharded plan."""
    import tempfile
    import torch.multiprocessing as mp
    torch, nk, nkd = env
    modes, eps, prec, M = cfg
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gpu_worker, args=(2, port, d, cfg), nprocs=2, join=True)
        outs = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(2)]
    grid = orc.make_grid(modes, eps, prec)
    rdt = np.float32 if prec == "single" else np.float64
    cdt = np.complex64 if prec == "single" else np.complex128
    pts = orc.gen_points("rand", M, grid, 8, rdt)
    c = torch.from_numpy(orc.gen_strengths(M, 8, cdt)).cuda()
    f = torch.from_numpy(orc.gen_strengths(int(np.prod(modes)), 9, cdt).reshape(modes[::-1])).cuda()
    p1 = nk.make_plan(1, modes, eps, precision=prec)
    p1.set_points(pts)
    ref1 = p1.execute(c).cpu().numpy()
    p2 = nk.make_plan(2, modes, eps, precision=prec)
    p2.set_points(pts)
    ref2 = p2.execute(f).cpu().numpy()
    tol = 1e-5 if prec == "single" else 1e-12
    for o in outs:
        assert orc.rel_l2_error(o["t1"], ref1) < tol
        lo, hi = int(o["lo"]), int(o["hi"])
        assert orc.rel_l2_error(o["t2"], ref2[lo:hi]) < tol
    assert int(outs[0]["hi"]) == int(outs[1]["lo"]) and int(outs[1]["hi"]) == M
