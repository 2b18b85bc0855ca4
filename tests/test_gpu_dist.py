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
