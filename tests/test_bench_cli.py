"""SPEC.md:518-567 benchmark module (the reference's missing nufftkit.bench):
CSV schema, Eq. (18) density arithmetic, generators, CLI validation (CPU);
determinism and accuracy column on the GPU."""

import io

import numpy as np
import pytest


def test_header_byte_exact():
    from paper_2102_08463_b200 import bench
    assert bench.HEADER == ("dim,type,method,prec,dist,N1,N2,N3,M,tol,setup_ns_per_pt,"
                            "exec_ns_per_pt,total_ns_per_pt,rel_l2_err,workspace_bytes,seed")
    buf = io.StringIO()
    bench.write_csv([], buf)
    assert buf.getvalue() == bench.HEADER + "\n"


def test_density_eq18():
    """rho = 1, N = (1000, 1000), sigma = 2 -> M = 4,000,000."""
    from paper_2102_08463_b200 import bench
    fine = bench.fine_sizes((1000, 1000), 1e-6, "double")
    assert fine == (2000, 2000)
    assert bench.points_for_density(1.0, fine) == 4_000_000
    assert bench.points_for_density(0.5, (27, 27, 27)) == int(np.ceil(0.5 * 27 ** 3))


def test_generators_deterministic_and_cluster_box():
    from paper_2102_08463_b200 import bench
    a = bench.gen_points("rand", 1000, (64, 64), 5)
    b = bench.gen_points("rand", 1000, (64, 64), 5)
    np.testing.assert_array_equal(a, b)
    assert a.min() >= -np.pi and a.max() < np.pi
    c = bench.gen_points("cluster", 5000, (64, 32), 1)
    h = np.array([2 * np.pi / 64, 2 * np.pi / 32])
    assert (c >= 0).all() and (c <= 8 * h).all()
    s = bench.gen_strengths(10, 3)
    assert s.dtype == np.complex128 and (s.real >= 0).all() and (s.imag < 1).all()


@pytest.mark.parametrize("argv", [
    ["--dim", "4", "--type", "1", "--n", "8,8", "--M", "10"],
    ["--dim", "2", "--type", "3", "--n", "8,8", "--M", "10"],
    ["--dim", "2", "--type", "1", "--n", "8", "--M", "10"],
    ["--dim", "2", "--type", "1", "--n", "8,8"],
    ["--dim", "2", "--type", "1", "--n", "8,8", "--M", "10", "--dist", "ring"],
    ["--dim", "2", "--type", "1", "--n", "8,8", "--M", "10", "--tol", "2"],
    ["--dim", "2", "--type", "1", "--n", "8,8", "--M", "10", "--method", "fast"],
    ["--dim", "2", "--type", "1", "--n", "8,8", "--M", "10", "--prec", "f16"],
])
def test_cli_validation_nonzero_exit(argv, capsys):
    from paper_2102_08463_b200 import bench
    assert bench.main(argv) != 0
    assert "nufftkit-bench:" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_runs_deterministic_error_column(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2102_08463_b200 import bench
    rows = []
    for method in ("sm", "sm", "gmsort", "gm"):
        cfg = bench.BenchConfig(dim=2, type=1, modes=(32, 24), density=1.0, dist="cluster",
                                tol=1e-9, method=method, prec="f64", repeats=2, seed=3)
        rows.append(bench.run_benchmark(cfg))
    errs = [float(r["rel_l2_err"]) for r in rows]
    assert all(e < 1e-8 for e in errs)                      # 10 eps
    assert abs(errs[0] - errs[1]) <= 1e-3 * errs[0]         # same seed/config
    assert rows[0]["M"] == int(np.ceil(64 * 48))            # rho = 1
    out = tmp_path / "r.csv"
    assert bench.main(["--dim", "3", "--type", "2", "--n", "8,10,12", "--density", "1",
                       "--tol", "1e-5", "--prec", "f32", "--repeats", "2",
                       "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == bench.HEADER and len(lines) == 2
    assert float(lines[1].split(",")[13]) < 1e-4
