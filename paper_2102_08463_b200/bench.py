"""Benchmark CLI and CSV report (pyproject.toml:22-23 names
the entry point ``nufftkit-bench = nufftkit.bench:main``, which the shipped
reference does not contain).

    python -m paper_2102_08463_b200.bench --dim 2 --type 1 --n 1000,1000 \
        --density 1 --dist rand --tol 1e-6 --method sm --prec f64 \
        --repeats 5 --seed 0 --out report.csv

Timing categories (the paper's §IV-C): ``setup`` = set_points
(fold, bin sort, subproblems; "after its nonuniform points have already been
preprocessed"), ``exec`` = execute with points bound, ``total`` = setup +
exec, each the median over ``repeats`` and reported as ns per nonuniform
point.  Times are CUDA-event device times on the plan's stream with inputs
resident on the device: the paper's "total+mem" (host<->device transfer) is
not reported, as SPEC.md:566 asks, so the header comment states the mapping.
The accuracy column is the relative l2 error against a direct sum evaluated
in float64 on the same GPU (torch), computed when N_tot * M <= the oracle
budget (default 1e9) and blank otherwise.
"""

from __future__ import annotations

import argparse
import csv
import math
import sys
from dataclasses import dataclass, field

import numpy as np
import torch

from .plan import TransformPlan, next_smooth
from .kernel import tolerance_to_width

__all__ = ["HEADER", "BenchConfig", "fine_sizes", "points_for_density", "gen_points",
           "gen_strengths", "run_benchmark", "main"]

# byte-exact
HEADER = ("dim,type,method,prec,dist,N1,N2,N3,M,tol,setup_ns_per_pt,exec_ns_per_pt,"
          "total_ns_per_pt,rel_l2_err,workspace_bytes,seed")
TIMING_NOTE = ("# setup = set_points (sort + subproblems); exec = execute with points bound "
               "(paper 'exec'); total = setup + exec; device-resident inputs, CUDA-event "
               "device times, median over repeats; the paper's 'total+mem' (host-device "
               "transfer) is not reported")


@dataclass
class BenchConfig:
    """SPEC.md:523-528."""

    dim: int
    type: int
    modes: tuple
    density: float | None = None
    M: int | None = None
    dist: str = "rand"
    tol: float = 1e-6
    method: str = "sm"
    prec: str = "f64"
    repeats: int = 5
    seed: int = 0
    threads: int = 0
    points_file: str | None = None
    oracle_budget: float = 1e9
    device: int | None = None
    extra: dict = field(default_factory=dict)

    def validate(self):
        if self.dim not in (2, 3):
            raise ValueError(f"--dim must be 2 or 3, got {self.dim}")
        if self.type not in (1, 2):
            raise ValueError(f"--type must be 1 or 2, got {self.type}")
        if len(self.modes) != self.dim or any(int(n) < 1 for n in self.modes):
            raise ValueError(f"--n needs {self.dim} positive sizes, got {self.modes}")
        if (self.density is None) == (self.M is None) and self.points_file is None:
            raise ValueError("give exactly one of --density and --M")
        if self.density is not None and not self.density > 0:
            raise ValueError(f"--density must be > 0, got {self.density}")
        if self.M is not None and self.M < 0:
            raise ValueError(f"--M must be >= 0, got {self.M}")
        if self.dist not in ("rand", "cluster"):
            raise ValueError(f"--dist must be rand or cluster, got {self.dist!r}")
        if not 0 < self.tol < 1:
            raise ValueError(f"--tol must be in (0, 1), got {self.tol}")
        if self.method not in ("gm", "gmsort", "sm"):
            raise ValueError(f"--method must be gm, gmsort or sm, got {self.method!r}")
        if self.prec not in ("f32", "f64"):
            raise ValueError(f"--prec must be f32 or f64, got {self.prec!r}")
        if self.repeats < 1:
            raise ValueError(f"--repeats must be >= 1, got {self.repeats}")

    @property
    def precision(self):
        return "single" if self.prec == "f32" else "double"


def fine_sizes(modes, tol, precision):
    """SPEC.md:132-140 sizing: n_i = next_smooth(max(2 N_i, 2 w))."""
    _, w, _ = tolerance_to_width(tol, precision)[:3]
    return tuple(next_smooth(max(2 * int(N), 2 * w)) for N in modes)


def points_for_density(density, fine):
    """Eq. (18): rho = M / prod(n_i)  ->  M = ceil(rho * prod(n_i))."""
    return int(math.ceil(density * float(np.prod(fine))))


def gen_points(dist, M, fine, seed, dtype=np.float64):
    """rand -> iid U[-pi, pi)^d; cluster -> iid U prod[0, 8 h_i]
    with h_i = 2 pi / n_i.  Deterministic in seed."""
    rng = np.random.default_rng(seed)
    d = len(fine)
    if dist == "rand":
        x = rng.uniform(-np.pi, np.pi, (M, d))
    elif dist == "cluster":
        h = np.array([2 * np.pi / n for n in fine])
        x = rng.uniform(0.0, 1.0, (M, d)) * (8 * h)
    else:
        raise ValueError(f"unknown distribution {dist!r}")
    return x.astype(dtype)


def gen_strengths(shape, seed, dtype=np.complex128):
    """iid complex with U[0, 1) real and imaginary parts."""
    rng = np.random.default_rng(seed + 1000003)
    return (rng.uniform(0, 1, shape) + 1j * rng.uniform(0, 1, shape)).astype(dtype)


def _read_points(path, dim):
    raw = np.fromfile(path, dtype="<f8")
    if raw.size % dim:
        raise ValueError(f"{path}: {raw.size} doubles is not a multiple of dim={dim}")
    return raw.reshape(-1, dim)


def _direct(cfg, x, inp, dev):
    """Direct sums in float64 on the device (the accuracy column's checker):
    type 1 f_k = sum_j c_j e^{-i k.x_j}; type 2 c_j = sum_k f_k e^{+i k.x_j}
    (PAPER.md:76-100), modes (N_d..N_1), k_i in -floor(N_i/2)..."""
    d = cfg.dim
    X = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)
    ks = [torch.arange(-(N // 2), N - N // 2, dtype=torch.float64, device=dev)
          for N in cfg.modes]
    grids = torch.meshgrid(*ks[::-1], indexing="ij")          # (N_d, ..., N_1)
    K = torch.stack([g.reshape(-1) for g in grids[::-1]], 1)  # (Ntot, d) axis 1 first
    v = torch.from_numpy(np.ascontiguousarray(inp).astype(np.complex128).reshape(-1)).to(dev)
    out = []
    chunk = max(1, int(2 ** 24 // max(K.shape[0], 1)))
    if cfg.type == 1:
        acc = torch.zeros(K.shape[0], dtype=torch.complex128, device=dev)
        for s in range(0, X.shape[0], chunk):
            ph = K @ X[s:s + chunk].T                          # (Ntot, m)
            acc += torch.exp(-1j * ph) @ v[s:s + chunk]
        return acc.cpu().numpy()
    for s in range(0, X.shape[0], chunk):
        ph = X[s:s + chunk] @ K.T                              # (m, Ntot)
        out.append((torch.exp(1j * ph) @ v).cpu().numpy())
    return np.concatenate(out) if out else np.zeros(0, np.complex128)


def run_benchmark(cfg: BenchConfig):
    """one setup, `repeats` executions; returns one report
    row (dict keyed by HEADER columns)."""
    cfg.validate()
    dev = torch.device("cuda", cfg.device if cfg.device is not None else
                       torch.cuda.current_device())
    rdt = np.float32 if cfg.prec == "f32" else np.float64
    cdt = np.complex64 if cfg.prec == "f32" else np.complex128
    fine = fine_sizes(cfg.modes, cfg.tol, cfg.precision)
    if cfg.points_file:
        x = _read_points(cfg.points_file, cfg.dim).astype(rdt)
    else:
        M = cfg.M if cfg.M is not None else points_for_density(cfg.density, fine)
        x = gen_points(cfg.dist, M, fine, cfg.seed, rdt)
    M = x.shape[0]
    Ntot = int(np.prod(cfg.modes))
    inp = gen_strengths((M,) if cfg.type == 1 else tuple(cfg.modes[::-1]), cfg.seed, cdt)
    with torch.cuda.device(dev):
        free0 = torch.cuda.mem_get_info(dev)[0]
        plan = TransformPlan(cfg.type, cfg.modes, cfg.tol, cfg.method, cfg.precision,
                             device=dev.index)
        xd = torch.from_numpy(x).to(dev)
        ind = torch.from_numpy(inp).to(dev)
        plan.set_points(xd)                 # allocates; timed calls below reuse
        out = plan.execute(ind)
        torch.cuda.synchronize(dev)
        workspace = max(0, free0 - torch.cuda.mem_get_info(dev)[0])
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        setup, exe = [], []
        for _ in range(cfg.repeats):
            ev[0].record()
            plan.set_points(xd)
            ev[1].record()
            plan.execute(ind, out)
            ev[2].record()
            torch.cuda.synchronize(dev)
            setup.append(ev[0].elapsed_time(ev[1]) * 1e6)
            exe.append(ev[1].elapsed_time(ev[2]) * 1e6)
        err = ""
        if M > 0 and float(Ntot) * M <= cfg.oracle_budget:
            ref = _direct(cfg, x, inp, dev)
            got = out.cpu().numpy().reshape(-1)
            err = f"{np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300):.6e}"
        plan.destroy()
    per = max(M, 1)
    s_ns, e_ns = float(np.median(setup)) / per, float(np.median(exe)) / per
    N = list(cfg.modes) + [1] * (3 - cfg.dim)
    return {"dim": cfg.dim, "type": cfg.type, "method": cfg.method, "prec": cfg.prec,
            "dist": cfg.dist if not cfg.points_file else "file", "N1": N[0], "N2": N[1],
            "N3": N[2], "M": M, "tol": f"{cfg.tol:g}", "setup_ns_per_pt": f"{s_ns:.6g}",
            "exec_ns_per_pt": f"{e_ns:.6g}", "total_ns_per_pt": f"{s_ns + e_ns:.6g}",
            "rel_l2_err": err, "workspace_bytes": int(workspace), "seed": cfg.seed,
            "_min_exec_ns_per_pt": float(np.min(exe)) / per}


def write_csv(rows, fh):
    fh.write(HEADER + "\n")
    w = csv.writer(fh, lineterminator="\n")
    cols = HEADER.split(",")
    for r in rows:
        w.writerow([r[c] for c in cols])


def _parse(argv):
    ap = argparse.ArgumentParser(prog="nufftkit-bench", description=__doc__.split("\n")[0])
    ap.add_argument("--dim", type=int, required=True)
    ap.add_argument("--type", type=int, required=True)
    ap.add_argument("--n", required=True, help="N1[,N2[,N3]]")
    g = ap.add_mutually_exclusive_group()
    g.add_argument("--density", type=float)
    g.add_argument("--M", type=int)
    ap.add_argument("--dist", default="rand")
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--method", default="sm")
    ap.add_argument("--prec", default="f64")
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0,
                    help="accepted for compatibility; the GPU grid replaces host workers")
    ap.add_argument("--points", default=None,
                    help="little-endian float64 records, dim values per point")
    ap.add_argument("--out", default=None)
    ap.add_argument("--device", type=int, default=None)
    return ap.parse_args(argv)


def config_from_args(a):
    try:
        modes = tuple(int(v) for v in a.n.split(","))
    except ValueError:
        raise ValueError(f"--n must be comma-separated integers, got {a.n!r}")
    return BenchConfig(dim=a.dim, type=a.type, modes=modes, density=a.density, M=a.M,
                       dist=a.dist, tol=a.tol, method=a.method, prec=a.prec,
                       repeats=a.repeats, seed=a.seed, threads=a.threads,
                       points_file=a.points, device=a.device)


def main(argv=None):
    a = _parse(sys.argv[1:] if argv is None else argv)
    try:
        cfg = config_from_args(a)
        cfg.validate()
    except ValueError as e:
        print(f"nufftkit-bench: {e}", file=sys.stderr)
        return 2
    row = run_benchmark(cfg)
    if a.out:
        with open(a.out, "w") as fh:
            write_csv([row], fh)
    write_csv([row], sys.stdout)
    print(TIMING_NOTE)
    return 0


if __name__ == "__main__":
    sys.exit(main())
