"""set_points only (for ncu launch lists of the setpts kernels).

    python scripts/setpts_only.py [M] [c4|c2]

c4: 3D type 1 f64, N = 256^3, eps = 1e-12 (default); c2: 2D type 2 f32,
N = 1024^2, eps = 1e-5.  Uniform points; set_points runs twice."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2102_08463_b200.plan import TransformPlan  # noqa: E402

M = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
cfg = sys.argv[2] if len(sys.argv) > 2 else "c4"
dim, ttype, modes, eps, prec = {"c4": (3, 1, (256,) * 3, 1e-12, "double"),
                                "c2": (2, 2, (1024,) * 2, 1e-5, "single")}[cfg]
dt = torch.float64 if prec == "double" else torch.float32
g = torch.Generator(device="cuda").manual_seed(1)
pts = [(torch.rand(M, device="cuda", dtype=dt, generator=g) * 2 - 1) * torch.pi
       for _ in range(dim)]
p = TransformPlan(ttype, modes, eps, precision=prec)
for _ in range(2):
    p.set_points(*pts)
torch.cuda.synchronize()
print("ok")
