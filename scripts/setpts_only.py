"""set_points only (for ncu launch lists of the setpts kernels): C4 geometry
(3D type 1 f64, N = 256^3, eps = 1e-12), uniform points, M from argv."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2102_08463_b200.plan import TransformPlan

M = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
g = torch.Generator(device="cuda").manual_seed(1)
pts = [(torch.rand(M, device="cuda", dtype=torch.float64, generator=g) * 2 - 1) * torch.pi
       for _ in range(3)]
p = TransformPlan(1, (256, 256, 256), 1e-12, precision="double")
for _ in range(2):
    p.set_points(*pts)
torch.cuda.synchronize()
print("ok")
