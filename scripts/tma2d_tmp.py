import sys, numpy as np
sys.path.insert(0, ".")
import paper_2102_08463_b200 as nk
from oracle import oracle as orc
modes, eps, M = (256, 256), 1e-5, 200000
grid = orc.make_grid(modes, eps, "single")
pts = orc.gen_points("rand", M, grid, 1, np.float32)
rng = np.random.default_rng(0)
f = (rng.standard_normal(modes[::-1]) + 1j*rng.standard_normal(modes[::-1])).astype(np.complex64)
p = nk.make_plan(2, modes, eps, "sm", "single")
p.set_points(pts)
out = p.execute(f)
ref = orc.direct_type2(pts[:2000], f, modes)
print("err", orc.rel_l2_error(out[:2000], ref))
