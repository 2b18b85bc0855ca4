cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/q_pytest.log 2>&1; tail -2 gpurun_out/q_pytest.log
cat > /tmp/det.py <<'PY'
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2102_08463_b200 as nk
from oracle import oracle as orc
modes, eps, M = (128,128,128), 1e-12, 10_000_000
grid = orc.make_grid(modes, eps, "double")
pts = torch.from_numpy(orc.gen_points("rand", M, grid, 1)).cuda()
c = torch.from_numpy(orc.gen_strengths(M, 2)).cuda()
for det in (False, True):
    p = nk.make_plan(1, modes, eps, "sm", "double", deterministic=det)
    p.set_points(pts)
    out = p.execute(c); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3): out = p.execute(c)
    e1.record(); torch.cuda.synchronize()
    print("deterministic", det, "ms per execute", e0.elapsed_time(e1) / 3)
PY
python /tmp/det.py
