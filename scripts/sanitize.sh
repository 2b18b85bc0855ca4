#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over the shared-memory
# spread / interp kernels at small sizes; logs under gpurun_out/sanitize/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/sanitize
cat > /tmp/nk_san.py <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2102_08463_b200 as nk
from oracle import oracle as orc
rng = np.random.default_rng(3)
cases = [((24, 20, 16), 1e-12, "double", 1, None), ((24, 20, 16), 1e-12, "double", 2, None),
         ((24, 20, 16), 1e-9, "double", 1, (5, 3, 7)), ((24, 20, 16), 1e-9, "double", 2, (5, 3, 7)),
         ((20, 20, 20), 1e-6, "single", 1, None), ((20, 20, 20), 1e-6, "single", 2, None),
         ((64, 48), 1e-5, "single", 1, None), ((64, 48), 1e-5, "single", 2, None),
         ((32, 32), 1e-12, "double", 1, None), ((32, 32), 1e-12, "double", 2, None)]
for modes, eps, prec, t, bins in cases:
    M = 3000
    grid = orc.make_grid(modes, eps, prec)
    rdt = np.float64 if prec == "double" else np.float32
    pts = orc.gen_points("rand", M, grid, 5, rdt)
    kw = {} if bins is None else {"bin_dims": bins}
    p = nk.make_plan(t, modes, eps, "sm", prec, **kw)
    p.set_points(pts)
    if t == 1:
        out = p.execute(orc.gen_strengths(M, 1).astype(np.complex128 if prec == "double" else np.complex64))
    else:
        f = (rng.standard_normal(modes[::-1]) + 1j * rng.standard_normal(modes[::-1]))
        out = p.execute(f.astype(np.complex128 if prec == "double" else np.complex64))
    print(modes, eps, prec, t, bins, "ok", np.abs(out).max())
PY
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python /tmp/nk_san.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitize/$tool.log)"
done
