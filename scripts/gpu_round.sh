#!/bin/bash
# Round-end evidence: all bench configs (N=1) + launch list + ncu captures.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/round
for c in c2 c1 c3a c3b c3t1u c3t2 c3t2u c5 c5t1 c5t2 c4t2 c4t1; do
  st=10; case $c in c4*) st=2;; c5*) st=3;; esac
  timeout 900 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/round/bench_$c.json 2> gpurun_out/round/bench_$c.err
  echo "$c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/round/bench_ref_c2.json 2>&1
TAG=${TAG:-r1z} NCU_JOBS="c2:interp:--config,c2 c2f:rowfft:--config,c2 c1:spread:--config,c1 c3a:spread:--config,c3a c3t1u:spread:--config,c3t1u c3t2:interp:--config,c3t2 c5s:spread:--config,c5t1 c5i:interp:--config,c5t2" bash scripts/gpu_profile.sh
