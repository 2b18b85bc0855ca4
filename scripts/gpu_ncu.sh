#!/bin/bash
# ncu --set full captures: $NCU_JOBS = "name:regex:bench-args(comma-separated)" items
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/ncu
export NK_BENCH_NO_CLOCKS=1
for item in $NCU_JOBS; do
  name=${item%%:*}; rest=${item#*:}; rx=${rest%%:*}; args=${rest#*:}; args=${args//,/ }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 \
      -o gpurun_out/ncu/$name python bench.py --no-cpu-baseline --steps 1 --warmup 3 $args \
      > gpurun_out/ncu/$name.log 2>&1
  echo "$name rc=$?"
done
