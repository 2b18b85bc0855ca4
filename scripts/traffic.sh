#!/bin/bash
# DRAM bytes (read + write) per launch of each config's dominant kernel:
# one ncu pass per config, the values go to profiles/traffic.json.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/traffic
export NK_BENCH_NO_CLOCKS=1
for item in c4:spread_tiled c4t1:spread_tiled c4t2:interp_tiled c5t1:spread_tiled c5t2:interp_tiled c5:spread_tiled c2:interp c1:spread c3a:spread c3b:spread c3t1u:spread c3t2:interp c3t2u:interp; do
  cfg=${item%%:*}; rx=${item#*:}
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
     --clock-control none -k regex:$rx -s 2 -c 1 --csv --log-file gpurun_out/traffic/$cfg.csv \
     python bench.py --no-cpu-baseline --config $cfg --steps 1 --warmup 2 > /dev/null 2>&1
  echo "$cfg rc=$?"
done
