#!/bin/bash
# Method/config sweep + ncu captures. Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/sweep
run() { # name args...
  local name=$1; shift
  timeout 900 python bench.py --no-cpu-baseline "$@" > gpurun_out/sweep/$name.json 2> gpurun_out/sweep/$name.err
  echo "$name: $(python -c "import json,sys; d=json.load(open('gpurun_out/sweep/$name.json')); print('%.3e'%d['value'], 'ms', round(d['ms_per_step'],4), d.get('stage_ms'), d['clocks'])" 2>&1 | tail -1)"
}
run c2_gmsort --config c2 --method gmsort
run c2_sm --config c2 --method sm
run c2_gm --config c2 --method gm
run c1_sm --config c1 --method sm
run c1_gmsort --config c1 --method gmsort
run c1_gm --config c1 --method gm
run c3a_sm --config c3a --method sm
run c3a_gmsort --config c3a --method gmsort
run c3b_sm --config c3b --method sm
run c3b_gmsort --config c3b --method gmsort
run c5 --config c5 --steps 3
run c4t2_gmsort --config c4t2 --method gmsort --steps 3
run c4t2_sm --config c4t2 --method sm --steps 3
run c4t1_gmsort --config c4t1 --method gmsort --steps 2
export NK_BENCH_NO_CLOCKS=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp -s 3 -c 1 -o gpurun_out/prof_c2_interp python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spread -s 3 -c 1 -o gpurun_out/prof_c1_spread python bench.py --config c1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1
ls -la gpurun_out
