cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -k "tiled or double or c4 or c5 or 3d or xwin" > gpurun_out/q_pytest.log 2>&1; tail -2 gpurun_out/q_pytest.log
run() { n=$1; shift; timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 2 "$@" > gpurun_out/$n.json 2>/dev/null; echo "$n: $(python -c "import json; d=json.load(open('gpurun_out/$n.json')); print(d['setpts_ms'], d['stage_ms'])")"; }
run c4t1 --config c4t1
run c4t2 --config c4t2
run c5t1 --config c5t1
run c5t2 --config c5t2
export NK_BENCH_NO_CLOCKS=1
for item in c4t1:spread_tiled c4t2:interp_tiled; do
  cfg=${item%%:*}; rx=${item#*:}
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:$rx -s 2 -c 1 --csv --log-file gpurun_out/tr_$cfg.csv python bench.py --no-cpu-baseline --config $cfg --steps 1 --warmup 2 > /dev/null 2>&1
  grep -E "dram__bytes|duration" gpurun_out/tr_$cfg.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
