cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/q_pytest.log 2>&1; tail -2 gpurun_out/q_pytest.log
run() { n=$1; shift; timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 2 "$@" > gpurun_out/$n.json 2>/dev/null; echo "$n: $(python -c "import json; d=json.load(open('gpurun_out/$n.json')); print(d['setpts_ms'], d['stage_ms'], d['config']['bin_dims'], d['config']['method'])")"; }
run c4 --config c4
run c5 --config c5
run c4t2_7117 --config c4t2 --bins 7,11,7
run c5t1_7117 --config c5t1 --bins 7,11,7
run c5t1_7711 --config c5t1 --bins 7,7,11
