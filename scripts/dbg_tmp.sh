cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/q_pytest.log 2>&1; tail -2 gpurun_out/q_pytest.log
run() { n=$1; shift; timeout 300 python bench.py --no-cpu-baseline --steps 5 --warmup 2 "$@" > gpurun_out/$n.json 2>/dev/null; echo "$n: $(python -c "import json; d=json.load(open('gpurun_out/$n.json')); print(d['stage_ms'])")"; }
run c2 --config c2
run c3t2 --config c3t2
run c3t2u --config c3t2u
