cd $GRAFT_REPO_ROOT
run() { n=$1; shift; timeout 300 python bench.py --no-cpu-baseline --steps 2 --warmup 2 "$@" > gpurun_out/$n.json 2>/dev/null; echo "$n: $(python -c "import json; d=json.load(open('gpurun_out/$n.json')); print(d['setpts_ms'], d['stage_ms'])")"; }
run c4t2 --config c4t2
run c4t2_888 --config c4t2 --bins 8,8,8
run c4t2_777 --config c4t2 --bins 7,7,7
run c5t2_666 --config c5t2 --bins 6,6,6
run c5t2_776 --config c5t2 --bins 7,7,6
