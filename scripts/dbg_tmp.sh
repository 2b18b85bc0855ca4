cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "tiled or double or c4 or c5 or 3d" > gpurun_out/q_pytest.log 2>&1; tail -2 gpurun_out/q_pytest.log
for d in 0 15; do
  NK_DBG=$d timeout 300 python bench.py --no-cpu-baseline --config c5t1 --steps 3 --warmup 2 > gpurun_out/dbg_$d.json 2>/dev/null
  echo "dbg $d: $(python -c "import json; d=json.load(open('gpurun_out/dbg_$d.json')); print(d['stage_ms'])")"
done
timeout 300 python bench.py --no-cpu-baseline --config c4t1 --steps 2 --warmup 2 > gpurun_out/c4t1.json 2>/dev/null
echo "c4t1: $(python -c "import json; d=json.load(open('gpurun_out/c4t1.json')); print(d['stage_ms'])")"
