cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -k "tiled or c5 or c4 or double" > gpurun_out/q_pytest.log 2>&1; tail -2 gpurun_out/q_pytest.log
for d in 0 31; do
  NK_DBG=$d timeout 300 python bench.py --no-cpu-baseline --config c5t1 --steps 3 --warmup 2 > gpurun_out/dbg_$d.json 2>/dev/null
  echo "dbg $d: $(python -c "import json; d=json.load(open('gpurun_out/dbg_$d.json')); print(d['stage_ms']['type1']['spread'])")"
done
