cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/q_pytest.log 2>&1; tail -2 gpurun_out/q_pytest.log
for c in c2 c5t1 c4t1 c3a; do
timeout 300 python bench.py --no-cpu-baseline --config $c --steps 2 --warmup 2 > gpurun_out/$c.json 2>/dev/null
echo "$c: $(python -c "import json; d=json.load(open('gpurun_out/$c.json')); print(d['setpts_ms'], d['stage_ms'])")"
done
