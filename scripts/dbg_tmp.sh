cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "tiled or double or c4 or c5 or 3d or xwin" > gpurun_out/q_pytest.log 2>&1; tail -2 gpurun_out/q_pytest.log
for c in c5t2 c4t2; do
timeout 300 python bench.py --no-cpu-baseline --config $c --steps 2 --warmup 2 > gpurun_out/$c.json 2>/dev/null
echo "$c: $(python -c "import json; d=json.load(open('gpurun_out/$c.json')); print(d['stage_ms'])")"
NK_NO_TMA=1 timeout 300 python bench.py --no-cpu-baseline --config $c --steps 2 --warmup 2 > gpurun_out/${c}_notma.json 2>/dev/null
echo "$c notma: $(python -c "import json; d=json.load(open('gpurun_out/${c}_notma.json')); print(d['stage_ms'])")"
done
