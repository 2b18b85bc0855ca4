cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q -x -k "sort or bin or layout or golden or sub" 2>&1 | tail -2
b() { python bench.py --no-cpu-baseline --config $2 --steps ${3:-5} ${4} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1 $2 $4', '%.3e'%d['value'], d['setpts_ms'])"; }
for c in c2 c3a c3t2; do b d $c; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv python bench.py --no-cpu-baseline --config c2 --steps 1 --warmup 3 2>/dev/null | grep -v "^==" | head -40 > gpurun_out/setpts_launch.csv
