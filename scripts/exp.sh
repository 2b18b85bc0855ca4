cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q -x -k "sort or bin or layout or golden or sub or accuracy" 2>&1 | tail -2
b() { python bench.py --no-cpu-baseline --config $2 --steps ${3:-5} ${4} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1 $2 $4', '%.3e'%d['value'], d['setpts_ms'])"; }
for c in c2 c3a c3t2 c1; do b d $c; done
