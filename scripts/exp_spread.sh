cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()"
b() { python bench.py --no-cpu-baseline --config $2 --steps ${3:-5} ${4} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1 $2 $4', '%.3e'%d['value'], {k:round(v,4) for k,v in d['stage_ms'].items()}, d['setpts_ms'])"; }
for c in c1 c2 c3a c3t2; do b d $c; done; b d c5 3
