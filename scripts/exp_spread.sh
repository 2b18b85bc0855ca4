cd $GRAFT_REPO_ROOT
b() { python bench.py --no-cpu-baseline --config $2 --steps ${3:-5} ${4} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1 $2 $4', '%.3e'%d['value'], {k:round(v,4) for k,v in d['stage_ms'].items()}, d['config']['bin_dims'])"; }
for c in c3a c3b c3t1u; do b $NWTAG $c; done
