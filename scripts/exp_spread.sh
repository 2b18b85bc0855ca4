cd $GRAFT_REPO_ROOT
b() { python bench.py --no-cpu-baseline --config $2 --steps ${3:-5} ${4} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1 $2 $4', '%.3e'%d['value'], {k:round(v,4) for k,v in d['stage_ms'].items()}, d['config']['bin_dims'])"; }
for m in 1024 2048 4096 8192 16384; do b m c2 10 "--msub $m"; done
for m in 1024 4096 16384; do b m c3t2 5 "--msub $m"; done
