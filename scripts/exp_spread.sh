cd $GRAFT_REPO_ROOT
b() { python bench.py --no-cpu-baseline --config $2 --steps ${3:-5} ${4} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1 $2 $4', '%.3e'%d['value'], d['stage_ms'], d['setpts_ms'])"; }
for m in 128 256 512 1024 4096; do b new c1 5 "--msub $m"; done
for m in 256 1024 4096; do b new c3a 5 "--msub $m"; b new c3b 5 "--msub $m"; done
