cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q -x -k "spread or type1 or transform or accuracy or batched or adjoint" 2>&1 | tail -2
b() { python bench.py --no-cpu-baseline --config $2 --steps ${3:-5} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1 $2', '%.3e'%d['value'], d['stage_ms'], d['setpts_ms'])"; }
for c in c3a c3b c3t1u; do b new $c; done
b new c5 3
b new c4t1 2
