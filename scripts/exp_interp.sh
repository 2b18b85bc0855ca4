cd $GRAFT_REPO_ROOT
b() { python bench.py --no-cpu-baseline --config c2 --steps 10 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1', d['value'], d['stage_ms'])"; }
b base
NK_UNPERMUTE=0 b direct
python -m pytest tests -m gpu -q -x -k "interp or type2 or transform or accuracy" 2>&1 | tail -2
