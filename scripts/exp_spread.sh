cd $GRAFT_REPO_ROOT
b() { python bench.py --no-cpu-baseline --config $2 --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1 $2', '%.3e'%d['value'], d['stage_ms'], d['setpts_ms'])"; }
for nw in 8 4 2; do for c in c3a c3b; do NK_SM3_WARPS=$nw b nw$nw $c; done; done
