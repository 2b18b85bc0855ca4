#!/bin/bash
# A/B check: GPU tests ($PYK subset or all) + bench configs ($CFGS) with the
# default kernels and with $ABENV set (e.g. NK_RADIX_LEGACY=1).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/ab; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 ${PYK:+-k "$PYK"} > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for cfg in $CFGS; do
  for v in new old; do
    if [ $v = old ]; then E="env $ABENV"; else E=""; fi
    timeout 600 $E python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 > $O/${cfg}_$v.json 2> $O/${cfg}_$v.err
    echo "$cfg $v: $(python -c "import json; d=json.load(open('$O/${cfg}_$v.json')); print('%.4e'%d['value'], 'setpts', d.get('setpts_ms'), 'stages', d.get('stage_ms'))" 2>&1 | tail -1)"
  done
done
