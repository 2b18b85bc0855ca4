#!/bin/bash
# Focused GPU check: pytest subset ($PYK) + bench configs ($CFGS, "name:args" items)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/q
if [ -n "$PYK" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "$PYK" > gpurun_out/q/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q/pytest.log
  tail -4 gpurun_out/q/pytest.log
fi
for item in $CFGS; do
  name=${item%%:*}; args=${item#*:}; args=${args//,/ }
  timeout 900 python bench.py --no-cpu-baseline $args > gpurun_out/q/$name.json 2> gpurun_out/q/$name.err
  echo "$name: $(python -c "import json,sys; d=json.load(open('gpurun_out/q/$name.json')); print('%.3e'%d['value'], 'ms', round(d['ms_per_step'],4), d.get('stage_ms'), d['config'].get('bin_dims'))" 2>&1 | tail -1)"
done
