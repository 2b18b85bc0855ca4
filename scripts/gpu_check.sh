#!/bin/bash
# One GPU round: smoke, GPU tests, bench lines. Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in ${BENCH_CONFIGS:-c2 c1}; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
done
tail -3 gpurun_out/smoke.log; tail -15 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_*.json
