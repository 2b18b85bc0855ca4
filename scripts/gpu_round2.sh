#!/bin/bash
# Round-2 evidence: every bench config (N=1), the paper's method comparison
# (GM / GM-sort / SM), the reference arm, the launch list of the default
# bench and ncu --set full captures of the dominant kernels.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out/round2; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
for c in c4 c2 c1 c3a c3b c3t1u c3t2 c3t2u c5 c5t1 c5t2 c4t1 c4t2; do
  st=10; case $c in c4*) st=3;; c5*) st=5;; esac
  timeout 900 python bench.py --config $c --steps $st --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "$c rc=$?"
done
for m in gm gmsort; do
  for c in c2 c1 c5t1 c5t2 c3a; do
    timeout 900 python bench.py --no-cpu-baseline --config $c --method $m --steps 3 --warmup 3 > $OUT/method_${c}_$m.json 2> $OUT/method_${c}_$m.err
    echo "$c $m rc=$?"
  done
done
timeout 900 python bench.py --no-cpu-baseline --config c4t2 --method gmsort --steps 2 --warmup 3 > $OUT/method_c4t2_gmsort.json 2> $OUT/method_c4t2_gmsort.err
timeout 1800 python bench.py --no-cpu-baseline --config c4t1 --method gmsort --steps 2 --warmup 3 > $OUT/method_c4t1_gmsort.json 2> $OUT/method_c4t1_gmsort.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_c4.json 2> $OUT/bench_ref_c4.err
echo "ref rc=$?"
export NK_BENCH_NO_CLOCKS=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
  --log-file $OUT/r2_launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/r2_launches_c4.log 2>&1
for item in c5s:spread_tiled:--config,c5t1 c5i:interp_tiled:--config,c5t2 c2:interp:--config,c2 c4r:radix_scatter:--config,c4t1 c3a:spread:--config,c3a; do
  name=${item%%:*}; rest=${item#*:}; rx=${rest%%:*}; args=${rest#*:}; args=${args//,/ }
  rep=/tmp/r2_$name
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 \
      -o $rep -f python bench.py --no-cpu-baseline --steps 1 --warmup 3 $args > $OUT/r2_$name.log 2>&1
  echo "$name rc=$?"
  python scripts/ncu_summary.py $rep.ncu-rep > $OUT/r2_${name}_ncu_full.txt 2>&1
  ncu -i $rep.ncu-rep --page source --csv > $OUT/r2_$name.source.csv 2>/dev/null
done
cuobjdump -sass paper_2102_08463_b200/libnufft_b200.so | grep -oE "UTMALDG|UBLKCP|UBLKRED[.A-Z0-9]*|DMMA\.8x8x4|LDGSTS[.A-Z0-9]*" | sort | uniq -c > $OUT/sass_mnemonics.txt
