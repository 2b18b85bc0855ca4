#!/bin/bash
# Evidence pass: launch list of the default bench (ncu gpu__time_duration,
# serialised, cold) + one --set full capture per dominant kernel, summarised
# on the box (reports are ~16 MB each; only $KEEP_REP ones come back).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/prof
export NK_BENCH_NO_CLOCKS=1
TAG=${TAG:-r1}
if [ -z "$NO_LAUNCHES" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/prof/${TAG}_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/prof/${TAG}_launches_c2.log 2>&1
fi
for item in ${NCU_JOBS:-c2:interp:--config,c2 c1:spread:--config,c1 c3a:spread:--config,c3a}; do
  name=${item%%:*}; rest=${item#*:}; rx=${rest%%:*}; args=${rest#*:}; args=${args//,/ }
  rep=/tmp/${TAG}_$name
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 \
      -o $rep -f python bench.py --no-cpu-baseline --steps 1 --warmup 3 $args \
      > gpurun_out/prof/${TAG}_$name.log 2>&1
  echo "$name rc=$?"
  python scripts/ncu_summary.py $rep.ncu-rep > gpurun_out/prof/${TAG}_$name.txt 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/prof/${TAG}_$name.raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv > gpurun_out/prof/${TAG}_$name.source.csv 2>/dev/null
  case " $KEEP_REP " in *" $name "*) cp $rep.ncu-rep gpurun_out/prof/ ;; esac
done
du -sh gpurun_out
