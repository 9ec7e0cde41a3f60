#!/bin/bash
# Lane-local decision periods (sweep_fast_kernel<3>, <4>): bench lines for
# P = 2, 6, 12 (plus 24 and 168 for the table), one `ncu --set full` capture and
# one launch list each for P = 2 (<4>) and P = 12 (<3>), at C5.
mkdir -p gpurun_out/ll
run() { name=$1; shift; timeout 600 python bench.py "$@" > gpurun_out/ll/$name.json 2> gpurun_out/ll/$name.err; echo "$name rc=$?"; }
for P in 2 6 12 24 168; do
  run bench_p$P --period-steps $P --steps 10 --warmup 3 --no-cpu-baseline
done
B="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
for P in 2 12; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_fast -s 3 -c 1 \
      -o gpurun_out/ll/p$P python bench.py --period-steps $P $B > gpurun_out/ll/ncu_p$P.log 2>&1
  echo "ncu p$P rc=$?"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/ll/launch_p$P.csv python bench.py --period-steps $P --steps 2 --warmup 3 --no-e2e \
      --no-cpu-baseline > gpurun_out/ll/launch_p$P.log 2>&1
  echo "launches p$P rc=$?"
done
