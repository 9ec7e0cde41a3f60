#!/bin/bash
# Decision-period captures (profiles/r1_p*): one `ncu --set full` capture of the
# period kernel and one launch list per P, at C5, then the bench lines.
mkdir -p gpurun_out/fin
B="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
for P in 24 168 2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_fast -s 3 -c 1 \
      -o gpurun_out/fin/p$P python bench.py --period-steps $P $B > gpurun_out/fin/ncu_p$P.log 2>&1
  echo "ncu p$P rc=$?"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/fin/launch_p$P.csv python bench.py --period-steps $P --steps 2 --warmup 3 --no-e2e \
      --no-cpu-baseline > gpurun_out/fin/launch_p$P.log 2>&1
  echo "launches p$P rc=$?"
done
