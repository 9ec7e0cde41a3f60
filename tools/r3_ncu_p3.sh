#!/bin/bash
# P = 3 and P = 15 period-kernel counters after the LDS.64 change (one launch each, C5)
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/r3ncu; rm -rf $OUT; mkdir -p $OUT
M=gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
for P in 3 15; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:sweep_fast -s 3 -c 1 --csv \
    python bench.py --period-steps $P --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/p$P.csv 2> $OUT/p$P.err
  echo "p$P rc=$?"
done
