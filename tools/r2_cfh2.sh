#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/cfh2; mkdir -p $OUT
for P in 24 2; do
  bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps $P" old cfh setuponly | sed "s/^/P$P /" >> $OUT/ab.txt 2>&1
done
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_cfh.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_fast -s 3 -c 1 \
      -o $OUT/p24_cfh python bench.py --period-steps 24 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-prefix-check > $OUT/ncu.log 2>&1
echo "ncu rc=$?" >> $OUT/ab.txt
