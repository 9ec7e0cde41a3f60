#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/long; rm -rf $OUT; mkdir -p $OUT
timeout 300 python tools/cfh_probe.py 4000 > $OUT/probe.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "period or headline or full_size or timeline" > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/ab.txt
for P in 64 100 168 720 1000; do
  bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps $P" longcf | sed "s/^/P$P direct /" >> $OUT/ab.txt 2>&1
  CHASE_PM2=1 bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps $P" longcf | sed "s/^/P$P batches /" >> $OUT/ab.txt 2>&1
done
