#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/db; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -k "period" > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/ab.txt
for P in 48 8 16 32 7 17; do bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps $P" nodb db | sed "s/^/P$P /" >> $OUT/ab.txt 2>&1; done
