#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/cfh; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -k "period or headline or timeline or full_size" > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log
for P in 3 5 24 12 10 6 48; do
  bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps $P" cfh3 cfh | sed "s/^/P$P /" >> $OUT/ab.txt 2>&1
done
