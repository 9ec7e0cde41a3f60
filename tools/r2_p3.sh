#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/p3; rm -rf $OUT; mkdir -p $OUT
for P in 3 2 6; do
  bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps $P" laddr2 base2 p3g4 | sed "s/^/P$P /" >> $OUT/ab.txt 2>&1
done
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_p3g4.so timeout 900 python -m pytest tests -m gpu -q -x -k "period" > $OUT/tests.log 2>&1; echo "p3g4 tests rc=$?" >> $OUT/ab.txt
