#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/runs2; rm -rf $OUT; mkdir -p $OUT
for P in 2 3 5 6 10 15; do bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps $P" runs1 runs2 runs2p2 | sed "s/^/P$P /" >> $OUT/ab.txt 2>&1; done
for v in runs2p2; do
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_$v.so timeout 900 python -m pytest tests -m gpu -q -x -k "period" > $OUT/tests_$v.log 2>&1; echo "$v tests rc=$?" >> $OUT/ab.txt
done
