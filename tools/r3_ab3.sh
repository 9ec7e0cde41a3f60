#!/bin/bash
# round-3: full GPU suite on variant $1, then period A/B (P = 2, 6, 3, 24) and C5
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/r3ab; mkdir -p $OUT
V1=$1; shift
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_$V1.so timeout 1200 python -m pytest -q -x -m gpu tests > $OUT/tests_$V1.log 2>&1
echo "tests rc=$?" >> $OUT/tests_$V1.log
for P in ${PERIODS:-2 6}; do bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps $P" "$@" | sed "s/^/P$P /" >> $OUT/ab3.txt 2>&1; done
for P in ${PERIODS:-2 6}; do bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps $P" "$@" | sed "s/^/P$P /" >> $OUT/ab3.txt 2>&1; done
