#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/p2; rm -rf $OUT; mkdir -p $OUT
bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps 2" cfh p2cf p2cfg6 p2cfg10 > $OUT/ab.txt 2>&1
for v in p2cf p2cfg6; do
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_$v.so timeout 600 python -m pytest tests -m gpu -q -x -k "period" > $OUT/tests_$v.log 2>&1; echo "$v tests rc=$?" >> $OUT/ab.txt
done
