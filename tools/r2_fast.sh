#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/fast; rm -rf $OUT; mkdir -p $OUT
bash tools/ab_mode.sh "--steps 20 --warmup 3" base3 f1 f2 base3 f1 f2 > $OUT/ab.txt 2>&1
for v in f1 f2; do
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_$v.so timeout 900 python -m pytest tests -m gpu -q -x -k "headline or parity" > $OUT/tests_$v.log 2>&1; echo "$v tests rc=$?" >> $OUT/ab.txt
done
