#!/bin/bash
# round-3 A/B: variants on C5 (P = 1) + headline tests on the first variant
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/r3ab; rm -rf $OUT; mkdir -p $OUT
V1=$1; shift
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_$V1.so timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_headline.py tests/test_gpu_parity.py > $OUT/tests.log 2>&1
echo "tests rc=$?" >> $OUT/tests.log
bash tools/ab_mode.sh "--steps 10 --warmup 3" "$@" > $OUT/ab.txt 2>&1
bash tools/ab_mode.sh "--steps 10 --warmup 3" "$@" >> $OUT/ab.txt 2>&1
