#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/roll2; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rolling.py -q -x -p no:cacheprovider > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
bash tools/ab_mode.sh "--config C4 --refit-stride 1 --steps 10" base r1 > $OUT/ab.txt 2>&1
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_r1.so timeout 900 python -m pytest tests/test_gpu_rolling.py -q -x -p no:cacheprovider > $OUT/tests_r1.log 2>&1; echo "rc=$?" >> $OUT/tests_r1.log
