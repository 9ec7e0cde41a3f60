#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/roll7; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rolling.py -q -p no:cacheprovider > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
bash tools/ab_mode.sh "--config C4 --refit-stride 1 --steps 10" base t64w8 t32w12 t32w16 t16w16 > $OUT/ab.txt 2>&1
bash tools/ab_mode.sh "--config C4 --refit-stride 24 --steps 10" base t32w12 >> $OUT/ab.txt 2>&1
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_checked.so timeout 600 python tools/sanitize_driver.py > $OUT/checked_driver.log 2>&1; echo "rc=$?" >> $OUT/checked_driver.log
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_checked.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/checked_tests.log 2>&1; echo "rc=$?" >> $OUT/checked_tests.log
