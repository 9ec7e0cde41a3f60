#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/final2; mkdir -p $OUT
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_checked.so timeout 600 python tools/sanitize_driver.py > $OUT/checked_driver.log 2>&1; echo "checked driver rc=$?" | tee -a $OUT/status2.txt
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_checked.so timeout 1500 python -m pytest tests -m gpu -q > $OUT/checked_gpu_tests.log 2>&1; echo "checked tests rc=$?" | tee -a $OUT/status2.txt
timeout 900 python bench.py --mode mape --steps 10 --warmup 3 > $OUT/bench_mape.json 2> $OUT/bench_mape.err; echo "mape rc=$?" | tee -a $OUT/status2.txt
