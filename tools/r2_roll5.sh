#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/roll5; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rolling.py -q -x -p no:cacheprovider > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
bash tools/ab_mode.sh "--config C4 --refit-stride 1 --steps 10" base > $OUT/ab.txt 2>&1
bash tools/ab_mode.sh "--config C4 --refit-stride 24 --steps 10" base >> $OUT/ab.txt 2>&1
CHASE_ROLL_RUNS=1 bash tools/ab_mode.sh "--config C4 --refit-stride 1 --steps 10" base | sed 's/^base/runs/' >> $OUT/ab.txt 2>&1
