#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/roll8; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rolling.py -q -p no:cacheprovider > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
bash tools/ab_mode.sh "--config C4 --refit-stride 1 --steps 10" base t64w8 > $OUT/ab.txt 2>&1
bash tools/ab_mode.sh "--config C4 --refit-stride 24 --steps 10" base t64w8 >> $OUT/ab.txt 2>&1
