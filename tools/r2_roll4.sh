#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/roll4; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rolling.py -q -x -p no:cacheprovider > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
bash tools/ab_mode.sh "--config C4 --refit-stride 1 --steps 10" base g4m1 g2m2 g2m1 g1m2 g1m3 g8m1 > $OUT/ab.txt 2>&1
