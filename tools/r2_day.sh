#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/day; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -k "period" > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/ab.txt
bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps 24" noday day noday day >> $OUT/ab.txt 2>&1
