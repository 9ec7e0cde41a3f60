#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/p24; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -k "period" > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/ab.txt
bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps 24" cfh p24d cfh p24d >> $OUT/ab.txt 2>&1
