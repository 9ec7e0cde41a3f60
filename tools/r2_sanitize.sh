#!/bin/bash
# One compute-sanitizer tool per call (B200_PROFILING.md): TOOL=memcheck|racecheck|synccheck
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/sanitize; mkdir -p $OUT
timeout 600 python tools/sanitize_driver.py > $OUT/plain_$TOOL.log 2>&1 &&
timeout 2400 compute-sanitizer --tool $TOOL --print-limit 50 \
    python tools/sanitize_driver.py > $OUT/$TOOL.log 2>&1
echo "rc=$?" >> $OUT/$TOOL.log
