#!/bin/bash
# round-3 A/B only (no tests): variants on C5 (P = 1), three passes
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/r3ab; mkdir -p $OUT
ARGS=${ABARGS:-"--steps 10 --warmup 3"}
for r in 1 2 3; do bash tools/ab_mode.sh "$ARGS" "$@" >> $OUT/ab2.txt 2>&1; done
