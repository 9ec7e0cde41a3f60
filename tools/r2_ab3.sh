#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/ab3; mkdir -p $OUT
bash tools/ab_mode.sh "--steps 20 --warmup 3" base cfma base cfma > $OUT/ab.txt 2>&1
for P in 2 3 24 168; do bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps $P" base | sed "s/^base/P$P/" >> $OUT/ab.txt 2>&1; done
