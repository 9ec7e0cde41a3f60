#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/ab1
for rep in 1 2; do
bash tools/ab_mode.sh "--steps 20 --warmup 3" base f1 f2 >> gpurun_out/ab1/ab.txt 2>&1
CHASE_LEAN=1 bash tools/ab_mode.sh "--steps 20 --warmup 3" base | sed 's/^base/lean/' >> gpurun_out/ab1/ab.txt 2>&1
done
