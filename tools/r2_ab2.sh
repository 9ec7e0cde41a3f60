#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/ab2
bash tools/ab_mode.sh "--steps 20 --warmup 3" base w18c52 w20c44 w20c52 w24c44 w24c36 > gpurun_out/ab2/ab.txt 2>&1
bash tools/ab_mode.sh "--steps 20 --warmup 3" base w20c52 w24c44 >> gpurun_out/ab2/ab.txt 2>&1
