#!/bin/bash
# one ncu --set full command: the fused rolling-refit kernel at C4, R = 1 (second launch)
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/ncu_roll; rm -rf $OUT; mkdir -p $OUT
timeout 600 python bench.py --config C4 --refit-stride 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-prefix-check > $OUT/plain.json 2>&1 || { echo plain failed; exit 1; }
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"roll" -s 1 -c 1 \
    -o $OUT/roll1 python bench.py --config C4 --refit-stride 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-prefix-check > $OUT/ncu.log 2>&1
echo "ncu rc=$?"
