#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/nvtx; rm -rf $OUT; mkdir -p $OUT
timeout 300 python bench.py --config C4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-prefix-check > $OUT/plain.json 2>&1; echo "plain rc=$?"
timeout 600 ncu --nvtx --nvtx-include "chase_sweep/predict_argmin_replay/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/nvtx_launches.csv python bench.py --config C4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-prefix-check > $OUT/ncu.log 2>&1
echo "ncu rc=$?"
