#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/roll1; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rolling.py -q -x -p no:cacheprovider > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
timeout 600 python bench.py --config C4 --refit-stride 1 --no-e2e --steps 10 > $OUT/bench_r1.json 2> $OUT/bench_r1.err
timeout 600 python bench.py --config C4 --refit-stride 24 --no-e2e --no-cpu-baseline --steps 10 > $OUT/bench_r24.json 2> $OUT/bench_r24.err
bash tools/ab_mode.sh "--config C4 --refit-stride 1 --steps 10" base r1 > $OUT/ab.txt 2>&1
