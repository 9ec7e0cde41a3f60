#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/ws; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?" | tee -a $OUT/status.txt
run() { name=$1; shift; timeout 900 python bench.py "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$?" | tee -a $OUT/status.txt; }
run bench_p24_full --period-steps 24
run bench_p168_full --period-steps 168
run bench_roll1 --config C4 --refit-stride 1 --steps 5 --warmup 3
