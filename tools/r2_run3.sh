#!/bin/bash
# GPU call: headline tests + full gpu suite, smoke, C5 bench (one-fma key)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests/test_gpu_headline.py -q -x -p no:cacheprovider > gpurun_out/r2c/headline_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c/headline_tests.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c/gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c/gpu_tests.log
timeout 600 python bench.py --no-e2e > gpurun_out/r2c/bench_c5.json 2> gpurun_out/r2c/bench_c5.err
timeout 600 python bench.py --config C4 --no-e2e --no-cpu-baseline > gpurun_out/r2c/bench_c4.json 2> gpurun_out/r2c/bench_c4.err
