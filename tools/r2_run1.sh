#!/bin/bash
# Round 2, GPU call 1: the GPU suite, the smoke, then the bench lines of C5 (headline) and C1-C4.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/r2/gpu_tests.log 2>&1
echo "gpu_tests_rc=$?" >> gpurun_out/r2/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/r2/smoke.log
timeout 600 python bench.py > gpurun_out/r2/bench_c5.json 2> gpurun_out/r2/bench_c5.err
for c in C1 C2 C3 C4; do
  timeout 600 python bench.py --config $c > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err
done
