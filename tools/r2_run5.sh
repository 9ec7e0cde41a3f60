#!/bin/bash
# GPU call: lean kernel correctness + bench + ncu
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/${TAG:-r2d}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_headline.py -q -x -p no:cacheprovider > $OUT/headline_tests.log 2>&1
echo "rc=$?" >> $OUT/headline_tests.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gpu_tests.log 2>&1
echo "rc=$?" >> $OUT/gpu_tests.log
timeout 600 python bench.py --no-e2e > $OUT/bench_c5.json 2> $OUT/bench_c5.err
timeout 600 python bench.py --config C4 --no-e2e --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
ARGS="--traces 250000 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > $OUT/ncu_plain.json 2> $OUT/ncu_plain.err &&
ncu --set full --import-source on --clock-control none -k regex:lean -s 2 -c 1 -o $OUT/lean -f \
    python bench.py $ARGS > $OUT/ncu.log 2>&1
echo "ncu_rc=$?" >> $OUT/ncu.log
