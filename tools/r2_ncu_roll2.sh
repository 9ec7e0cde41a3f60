#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/roll6; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_rolling.py -q -p no:cacheprovider > $OUT/tests.log 2>&1; echo "rc=$?" >> $OUT/tests.log
ARGS="--config C4 --refit-stride ${RS:-1} --traces 20000 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > $OUT/plain.json 2> $OUT/plain.err &&
ncu --set full --import-source on --clock-control none -k regex:roll_lane -s 1 -c 1 -o $OUT/lane${RS:-1} -f \
    python bench.py $ARGS > $OUT/ncu.log 2>&1
echo "ncu_rc=$?" >> $OUT/ncu.log
