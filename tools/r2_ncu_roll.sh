#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/roll3; mkdir -p $OUT
ARGS="--config C4 --refit-stride 1 --traces 20000 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
export CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_${VAR:-r1}.so
python bench.py $ARGS > $OUT/plain.json 2> $OUT/plain.err &&
ncu --set full --import-source on --clock-control none -k regex:roll_fused -s 1 -c 1 -o $OUT/${VAR:-roll} -f \
    python bench.py $ARGS > $OUT/ncu.log 2>&1
echo "ncu_rc=$?" >> $OUT/ncu.log
