#!/bin/bash
# one ncu --set full command over C1-C4 (second call of each captured): tools/r2_ncu_cfg.sh configs|periods
cd "$GRAFT_REPO_ROOT" || exit 1
what=$1
OUT=gpurun_out/ncu_$what; rm -rf $OUT; mkdir -p $OUT
timeout 600 python tools/ncu_workloads.py $what > $OUT/plain.log 2>&1 || { echo "plain run failed"; cat $OUT/plain.log; exit 1; }
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:"sweep" -c 8 \
    -o $OUT/$what python tools/ncu_workloads.py $what > $OUT/ncu.log 2>&1
echo "ncu rc=$?"
