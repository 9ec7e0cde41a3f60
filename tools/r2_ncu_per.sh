#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/ncu_periods; rm -rf $OUT; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -k "shaped or nondyadic or band" > $OUT/tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/ncu_workloads.py periods > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:"sweep" -c 8 \
    -o $OUT/periods python tools/ncu_workloads.py periods > $OUT/ncu.log 2>&1
echo "ncu rc=$?"
