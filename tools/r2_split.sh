#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/split; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt
timeout 600 python bench.py --config C3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "c3 rc=$?" >> $OUT/status.txt
CHASE_NO_ETA_SPLIT=1 timeout 600 python bench.py --config C3 --no-cpu-baseline > $OUT/bench_c3_nosplit.json 2> $OUT/bench_c3_nosplit.err; echo "c3 nosplit rc=$?" >> $OUT/status.txt
