#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/final4; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?" | tee -a $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/status.txt
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_checked.so timeout 1500 python -m pytest tests -m gpu -q > $OUT/checked_gpu_tests.log 2>&1; echo "checked tests rc=$?" | tee -a $OUT/status.txt
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_checked.so timeout 600 python tools/sanitize_driver.py > $OUT/checked_driver.log 2>&1; echo "checked driver rc=$?" | tee -a $OUT/status.txt
run() { name=$1; shift; timeout 900 python bench.py "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$?" | tee -a $OUT/status.txt; }
run bench_roll1 --config C4 --refit-stride 1 --steps 5 --warmup 3
run bench_roll24 --config C4 --refit-stride 24 --steps 5 --warmup 3
run bench_svr_c4 --config C4 --forecaster svr --steps 5 --warmup 3
run bench_ref --impl reference --steps 3 --warmup 3
run bench_c3 --config C3
run bench_c5
