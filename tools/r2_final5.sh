#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/final5; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?" | tee -a $OUT/status.txt
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_checked.so timeout 1500 python -m pytest tests -m gpu -q > $OUT/checked_gpu_tests.log 2>&1; echo "checked tests rc=$?" | tee -a $OUT/status.txt
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_checked.so timeout 600 python tools/sanitize_driver.py > $OUT/checked_driver.log 2>&1; echo "checked driver rc=$?" | tee -a $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/status.txt
timeout 300 python tools/cfh_probe.py 4000 > $OUT/cfh_probe.txt 2>&1
run() { name=$1; shift; timeout 900 python bench.py "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$?" | tee -a $OUT/status.txt; }
for P in 2 3 4 5 6 10 12 15 24 48 168 720; do run bench_p$P --period-steps $P --steps 10 --warmup 3 --no-cpu-baseline; done
run bench_p24_full --period-steps 24
run bench_timeline_p24 --mode timeline --config C4 --period-steps 24 --steps 10 --warmup 3
