#!/bin/bash
# Round-2 final evidence: full GPU tests, smoke, checked build, bench lines, launch list.
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/final3; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?" | tee -a $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/status.txt
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_checked.so timeout 600 python tools/sanitize_driver.py > $OUT/checked_driver.log 2>&1; echo "checked driver rc=$?" | tee -a $OUT/status.txt
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_checked.so timeout 1500 python -m pytest tests -m gpu -q > $OUT/checked_gpu_tests.log 2>&1; echo "checked tests rc=$?" | tee -a $OUT/status.txt
run() { name=$1; shift; timeout 900 python bench.py "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$?" | tee -a $OUT/status.txt; }
run bench_c5
for c in C1 C2 C3 C4; do run bench_$(echo $c | tr C c) --config $c; done
for P in 2 3 5 12 24 168 720; do run bench_p$P --period-steps $P --steps 10 --warmup 3 --no-cpu-baseline; done
run bench_mape --mode mape --steps 10 --warmup 3
run bench_timeline_p24 --mode timeline --config C4 --period-steps 24 --steps 10 --warmup 3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-prefix-check > $OUT/launches_c5.log 2>&1
echo "launches rc=$?" | tee -a $OUT/status.txt
