#!/bin/bash
# round-3 session end: GPU suite (in-tree + checked build), smoke, C5 line,
# decision-period lines, and one ncu capture of the period kernels (P = 2, 3, 24, 168)
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/r3final; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?" | tee -a $OUT/status.txt
CHASE_LIB_OVERRIDE=$PWD/build/variants/libchase_checked.so timeout 1500 python -m pytest tests -m gpu -q > $OUT/checked_gpu_tests.log 2>&1; echo "checked tests rc=$?" | tee -a $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/status.txt
timeout 900 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench rc=$?" | tee -a $OUT/status.txt
for P in 2 3 4 5 6 12 15 24 168; do
  timeout 900 python bench.py --period-steps $P --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_p$P.json 2> $OUT/bench_p$P.err
  echo "p$P rc=$?" | tee -a $OUT/status.txt
done
timeout 600 python tools/ncu_workloads.py periods > $OUT/ncu_plain.log 2>&1 && \
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:"sweep" -c 8 \
    -o $OUT/periods python tools/ncu_workloads.py periods > $OUT/ncu.log 2>&1
echo "ncu rc=$?" | tee -a $OUT/status.txt
