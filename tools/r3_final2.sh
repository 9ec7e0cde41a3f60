#!/bin/bash
# round-3 session end, second pass: GPU suite on the in-tree build, C5 line, odd-period lines
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/r3final2; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "gpu tests rc=$?" | tee -a $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/status.txt
timeout 900 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench rc=$?" | tee -a $OUT/status.txt
for P in 3 5 15 2; do
  timeout 900 python bench.py --period-steps $P --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_p$P.json 2> $OUT/bench_p$P.err
  echo "p$P rc=$?" | tee -a $OUT/status.txt
done
