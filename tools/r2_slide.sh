#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/slide; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -k "rolling" > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/ab.txt
for R in 24 5 2 168; do bash tools/ab_mode.sh "--config C4 --refit-stride $R --steps 5 --warmup 3" r24o slide | sed "s/^/R$R /" >> $OUT/ab.txt 2>&1; done
timeout 900 python bench.py --config C4 --refit-stride 24 --steps 5 --warmup 3 > $OUT/bench_roll24.json 2> $OUT/bench_roll24.err; echo "bench roll24 rc=$?" >> $OUT/ab.txt
