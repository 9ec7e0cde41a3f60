#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/r24; rm -rf $OUT; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -k "rolling" > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/ab.txt
for R in 24 5; do bash tools/ab_mode.sh "--config C4 --refit-stride $R --steps 5 --warmup 3" r24base r24o r24base r24o | sed "s/^/R$R /" >> $OUT/ab.txt 2>&1; done
