#!/bin/bash
# headline kernel geometry A/B (warps per CTA x windows per lane per chunk)
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/geom; rm -rf $OUT; mkdir -p $OUT
bash tools/ab_mode.sh "--steps 10 --warmup 3" cfh w12c92 w12c84 w14c76 w10c108 w12c100 cfh > $OUT/ab.txt 2>&1
for P in 3 24 12; do bash tools/ab_mode.sh "--steps 10 --warmup 3 --period-steps $P" cfh w12c92 w12c84 | sed "s/^/P$P /" >> $OUT/ab.txt 2>&1; done
