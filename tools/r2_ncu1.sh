#!/bin/bash
# one ncu --set full capture of the headline kernel for the given bench args: tools/r2_ncu1.sh name "<bench args>"
cd "$GRAFT_REPO_ROOT" || exit 1
name=$1; args=$2
OUT=gpurun_out/ncu1; mkdir -p $OUT
timeout 300 python bench.py $args --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-prefix-check > $OUT/$name.plain.json 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_fast -s 3 -c 1 \
    -o $OUT/$name python bench.py $args --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-prefix-check > $OUT/$name.ncu.log 2>&1
echo "ncu rc=$?"
