#!/bin/bash
# ncu --set full capture (with source counters) of the headline kernel at a quarter of C5 (current build).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/r3
ARGS="--traces 250000 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r3/c5_plain.json 2> gpurun_out/r3/c5_plain.err
ncu --set full --import-source on --clock-control none -k regex:sweep_fast -s 2 -c 1 -o gpurun_out/r3/${TAG:-h0} -f \
    python bench.py $ARGS > gpurun_out/r3/ncu_h0.log 2>&1
echo "ncu_rc=$?" >> gpurun_out/r3/ncu_h0.log
