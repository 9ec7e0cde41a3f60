#!/bin/bash
# The round's bench lines (profiles/r1_bench/): every mode on its config.
mkdir -p gpurun_out/final
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/final/$name.json 2> gpurun_out/final/$name.err; echo "$name rc=$?"; }
run bench_full
run bench_ref --impl reference --steps 3 --warmup 1
run bench_svr_c4 --config C4 --forecaster svr --steps 5 --warmup 3
run bench_svr_mape_c4 --mode mape --config C4 --forecaster svr --steps 5 --warmup 3
run bench_roll1 --config C4 --refit-stride 1 --steps 5 --warmup 3
run bench_roll24 --config C4 --refit-stride 24 --steps 5 --warmup 3
run bench_p24 --period-steps 24 --steps 10 --warmup 3
run bench_p168 --period-steps 168 --steps 10 --warmup 3
run bench_p2 --period-steps 2 --steps 10 --warmup 3
run bench_mape --mode mape --steps 10 --warmup 3
run bench_timeline_p1 --mode timeline --config C4 --period-steps 1 --steps 10 --warmup 3
run bench_timeline_p24 --mode timeline --config C4 --period-steps 24 --steps 10 --warmup 3
