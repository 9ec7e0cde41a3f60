mkdir -p gpurun_out/final
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/final/$name.json 2> gpurun_out/final/$name.err; echo "$name rc=$?"; }
run bench_p24 --period-steps 24 --steps 10 --warmup 3
run bench_p168 --period-steps 168 --steps 10 --warmup 3
run bench_p2 --period-steps 2 --steps 10 --warmup 3
run bench_full
bash tools/period_profiles.sh
