#!/bin/bash
# A/B the sweep kernel variants built by tools/build_variant.sh (tuning only).
# Usage: tools/ab_bench.sh name1 name2 ...   -> gpurun_out/ab_<name>.json
mkdir -p gpurun_out
for v in "$@"; do
  lib=build/variants/libchase_$v.so
  [ "$v" = "base" ] && lib=paper_2303_02508_b200/libchase.so
  CHASE_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline \
     > gpurun_out/ab_$v.log 2>&1
  echo "$v rc=$? $(grep '^{' gpurun_out/ab_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("kernel_ms=%.3f frac=%.4f step_ms=%.3f" % (r["kernel_ms"], r["frac"], d["ms_per_step"]))')"
done
