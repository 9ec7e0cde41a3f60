#!/bin/bash
# A/B library variants on one bench mode (tuning only).
# Usage: tools/ab_mode.sh "<bench args>" name1 name2 ...  (base = the in-tree library)
args=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  lib=build/variants/libchase_$v.so; [ "$v" = "base" ] && lib=paper_2303_02508_b200/libchase.so
  CHASE_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/abx_$v.log 2>&1
  echo "$v $(grep '^{' gpurun_out/abx_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("kernel_ms=%.3f frac=%.4f step_ms=%.3f" % (r["kernel_ms"], r["frac"], d["ms_per_step"]))')"
done
