for v in base kv1 kv4 base; do
  lib=build/variants/libchase_$v.so; [ "$v" = "base" ] && lib=paper_2303_02508_b200/libchase.so
  CHASE_LIB_OVERRIDE=$PWD/$lib timeout 300 python bench.py --mode mape --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abm_$v.log 2>&1
  echo "$v $(grep '^{' gpurun_out/abm_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("kernel_ms=%.3f frac=%.4f" % (r["kernel_ms"], r["frac"]))')"
done
