#!/bin/bash
# Time bench.py (C5, FP64 and FP32 by default) with every library variant in var/.
#   PRECS="double single" ARGS="--steps 5 --warmup 3" tools/var/sweep.sh
OUT=gpurun_out; mkdir -p $OUT
PRECS=${PRECS:-"double"}
ARGS=${ARGS:-"--steps 5 --warmup 3 --no-cpu --no-e2e"}
for lib in ${LIBS:-var/*.so}; do
  for p in $PRECS; do
    HBEM_LIB=$lib timeout 600 python bench.py --precision $p $ARGS > $OUT/sweep_$(basename $lib .so)_$p.json 2>$OUT/sweep_$(basename $lib .so)_$p.err
    python - "$lib" "$p" $OUT/sweep_$(basename $lib .so)_$p.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], sys.argv[2], "ms/step %.1f" % d["ms_per_step"], "int_ms %.1f" % r["int_kernel_ms_per_step"],
          "waves_ms %.1f" % r["aca_waves_ms_per_step"], "frac %.3f" % r["frac"], "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e)
PY
  done
done
