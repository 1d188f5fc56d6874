#!/bin/bash
# One exploratory gpurun session: micro checks, GPU tests, variant sweep.
#   STAGES="micro tests sweep" tools/var/session.sh
OUT=gpurun_out; mkdir -p $OUT
STAGES=${STAGES:-"micro tests sweep"}
has() { [[ " $STAGES " == *" $1 "* ]]; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
if has micro; then
  for b in var/rsq_accuracy; do [ -x $b ] && timeout 120 $b > $OUT/$(basename $b).txt 2>&1; done
  cat $OUT/rsq_accuracy.txt
fi
if has tests; then
  timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q ${TESTS:-} > $OUT/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $OUT/pytest_gpu.log; tail -15 $OUT/pytest_gpu.log
fi
if has sweep; then
  tools/var/sweep.sh 2>&1 | tee $OUT/sweep.txt
fi
