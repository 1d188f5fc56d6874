#!/bin/bash
# Full ncu capture of one k_aca_p0 launch (SKIP selects the wave) exported per
# CUDA source line and per SASS instruction, for the epilogue/staging breakdown.
#   SKIP=14 TAG=w7 tools/var/ncu_lines.sh
OUT=gpurun_out; mkdir -p $OUT
TAG=${TAG:-x}
ARGS=${ARGS:-"--steps 1 --warmup 1 --no-e2e --no-cpu"}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_aca_p0} \
  -s ${SKIP:-14} -c 1 -f -o /tmp/prof python bench.py $ARGS > $OUT/lines_${TAG}_run.log 2>&1
echo "full exit $?"
ncu -i /tmp/prof.ncu-rep --page source --csv --print-source cuda 2>&1 | gzip > $OUT/lines_${TAG}_cuda.csv.gz
ncu -i /tmp/prof.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > $OUT/lines_${TAG}_sass.csv.gz
ncu -i /tmp/prof.ncu-rep --page raw --csv > $OUT/lines_${TAG}_raw.csv 2>&1
ls -la $OUT | grep lines_
