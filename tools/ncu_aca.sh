#!/bin/bash
# Full ncu capture of one big ACA wave (row + column kernels) at n=200;
# exports details/raw/source pages as CSV so the report itself need not travel.
OUT=gpurun_out/ncu_aca
mkdir -p $OUT
timeout 800 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_aca_} -s ${SKIP:-2} -c ${COUNT:-2} \
  -o /tmp/aca_prof python bench.py --n ${N:-200} --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/run.log 2>&1
ncu -i /tmp/aca_prof.ncu-rep --page details --csv > $OUT/details.csv 2>&1
ncu -i /tmp/aca_prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>&1
ncu -i /tmp/aca_prof.ncu-rep --page source --csv --print-source sass > $OUT/source_sass.csv 2>&1
ls -la $OUT
