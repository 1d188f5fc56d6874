#!/bin/bash
# ncu evidence for one library variant: launch list of one assembly + a full
# capture (with SASS source counters) of KREGEX launches [SKIP, SKIP+COUNT).
#   HBEM_LIB=var/lib_G1_M4.so KREGEX=k_aca_p0 SKIP=2 COUNT=2 tools/var/ncu_session.sh
OUT=gpurun_out; mkdir -p $OUT
TAG=${TAG:-x}
ARGS=${ARGS:-"--steps 1 --warmup 1 --no-e2e --no-cpu"}
if [ -z "$NO_LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_$TAG.csv python bench.py $ARGS > $OUT/launches_${TAG}_run.log 2>&1
echo "launches exit $?"
fi
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_aca_p0} \
  -s ${SKIP:-2} -c ${COUNT:-2} -f -o /tmp/prof python bench.py $ARGS > $OUT/full_${TAG}_run.log 2>&1
echo "full exit $?"
ncu -i /tmp/prof.ncu-rep --page details --csv > $OUT/full_${TAG}_details.csv 2>&1
ncu -i /tmp/prof.ncu-rep --page raw --csv > $OUT/full_${TAG}_raw.csv 2>&1
ncu -i /tmp/prof.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > $OUT/full_${TAG}_source.csv.gz
ls -la $OUT | tail -5
