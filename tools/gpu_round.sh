#!/bin/bash
# One gpurun call: GPU tests, smoke, bench line, ncu launch list and one full
# ncu capture of the top integration kernel.  Everything lands in gpurun_out/.
#   STAGES="tests smoke bench launches full ref" (default: all)
OUT=gpurun_out
mkdir -p $OUT
STAGES=${STAGES:-"tests smoke bench launches full"}
N=${N:-448}
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
has() { [[ " $STAGES " == *" $1 "* ]]; }
if has tests; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
fi
if has smoke; then
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
  echo "smoke exit $?" >> $OUT/smoke.log; tail -2 $OUT/smoke.log
fi
if has bench; then
  timeout 1500 python bench.py --n $N $BENCH_ARGS > $OUT/bench.json 2> $OUT/bench.err
  echo "bench exit $?"; tail -c 3000 $OUT/bench.json
fi
if has ref; then
  timeout 900 python bench.py --impl reference --n $N --steps 1 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
  echo "ref exit $?"; cat $OUT/bench_ref.json
fi
if has launches; then
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --n $N --steps 1 --warmup 1 --no-e2e --no-cpu \
    > $OUT/launches_run.log 2>&1
  echo "launches exit $?"; wc -l $OUT/launches.csv
fi
if has full; then
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_int} \
    -s ${SKIP:-4} -c ${COUNT:-2} -f -o /tmp/prof python bench.py --n $N --steps 1 --warmup 1 \
    --no-e2e --no-cpu > $OUT/full_run.log 2>&1
  echo "full exit $?"
  # the .ncu-rep (~85 MB) exceeds the 64 MiB gpurun_out cap: export CSV pages only
  ncu -i /tmp/prof.ncu-rep --page details --csv > $OUT/full_details.csv 2>&1
  ncu -i /tmp/prof.ncu-rep --page raw --csv > $OUT/full_raw.csv 2>&1
  ncu -i /tmp/prof.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > $OUT/full_source.csv.gz 2>&1
  ls -la $OUT
fi
if has full2; then
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:${KREGEX2:-k_near} \
    -s ${SKIP2:-0} -c 1 -f -o /tmp/prof2 python bench.py --n $N --steps 1 --warmup 1 \
    --no-e2e --no-cpu > $OUT/full2_run.log 2>&1
  echo "full2 exit $?"
  ncu -i /tmp/prof2.ncu-rep --page details --csv > $OUT/full2_details.csv 2>&1
  ncu -i /tmp/prof2.ncu-rep --page raw --csv > $OUT/full2_raw.csv 2>&1
  ncu -i /tmp/prof2.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > $OUT/full2_source.csv.gz
fi
