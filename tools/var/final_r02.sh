#!/bin/bash
# Round-2 closing evidence: launch lists, k_aca_p0 DRAM traffic per launch,
# full captures of the top kernels, phase cycles (HB_PROF build), bench lines.
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02f_pytest_gpu.log 2>&1; tail -2 gpurun_out/r02f_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; tail -1 gpurun_out/r02f_smoke.log
A="--steps 1 --warmup 1 --no-e2e --no-cpu"
TAG=r02f tools/var/launches.sh > $OUT/r02f_launches.txt 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_aca_p0 -s 30 -c 30 --csv --log-file $OUT/r02f_traffic_k_aca_p0.csv python bench.py $A > /dev/null 2>&1
for spec in "k_aca_p0:6:2:aca:double" "k_sing_lanes:0:1:sing:double" "k_jobs:10:1:jobs:double" "k_fin_col:6:1:fincol:double" "k_near_p0:1:1:near:double" "k_aca_p0:6:1:aca32:single"; do
  IFS=: read K S C T P <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C -f -o /tmp/p_$T python bench.py --precision $P $A > /dev/null 2>&1
  ncu -i /tmp/p_$T.ncu-rep --page raw --csv > $OUT/r02f_full_${T}_raw.csv 2>&1
  ncu -i /tmp/p_$T.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > $OUT/r02f_full_${T}_source.csv.gz
done
for p in double single; do
  HBEM_PROF=1 HBEM_LIB=var/lib_prof.so timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --precision $p 2>&1 | grep "hbem prof" | tail -1 >> $OUT/r02f_phase_cycles.txt
done
timeout 900 python bench.py > $OUT/r02f_bench.json 2> $OUT/r02f_bench.err
timeout 900 python bench.py --precision single --no-cpu > $OUT/r02f_bench_fp32.json 2> $OUT/r02f_bench_fp32.err
timeout 900 python bench.py --impl reference > $OUT/r02f_bench_ref.json 2> $OUT/r02f_bench_ref.err
ls -la $OUT | grep r02f
