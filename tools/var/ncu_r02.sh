#!/bin/bash
# Round-2 ncu evidence: launch lists (FP64, FP32), DRAM traffic of every
# k_aca_p0 launch of one assembly, full captures of the top kernels.
OUT=gpurun_out; mkdir -p $OUT
A="--steps 1 --warmup 1 --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r02_launches_fp64.csv python bench.py $A > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r02_launches_fp32.csv python bench.py --precision single $A > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_aca_p0 -s 30 -c 30 --csv --log-file $OUT/r02_traffic_k_aca_p0.csv python bench.py $A > /dev/null 2>&1
for spec in "k_aca_p0:2:2:fp64:double" "k_sing_table:1:1:sing:double" "k_near_p0:1:1:near:double" "k_aca_p0:2:1:fp32:single" "k_fin_col:4:1:fincol:double"; do
  IFS=: read K S C T P <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C -f -o /tmp/p_$T python bench.py --precision $P $A > /dev/null 2>&1
  ncu -i /tmp/p_$T.ncu-rep --page raw --csv > $OUT/r02_full_${T}_raw.csv 2>&1
  ncu -i /tmp/p_$T.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > $OUT/r02_full_${T}_source.csv.gz
done
ls -la $OUT | grep r02
