#!/bin/bash
# Closing run of the round: GPU tests, smoke, default bench lines (FP64, FP32, reference arm).
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/r02z_pytest_gpu.log 2>&1; tail -2 $OUT/r02z_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r02z_smoke.log 2>&1; tail -1 $OUT/r02z_smoke.log
timeout 900 python bench.py > $OUT/r02z_bench.json 2> $OUT/r02z_bench.err; tail -c 300 $OUT/r02z_bench.json
timeout 900 python bench.py --precision single --no-cpu > $OUT/r02z_bench_fp32.json 2> $OUT/r02z_bench_fp32.err
timeout 900 python bench.py --impl reference > $OUT/r02z_bench_ref.json 2> $OUT/r02z_bench_ref.err
