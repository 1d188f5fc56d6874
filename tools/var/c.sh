timeout 900 python -m pytest tests/test_gpu_c3.py tests/test_gpu_hmatrix.py tests/test_gpu_configs.py -q -x -k "not c4" 2>&1 | tail -3
HBEM_PROF=1 HBEM_LIB=var/lib_prof.so timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e 2>&1 | grep "hbem prof" | tail -1
LIBS="var/lib_head.so var/lib_stage.so" bash tools/var/cmp.sh
LIBS="var/lib_head.so var/lib_stage.so" PRECS=single tools/var/sweep.sh
