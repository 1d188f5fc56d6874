HBEM_LIB=var/lib_i8.so timeout 900 python -m pytest tests/test_gpu_c3.py tests/test_gpu_hmatrix.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
bash tools/var/cmp.sh 2>&1 | grep -v "^$"
