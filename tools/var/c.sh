timeout 900 python -m pytest tests/test_gpu_c3.py tests/test_gpu_hmatrix.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
bash tools/var/cmp.sh
for L in head tpiv; do HBEM_LIB=var/lib_$L.so timeout 300 python tools/var/digest.py 40 p0 helmholtz slp 3 double 2>&1 | tail -1 | cut -c1-80; done
