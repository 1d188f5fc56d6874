timeout 900 python -m pytest tests/test_gpu_c3.py tests/test_gpu_hmatrix.py tests/test_gpu_configs.py -q -x -k "not c4" 2>&1 | tail -3
bash tools/var/cmp.sh
