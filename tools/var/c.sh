HBEM_PROF=1 HBEM_LIB=var/lib_prof.so timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e 2>&1 | grep "hbem prof" | tail -3
HBEM_PROF=1 HBEM_LIB=var/lib_prof.so timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --precision single 2>&1 | grep "hbem prof" | tail -3
