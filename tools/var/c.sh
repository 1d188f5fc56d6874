for L in u4 u2 u8; do HBEM_LIB=var/lib_$L.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_sing_lanes --csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e 2>/dev/null | grep k_sing_lanes | awk -F'","' -v l=$L '{print l, $NF}'; done
bash tools/var/cmp.sh 2>&1 | grep -v "^$" | grep ms/step
