# timing-only comparison of experimental builds (results of the variants are not valid)
for v in default $(ls variants/*.so 2>/dev/null); do
  if [ "$v" = default ]; then unset HBEM_LIB; else export HBEM_LIB=$PWD/$v; fi
  echo "== $v"
  timeout 600 python bench.py --no-cpu --no-e2e --steps 3 --warmup 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['int_kernel_ms_per_step'], d['roofline']['aca_waves_ms_per_step'])"
done
