#!/bin/bash
# Build libhbem_b200 variants that differ only in the ACA P0 kernel's compile-time
# knobs (job group width, CTAs per SM), for a timing sweep on the GPU:
#   tools/var/build_variants.sh "1:4 1:5 2:3"  ->  var/lib_G1_M4.so ...
# Select one at run time with HBEM_LIB=var/lib_G1_M4.so.
set -e
cd "$(dirname "$0")/../.."
make -s -j8 all
mkdir -p var build/var
OTHER=$(ls build/*.o | grep -v kern_f64.o | grep -v kern_f32.o)
for v in $1; do
  G=${v%%:*}; M=${v##*:}
  for f in kern_f64 kern_f32; do
    nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
      -Xcompiler -ffp-contract=off --expt-relaxed-constexpr -DHB_JOB_GROUP=$G -DHB_ACA_P0_MINB=$M \
      -c paper_1711_01897_b200/csrc/$f.cu -o build/var/${f}_G${G}_M${M}.o &
  done
done
wait
for v in $1; do
  G=${v%%:*}; M=${v##*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o var/lib_G${G}_M${M}.so $OTHER \
    build/var/kern_f64_G${G}_M${M}.o build/var/kern_f32_G${G}_M${M}.o -lcudart
done
ls -la var/
