LIBS="var/lib_head.so var/lib_hoist.so" bash tools/var/cmp.sh 2>&1 | grep -v "^$"
LIBS="var/lib_head.so var/lib_hoist.so" PRECS=single tools/var/sweep.sh
