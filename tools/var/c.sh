LIBS="var/lib_head.so var/lib_redux.so" bash tools/var/cmp.sh
LIBS="var/lib_head.so var/lib_redux.so" PRECS=single tools/var/sweep.sh
