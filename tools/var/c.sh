LIBS="var/lib_j1.so var/lib_j8.so var/lib_j12.so" bash tools/var/cmp.sh
