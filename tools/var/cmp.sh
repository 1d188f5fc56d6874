#!/bin/bash
# Payload digests + C5 timing of library variants (LIBS, default every var/lib_*.so).
LIBS=${LIBS:-$(ls var/lib_*.so)}
for L in $LIBS; do echo "$L $(HBEM_LIB=$L timeout 300 python tools/var/digest.py 60 p0 laplace slp 0 double 2>&1 | tail -1 | cut -c1-80)"; done
LIBS="$LIBS $LIBS" PRECS=${PRECS:-double} tools/var/sweep.sh
