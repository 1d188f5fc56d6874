#!/bin/bash
# registers / spills of one kernel in a ptxas -v log:  tools/var/regs.sh LOG SYMBOL-SUBSTRING
awk -v s="$2" '/Compiling entry function/ {on = index($0, s) > 0} on && /spill|Used/ {print}' "$1" | head -4
