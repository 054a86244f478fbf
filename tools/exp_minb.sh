#!/bin/bash
# occupancy of the C2-shape pair kernels: pass 1 at 4 CTAs/SM (128 registers, small spill) and
# pass 2 (prefix sharing) at 5 CTAs/SM, against the defaults (3 and 4)
for V in "" "-DBSIDMAP_L1C_MINB=3" "-DBSIDMAP_L1C_MINB=4 -DBSIDMAP_L1_GROUP=1" "-DBSIDMAP_APP_MINB_PRE=5"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py C2:65536 C1:16384
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
