#!/bin/bash
# four-window APP kernel at 2 vs 3 CTAs/SM (C2)
for V in "-DBSIDMAP_APP4_MINB=2" "-DBSIDMAP_APP4_MINB=3"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  BSIDMAP_APP_X4=1 KTAG="[$V x4]" python tools/ktime.py C2:65536 C1:16384
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
