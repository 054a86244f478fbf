#!/bin/bash
# APP weight dot fused into the last lattice row's basic block (rows_then) vs after the branch merge
for V in "-DBSIDMAP_APP_FUSED_DOT=0" ""; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py C2:65536 C1:16384 C4:512 C3:2048 C5:32
done
