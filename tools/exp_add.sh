#!/bin/bash
# pass-1 class-sum update fused into the last row group's basic block (rows_then) vs after it
for V in "-DBSIDMAP_L1_FUSED_ADD=0" ""; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py C2:65536 C1:16384 C4:512
done
