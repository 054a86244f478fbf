#!/bin/bash
# rows per dispatch group after the fused tails (rows_then): APP and pass 1, single rows vs pairs
for V in "-DBSIDMAP_APP_GROUP=1" "-DBSIDMAP_L1_GROUP=1"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py C2:65536 C1:16384 --iters 5
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
