#!/bin/bash
# rows per dispatch group in the packed-pair lattice passes (C2, C4)
for V in "" "-DBSIDMAP_APP_GROUP=3" "-DBSIDMAP_L1_GROUP=3" "-DBSIDMAP_APP_GROUP=3 -DBSIDMAP_L1_GROUP=3 -DBSIDMAP_APP_MINB_PRE=3"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  echo "=== variant: '$V'"
  for c in "C2 65536" "C4 512" "C1 16384"; do
    python tools/quick_time.py $c 0 | grep -E "frames/s" | tail -1
  done
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
