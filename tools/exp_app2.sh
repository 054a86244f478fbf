#!/bin/bash
# pass-2 variants: row grouping, occupancy, prefix sharing (C2, C4, C1)
run() {
  for c in "C2 65536" "C4 512" "C1 16384"; do
    python tools/quick_time.py $c 0 | grep -E "frames/s" | tail -1
  done
}
for V in "" "-DBSIDMAP_APP_GROUP=1" "-DBSIDMAP_APP_MINB=4" "-DBSIDMAP_APP_MINB_PRE=5"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  echo "=== variant: '$V' (auto KP)"; run
  echo "=== variant: '$V' KP=0"; BSIDMAP_APP_KP=0 run
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
