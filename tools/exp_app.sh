#!/bin/bash
for V in "-DBSIDMAP_APP_PAIRS=true" "-DBSIDMAP_APP_MINB=5" "-DBSIDMAP_APP_MINB=5 -DBSIDMAP_APP_PAIRS=true"; do
  make clean >/dev/null; make -j16 EXTRA="$V" >/dev/null 2>&1
  echo "=== variant: $V"; python tools/quick_time.py C2 16384 3 | grep -E "TF/s|phases" | tail -2
done
make clean >/dev/null; make -j16 >/dev/null 2>&1
