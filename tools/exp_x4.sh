#!/bin/bash
# four-window APP kernel vs two-window (C1, C2)
for X in 0 1; do
  for c in "C2 65536" "C1 16384"; do
    echo "=== BSIDMAP_APP_X4=$X $c"
    BSIDMAP_APP_X4=$X python tools/quick_time.py $c 0 | grep -E "frames/s" | tail -1
  done
done
