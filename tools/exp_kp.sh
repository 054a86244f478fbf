#!/bin/bash
# pass-2 prefix sharing: BSIDMAP_APP_KP = 0 (off) vs automatic vs forced lengths, per config
for c in "C2 65536" "C3 2048" "C4 512" "C5 32" "C1 16384"; do
  for KP in 0 auto 2 3 4; do
    if [ "$KP" = auto ]; then unset BSIDMAP_APP_KP; else export BSIDMAP_APP_KP=$KP; fi
    echo "=== $c KP=$KP"
    python tools/quick_time.py $c 0 | grep -E "frames/s|phases|app_prefix" | tail -2
  done
done
