#!/bin/bash
# C4 (M_n = 26): pair core vs scalar core, prefix lengths
for V in "" "-DBSIDMAP_SCALAR_MN_MAX=26"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  for KP in auto 0 3 4; do
    if [ "$KP" = auto ]; then unset BSIDMAP_APP_KP; else export BSIDMAP_APP_KP=$KP; fi
    KTAG="[$V KP=$KP]" python tools/ktime.py C4:512 C3:2048
  done
done
unset BSIDMAP_APP_KP
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
