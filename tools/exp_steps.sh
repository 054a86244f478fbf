#!/bin/bash
# symbol indices per CTA in the pass-1 pair-core kernel (prefetch of the next step's words)
for V in "" "-DBSIDMAP_APP_STEPS=1" "-DBSIDMAP_APP_STEPS=4" "-DBSIDMAP_APP_STEPS=16"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py C2:65536 C4:512 C1:16384
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
