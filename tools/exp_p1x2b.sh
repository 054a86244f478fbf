#!/bin/bash
# pair pass 1 at 3 CTAs/SM for the 2-CTA shapes (default now) vs scalar pass 1; C4 at 3 vs 2
for V in "" "-DBSIDMAP_SCALAR_L1=1" "-DBSIDMAP_L1C_MINB_LOW=2"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py C3:2048 C5:32 C4:512 C2:65536 --iters 3
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
