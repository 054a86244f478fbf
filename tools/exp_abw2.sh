#!/bin/bash
# alpha/beta warp kernel (M_tau <= 128) at 2 tasks per CTA: TMA ring depth
for V in "-DBSIDMAP_AB_STAGES=2" "-DBSIDMAP_AB_STAGES=3" "" "-DBSIDMAP_AB_STAGES=5" "-DBSIDMAP_AB_STAGES=8"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py C2:65536 C1:16384 --iters 5
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
