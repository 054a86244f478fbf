#!/bin/bash
# alpha/beta warp kernel: warps per CTA and TMA ring depth (residency vs bytes in flight)
for V in "" "-DBSIDMAP_AB_WARP_THREADS=64" "-DBSIDMAP_AB_WARP_THREADS=32" "-DBSIDMAP_AB_WARP_THREADS=64 -DBSIDMAP_AB_STAGES=3" "-DBSIDMAP_AB_WARP_THREADS=32 -DBSIDMAP_AB_STAGES=3" "-DBSIDMAP_AB_WARP_THREADS=64 -DBSIDMAP_AB_STAGES=6" "-DBSIDMAP_AB_WARP_THREADS=32 -DBSIDMAP_AB_STAGES=2"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py C2:65536 C1:16384 --iters 5
done
