#!/bin/bash
for V in "" "-DBSIDMAP_LOCAL_CTA_MINB=1"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py C3:2048 C4:512 C5:32 --mode 2 --iters 2
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
