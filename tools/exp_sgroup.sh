#!/bin/bash
for V in "" "-DBSIDMAP_SCALAR_GROUP=1"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py C3:2048 C5:32
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
