#!/bin/bash
# pass-1 / pass-2 variants (kernel tuning); each variant rebuilds the library
CFGS="C2:65536 C4:512 C3:2048 C5:32 C1:16384"
for V in "" "-DBSIDMAP_LATTICE_MIN_BLOCKS=3"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py $CFGS
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
