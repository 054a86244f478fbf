#!/bin/bash
# C3 / C5 pass 1: pair core at 3 CTAs/SM (168 registers, ~100 B spills) against the scalar core
# (look at the pass-1 column only: SCALAR_MN_MAX=16 also moves their APP to the pair core)
for V in "" "-DBSIDMAP_SCALAR_MN_MAX=16" "-DBSIDMAP_SCALAR_MN_MAX=16 -DBSIDMAP_L1C_MINB=3"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  BSIDMAP_AB_SUB=1 KTAG="[$V]" python tools/ktime.py C3:2048 C5:32 --iters 3
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
