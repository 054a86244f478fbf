#!/bin/bash
# C3 / C5 APP: pair core at 3 CTAs/SM (165-168 registers, no spills with prefix sharing) vs the scalar
# core (default); KS = 1 (two weight tables; 3 CTAs fit the smem) and KS = 2
V="-DBSIDMAP_SCALAR_MN_MAX=16 -DBSIDMAP_APP_MINB_KS2=3 -DBSIDMAP_APP_MINB_PRE=3 -DBSIDMAP_APP_MINB=3 -DBSIDMAP_L1C_MINB=3"
make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; exit 1; }
for KS in 1 2; do
  BSIDMAP_APP_KS=$KS KTAG="[pair3 KS=$KS]" python tools/ktime.py C3:2048 C5:32 --iters 3
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
