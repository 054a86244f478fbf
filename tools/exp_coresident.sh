#!/bin/bash
# alpha/beta co-residency: cap the lattice passes at 3 CTAs/SM through a dynamic-smem floor so that
# exactly one small alpha/beta block (2 warps: ~30 KB smem, 8K registers for C2) fits beside them,
# then overlap sub-batches (alpha/beta of sub-batch k on the side stream)
for V in "" "-DBSIDMAP_AB_WARP_THREADS=64"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py C2:65536
  for CAP in 57344 61440; do for S in 2 4; do
    BSIDMAP_PASS_SMEM_MIN=$CAP BSIDMAP_AB_SUB=$S KTAG="[$V cap$CAP sub$S]" python tools/ktime.py C2:65536
  done; done
done
