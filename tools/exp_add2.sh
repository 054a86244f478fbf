#!/bin/bash
# scalar class-ordered pass 1 (C3, C5): class-sum update fused into the last row's basic block, and
# row pairs instead of single rows (measured: fused C3 equal, C5 215.4 -> 221.7 ms; pairs slower; not kept)
for V in "-DBSIDMAP_L1_FUSED_ADD=0" "" "-DBSIDMAP_SCALAR_L1_GROUP=2"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  KTAG="[$V]" python tools/ktime.py C3:2048 C5:32 --iters 3
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
