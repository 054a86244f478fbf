#!/bin/bash
# Live-window APP of the register-heavy shapes (C3, C5): scalar core (default) vs pair core (64-bit
# pairs), per-phase device times (tools/ktime.py)
OUT=gpurun_out/exp_apppair2; mkdir -p $OUT
for v in 20 0; do
  touch paper_1802_08483_b200/csrc/*.cu
  make -s -j16 all EXTRA="-DBSIDMAP_SCALAR_APP_MN_MAX=$v" > $OUT/build_$v.log 2>&1 || { tail $OUT/build_$v.log; continue; }
  for G in 0 4 8; do
    echo "scalar_app_mn_max=$v G=$G"; BSIDMAP_APP_G=$G timeout 300 python tools/ktime.py C3:2048 C5:32 2>&1 | tail -2
  done
done
