#!/bin/bash
# pass-1 variants on the float2 pair cores (compile-time): symbol indices per CTA, row groups,
# CTAs/SM of the register-heavy shapes.  ktime per-phase device times.
OUT=gpurun_out/exp_p1f2; mkdir -p $OUT
for v in "" "-DBSIDMAP_L1_STEPS=16" "-DBSIDMAP_L1_GROUP=2" "-DBSIDMAP_L1C_MINB_LOW=2" "-DBSIDMAP_L1_GROUP=1"; do
  touch paper_1802_08483_b200/csrc/*.cu
  make -s -j16 all EXTRA="$v" > $OUT/build.log 2>&1 || { tail $OUT/build.log; continue; }
  echo "[$v]"; timeout 300 python tools/ktime.py C2:65536 C3:2048 C4:512 C5:32 2>&1 | tail -4 | awk '{print $1, "pass1", $12}'
done
