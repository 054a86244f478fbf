#!/bin/bash
# the pair live-APP's CTAs per SM (register cap) with the float2 builtins: C1/C2 shapes
OUT=gpurun_out/exp_liveminb; mkdir -p $OUT
for v in 4 3; do
  touch paper_1802_08483_b200/csrc/*.cu
  make -s -j16 all EXTRA="-DBSIDMAP_LIVE_MINB=$v" > $OUT/build_$v.log 2>&1 || { tail $OUT/build_$v.log; continue; }
  echo "LIVE_MINB=$v"; timeout 300 python tools/ktime.py C2:65536 C4:512 2>&1 | tail -2
done
