#!/bin/bash
# C2 live-APP variants at run time (prefix bits KP, folded rows KS)
make -s > /dev/null 2>&1
for v in "" "BSIDMAP_APP_KP=2" "BSIDMAP_APP_KP=4" "BSIDMAP_APP_KP=0" "BSIDMAP_APP_KS=2" "BSIDMAP_APP_KS=2 BSIDMAP_APP_KP=2"; do
  echo "[$v]"; env $v timeout 300 python tools/ktime.py C2:65536 2>&1 | tail -1
done
