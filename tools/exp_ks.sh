#!/bin/bash
for KS in 1 2; do
  BSIDMAP_APP_KS=$KS KTAG="[KS=$KS]" python tools/ktime.py C2:65536 C4:512 C1:16384
done
