#!/bin/bash
for KS in 1 2; do
  BSIDMAP_APP_KS=$KS KTAG="[KS=$KS]" python tools/ktime.py C3:2048 C5:32 C4:512
done
