#!/bin/bash
for PRE in 0 1; do
  BSIDMAP_L1_PRE=$PRE KTAG="[L1_PRE=$PRE]" python tools/ktime.py C2:65536 C4:512 C1:16384
done
