#!/bin/bash
# C2 pass-2 variants through the create-time overrides: folded rows (KS) and prefix length (KP)
make -j$(nproc) >/dev/null 2>&1
python tools/ktime.py C2:65536 C1:16384
for KS in 1 2; do for KP in 2 3 4; do
  BSIDMAP_APP_KS=$KS BSIDMAP_APP_KP=$KP KTAG="[KS=$KS KP=$KP]" python tools/ktime.py C2:65536
done; done
