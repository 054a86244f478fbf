#!/bin/bash
# CTA alpha/beta kernel (C3: M_tau 267, C4: 611): TMA ring depth and block size
make -j$(nproc) >/dev/null 2>&1
python tools/ktime.py C3:2048 C4:512 --iters 5
for ST in 1 2 3; do for TH in 0 320 160; do
  BSIDMAP_AB_CTA_STAGES=$ST BSIDMAP_AB_CTA_THREADS=$TH KTAG="[stages=$ST threads=$TH]" python tools/ktime.py C3:2048 C4:512 --iters 5
done; done
