#!/bin/bash
# CTA alpha/beta kernel: finer sweep of (ring depth, block size) around the best of exp_abcta.sh
make -j$(nproc) >/dev/null 2>&1
for ST in 1 2; do for TH in 96 128 192 224 256 384; do
  BSIDMAP_AB_CTA_STAGES=$ST BSIDMAP_AB_CTA_THREADS=$TH KTAG="[stages=$ST threads=$TH]" python tools/ktime.py C3:2048 C4:512 --iters 5
done; done
for ST in 1 2; do for TH in 256 320 448; do
  BSIDMAP_AB_SUB=1 BSIDMAP_AB_CTA_STAGES=$ST BSIDMAP_AB_CTA_THREADS=$TH KTAG="[C5 sub1 stages=$ST threads=$TH]" python tools/ktime.py C5:32 --iters 3
done; done
BSIDMAP_AB_SUB=1 KTAG="[C5 sub1 default]" python tools/ktime.py C5:32 --iters 3
