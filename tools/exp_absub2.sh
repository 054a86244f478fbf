#!/bin/bash
# alpha/beta side-stream sub-batches after the alpha/beta instruction diet (C2, C3, C4)
make -s > /dev/null 2>&1
for S in 1 2 3 4; do echo "[AB_SUB=$S]"; BSIDMAP_AB_SUB=$S timeout 300 python tools/ktime.py C2:65536 C3:2048 C4:512 2>&1 | tail -3 | awk '{print $1, "total", $5}'; done
