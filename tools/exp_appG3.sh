#!/bin/bash
# frames per warp of the pair live APP (C2, C4): G = 8, 12, 16
make -s > /dev/null 2>&1
for G in 8 12 14 16; do echo "[G=$G]"; BSIDMAP_APP_G=$G timeout 300 python tools/ktime.py C2:65536 C4:512 2>&1 | tail -2 | awk '{print $1, "pass2", $17}'; done
