#!/bin/bash
# prefix length of the APP pass after the fused weight dot (C3, C4, C5 shapes)
make -j$(nproc) >/dev/null 2>&1
for KP in 0 2 3 4; do
  BSIDMAP_APP_KP=$KP KTAG="[KP=$KP]" python tools/ktime.py C3:2048 C4:512 C5:32 --iters 5
done
python -c "
import bsidgen
from paper_1802_08483_b200 import Decoder
for c,F in (('C3',2048),('C4',512),('C5',32)):
    cfg=bsidgen.configs()[c]; b=bsidgen.make_batch(cfg,0,2); d=Decoder.from_config(cfg,b.C,mode=0,device=0); print(c, d.plan(F))
"
