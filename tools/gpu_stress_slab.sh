#!/bin/bash
# randomized parity stress with the slab schedule as RECOMPUTE (default slab length, and 3 symbol
# indices per slab: many slabs, ragged last ones)
OUT=gpurun_out/stress_slab; mkdir -p $OUT
make -s > /dev/null 2>&1
timeout 1200 python tools/stress.py 300 31 > $OUT/seed31.log 2>&1; tail -2 $OUT/seed31.log
BSIDMAP_SLAB_LEN=3 timeout 1200 python tools/stress.py 300 32 > $OUT/seed32_len3.log 2>&1; tail -2 $OUT/seed32_len3.log
