#!/bin/bash
# slab backward sweep on the alpha support: slab/recompute tests, timing vs Gamma-sum (C5, C4, C2) and
# the default path's phases (pass-1 regression check).  usage: bash tools/gpu_slab3.sh <tag>
TAG=${1:-slab4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
make -s > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -k "slab or recompute or c3_parity or c4_parity or c5_shape or modes_agree or soft_boundary or underflow" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 900 python tools/exp_slab.py C5:32 C4:512 C3:2048 C2:65536 > $OUT/exp_slab.jsonl 2> $OUT/exp_slab.err; cat $OUT/exp_slab.jsonl
timeout 600 python tools/ktime.py C2:65536 C5:32 > $OUT/ktime.txt 2>&1; cat $OUT/ktime.txt
