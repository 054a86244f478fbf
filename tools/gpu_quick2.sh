#!/bin/bash
# quick check of a kernel change: a parity subset and the per-phase device times.  usage: bash tools/gpu_quick2.sh <tag> [-k expr]
TAG=${1:-q}; K=${2:-"live or c2_parity or c3_parity or c5_shape or slab_lengths or bench_batch or modes_agree"}
OUT=gpurun_out/$TAG; mkdir -p $OUT
make -s > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -k "$K" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 600 python tools/ktime.py C2:65536 C3:2048 C4:512 C5:32 > $OUT/ktime.txt 2>&1; cat $OUT/ktime.txt
