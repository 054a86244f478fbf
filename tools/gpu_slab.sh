#!/bin/bash
# The slab schedule on the GPU box: its tests, then the timing comparison (tools/exp_slab.py).
# usage (under gpurun): bash tools/gpu_slab.sh <tag> [pytest -k expr] [exp_slab specs...]
TAG=${1:-slab}; K=${2:-"slab or recompute or c3_parity or c4_parity or c5_shape or modes_agree or soft_boundary or extrinsic or edge_configuration or underflow or status_edge"}
shift $(( $# < 2 ? $# : 2 ))
OUT=gpurun_out/$TAG; mkdir -p $OUT
make -s > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "$K" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
SPECS=${@:-"C5:32 C4:512 C3:2048 C2:65536"}
timeout 1500 python tools/exp_slab.py $SPECS > $OUT/exp_slab.jsonl 2> $OUT/exp_slab.err; cat $OUT/exp_slab.jsonl; tail -3 $OUT/exp_slab.err
