#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over GPU test subsets (small batches of every
# schedule and core: spec units, run-time compiled shapes, live-window APP, local and slab schedules).
# usage (under gpurun): bash tools/gpu_sanitize.sh <tag>
TAG=${1:-san}; OUT=gpurun_out/$TAG; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
MEM="c1_parity or c2_parity or c3_parity or c5_shape or live_window or jit_shape_parity or edge_configuration or status or floor or next or mc or slab or recompute_parity"
RACE="c1_parity or c2_parity or c3_parity or live_window_app_mixed or jit_shape_parity or slab_lengths or slab_chunked"
SYNC="c2_parity or c3_parity or live_window_app_mixed or jit_shape_parity or slab_lengths"
for tool in memcheck racecheck synccheck; do
  case $tool in memcheck) K=$MEM;; racecheck) K=$RACE;; synccheck) K=$SYNC;; esac
  timeout 1500 $CS --tool $tool --print-limit 20 python -m pytest tests -q -m gpu -p no:cacheprovider -k "$K" \
    > $OUT/$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|hazard" $OUT/$tool.log | tail -4
done
