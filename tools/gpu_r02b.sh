#!/bin/bash
# Round-2 GPU pass: build + smoke, the gpu test suite, then bench line + launch list + ncu capture per config.
# usage (under gpurun): bash tools/gpu_r02b.sh <tag> "<pytest -k expr or empty>" <config:frames> ...
TAG=${1:-r02b}; K=${2:-}; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/build_smoke.log 2>&1
if [ "$K" != "skip" ]; then
  if [ -n "$K" ]; then timeout 2400 python -m pytest tests -q -m gpu -k "$K" --durations=10 > $OUT/pytest_gpu.log 2>&1
  else timeout 2400 python -m pytest tests -q -m gpu --durations=15 > $OUT/pytest_gpu.log 2>&1; fi
  tail -3 $OUT/pytest_gpu.log
fi
for cf in "$@"; do
  CFG=${cf%%:*}; NF=${cf#*:}
  timeout 1500 bash tools/gpu_prof.sh $TAG $CFG $NF
done
