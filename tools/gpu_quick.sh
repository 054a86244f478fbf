#!/bin/bash
# Quick GPU iteration: build, a pytest -k subset, and bench lines (no ncu).
# usage (under gpurun): bash tools/gpu_quick.sh <tag> "<pytest -k expr | skip>" <config[:frames]> ...
TAG=${1:-q}; K=${2:-skip}; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/build_smoke.log 2>&1 || { tail -20 $OUT/build_smoke.log; exit 1; }
tail -1 $OUT/build_smoke.log
if [ "$K" != "skip" ]; then
  timeout 1800 python -m pytest tests -q -m gpu -x -k "$K" > $OUT/pytest_gpu.log 2>&1
  tail -15 $OUT/pytest_gpu.log
fi
for cf in "$@"; do
  CFG=${cf%%:*}; NF=${cf#*:}; [ "$NF" = "$cf" ] && NF=""
  timeout 900 python bench.py --config $CFG ${NF:+--frames $NF} --no-cpu-baseline > $OUT/bench_$CFG.json 2> $OUT/bench_$CFG.err
  python -c "import json,sys; d=json.load(open('$OUT/bench_$CFG.json')); print('$CFG', round(d['value'],2), 'frames/s', round(d['ms_per_step'],2), 'ms', {k: round(v,2) for k,v in d['phase_ms'].items()}, 'e2e', round(d['e2e']['value'],1))" || tail -5 $OUT/bench_$CFG.err
done
