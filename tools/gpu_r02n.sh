#!/bin/bash
# Round-2 head check: build+smoke, the gpu test suite, bench lines for C2-C5 and J1, and the C2/C5
# launch lists + ncu captures at the same source digest (tools/gpu_prof.sh).
# usage (under gpurun): bash tools/gpu_r02n.sh <tag> [skip-tests]
TAG=${1:-r02n}; SKIP=${2:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nproc > $OUT/nproc.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/build_smoke.log 2>&1
echo "smoke exit $?" >> $OUT/build_smoke.log
if [ -z "$SKIP" ]; then
  timeout 1500 python -m pytest tests -q -m gpu --durations=15 > $OUT/pytest_gpu.log 2>&1
  tail -3 $OUT/pytest_gpu.log
fi
for c in C2 C3 C4 C5 J1; do
  timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  cat $OUT/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'))"
done
for c in C2 C5; do timeout 900 bash tools/gpu_prof.sh $TAG $c > /dev/null 2>&1; done
ls -R $OUT | head -50
