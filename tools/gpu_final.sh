#!/bin/bash
# Round-end evidence on one B200: build + smoke, the full GPU suite, then per config a bench line,
# a launch list and an ncu capture (summarised on the box), and the C1 latency.
TAG=${1:-r02_final}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/build_smoke.log 2>&1 || { tail -30 $OUT/build_smoke.log; exit 1; }
tail -1 $OUT/build_smoke.log
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 2400 python -m pytest tests -q -m gpu --durations=15 > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
fi
for cf in C2:65536 C5:32 C3:2048 C4:512 J1:65536; do
  CFG=${cf%%:*}; NF=${cf#*:}
  timeout 1500 bash tools/gpu_prof.sh $TAG $CFG $NF > /dev/null 2>&1
  python -c "import json; d=json.load(open('$OUT/$CFG/bench.json')); print('$CFG', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['phase_ms'].items()})" 2>&1 | tail -1
done
timeout 600 python tools/latency.py > $OUT/latency.json 2> $OUT/latency.err; cat $OUT/latency.json
