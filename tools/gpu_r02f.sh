#!/bin/bash
# JIT shapes on the GPU: tests, J1 bench (run-time compiled core vs the generic core), C2 bench, sanitizers.
TAG=${1:-r02f}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/build_smoke.log 2>&1 || { tail -30 $OUT/build_smoke.log; exit 1; }
tail -1 $OUT/build_smoke.log
timeout 1800 python -m pytest tests -q -m gpu -k "jit or live or c2_parity or c1_parity" --durations=8 > $OUT/pytest_gpu.log 2>&1; tail -12 $OUT/pytest_gpu.log
python bench.py --config J1 --no-cpu-baseline > $OUT/bench_J1.json 2> $OUT/bench_J1.err; tail -2 $OUT/bench_J1.err
BSIDMAP_JIT=0 python bench.py --config J1 --no-cpu-baseline --steps 3 --no-e2e > $OUT/bench_J1_generic.json 2> $OUT/bench_J1_generic.err
python bench.py --config C2 --no-cpu-baseline > $OUT/bench_C2.json 2> $OUT/bench_C2.err
for f in J1 J1_generic C2; do python -c "import json; d=json.load(open('$OUT/bench_$f.json')); print('$f', d['config']['core'], round(d['value'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],3))"; done
bash tools/gpu_sanitize.sh $TAG/san
