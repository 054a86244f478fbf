#!/bin/bash
# Round-2 GPU pass: FP32/FP64 peak microbenchmark (clock-sampled), the gpu test suite, the C2 bench line.
# usage (under gpurun): bash tools/gpu_r02.sh <tag> [pytest -k expr]
TAG=${1:-r02}; K=${2:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nproc > $OUT/nproc.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv,noheader,nounits -lms 100 > $OUT/peak_clocks.csv &
SMI=$!
for i in 1 2 3; do ./tools/ubench/fp32_peak; done > $OUT/fp32_peak.txt 2>&1
kill $SMI
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/build_smoke.log 2>&1
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -q -m gpu -s -k "$K" > $OUT/pytest_gpu.log 2>&1
else
  timeout 2400 python -m pytest tests -q -m gpu -s --durations=15 > $OUT/pytest_gpu.log 2>&1
fi
python bench.py --config C2 > $OUT/bench_C2.json 2> $OUT/bench_C2.err
tail -5 $OUT/pytest_gpu.log; cat $OUT/bench_C2.json; cat $OUT/fp32_peak.txt
