#!/bin/bash
# Full GPU suite + C2 bench + C2 profile (ncu kernels: $NCU_KERNELS).  usage: bash tools/gpu_check.sh <tag>
TAG=${1:-check}
OUT=gpurun_out/$TAG; mkdir -p $OUT
make -s > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/build_smoke.log 2>&1; tail -1 $OUT/build_smoke.log
timeout 1500 python -m pytest tests -q -m gpu --durations=10 > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 900 bash tools/gpu_prof.sh $TAG C2 65536 > /dev/null 2>&1
python -c "import json; d=json.load(open('$OUT/C2/bench.json')); print(d['value'], d['ms_per_step'], d['phase_ms'])"
grep -A12 "launch list" $OUT/C2/ncu_summary.md
