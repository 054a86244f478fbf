#!/bin/bash
# Round-end style GPU pass: build, full gpu test suite, smoke, bench line, launch list, full ncu capture.
# usage (under gpurun): bash tools/gpu_round.sh <tag> [config]
TAG=${1:-r01}; CFG=${2:-C2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/build_smoke.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1
python bench.py --config $CFG > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_gamma_sum|k_app|k_alpha_beta' -c 3 \
    -o $OUT/prof python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $OUT/ncu.log 2>&1
tail -3 $OUT/pytest_gpu.log; cat $OUT/bench.json
