#!/bin/bash
# One GPU round: build, bench line, launch list, full ncu capture of the lattice kernels.
# usage (under gpurun): bash tools/gpu_profile.sh <tag> [config] [frames_for_ncu]
set -x
TAG=${1:-r01}; CFG=${2:-C2}; NF=${3:-65536}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python bench.py --config $CFG > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_gamma_sum|k_app<|k_alpha_beta' -c 3 \
    -o $OUT/prof python bench.py --config $CFG --frames $NF --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $OUT/ncu.log 2>&1
ls -la $OUT
