#!/bin/bash
# Profile one config on the GPU box: bench line, launch list (serialised per-launch times) and one
# `ncu --set full` capture of the lattice / alpha-beta kernels with the executed-FP32 op counters.
# The source digest the capture was taken at goes beside it (bench.py refuses a stale capture).
# usage (under gpurun): bash tools/gpu_prof.sh <tag> <config> [frames] [extra bench args...]
TAG=${1:-r02}; CFG=${2:-C2}; NF=${3:-}; shift 3 2>/dev/null
OUT=gpurun_out/$TAG/$CFG; mkdir -p $OUT
FR=${NF:+--frames $NF}
python -c "from paper_1802_08483_b200._lib import source_digest; print(source_digest())" > $OUT/digest.txt
python bench.py --config $CFG $FR "$@" > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --config $CFG $FR --steps 2 --warmup 1 --no-cpu-baseline --no-e2e "$@" > $OUT/launches.log 2>&1
EXTRA=smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
ncu --set full --metrics $EXTRA --clock-control none --import-source on -k regex:'k_gamma_sum|k_app|k_alpha_beta|k_local' -c 3 \
    -o $OUT/prof python bench.py --config $CFG $FR --steps 1 --warmup 0 --no-cpu-baseline --no-e2e "$@" > $OUT/ncu.log 2>&1
ls -la $OUT; cat $OUT/bench.json
