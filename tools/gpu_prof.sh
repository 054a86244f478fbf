#!/bin/bash
# Profile one config on the GPU box: bench line, launch list (serialised per-launch times) and one
# `ncu --set full` capture of the lattice / alpha-beta kernels with the executed-FP32 op counters.
# The report is summarised on the box (tools/ncu_summary.py, tools/sass_mix.py: gpurun brings back
# at most 64 MiB) and kept only when KEEP_REP=1.  The source digest the capture was taken at goes
# beside it (bench.py refuses a stale capture).
# usage (under gpurun): bash tools/gpu_prof.sh <tag> <config> [frames] [extra bench args...]
TAG=${1:-r02}; CFG=${2:-C2}; NF=${3:-}; shift $(( $# < 3 ? $# : 3 ))
OUT=gpurun_out/$TAG/$CFG; mkdir -p $OUT
FR=${NF:+--frames $NF}
python -c "from paper_1802_08483_b200._lib import source_digest; print(source_digest())" > $OUT/digest.txt
python bench.py --config $CFG $FR "$@" > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --config $CFG $FR --steps 2 --warmup 1 --no-cpu-baseline --no-e2e "$@" > $OUT/launches.log 2>&1
EXTRA=smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
ncu --set full --metrics $EXTRA --clock-control none --import-source on -k regex:"${NCU_KERNELS:-k_gamma_sum|k_app|k_alpha_beta|k_live}" -c ${NCU_COUNT:-4} \
    -o $OUT/prof python bench.py --config $CFG $FR --steps 1 --warmup 0 --no-cpu-baseline --no-e2e "$@" > $OUT/ncu.log 2>&1
NF2=$(python -c "import json; print(json.load(open('$OUT/bench.json'))['config']['frames_per_gpu'])" 2>/dev/null || echo ${NF:-0})
python tools/ncu_summary.py ${TAG} $OUT $CFG $NF2 --no-write > $OUT/ncu_summary.md 2>&1
for k in k_gamma_sum k_app k_alpha_beta; do python tools/sass_mix.py $OUT/prof.ncu-rep $k 20 > $OUT/sass_mix_$k.txt 2>&1; done
ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
[ "${KEEP_REP:-0}" = "1" ] || rm -f $OUT/prof.ncu-rep
ls -la $OUT; cat $OUT/bench.json
