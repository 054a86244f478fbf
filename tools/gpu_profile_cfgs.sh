#!/bin/bash
# launch list + ncu --set full of the main kernels for C3, C4, C5 at their per-GPU batches
for spec in C3:2048 C4:512 C5:32; do
  CFG=${spec%%:*}; NF=${spec##*:}; OUT=gpurun_out/${1:-r01f}_$CFG; mkdir -p $OUT
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py --config $CFG --frames $NF --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/launches.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:'k_gamma_sum|k_app|k_alpha_beta' -c 3 \
      -o $OUT/prof python bench.py --config $CFG --frames $NF --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $OUT/ncu.log 2>&1
  tail -1 $OUT/ncu.log
done
