#!/bin/bash
# ncu captures of the alpha/beta kernels: CTA form (C4) and warp form (C2)
OUT=gpurun_out/ab_prof; mkdir -p $OUT
ncu --set full --clock-control none --import-source on -k regex:'k_alpha_beta' -c 1 -o $OUT/ab_c4 \
  python tools/ktime.py C4:512 --iters 1 > $OUT/ab_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_alpha_beta_warp' -c 1 -o $OUT/ab_c2 \
  python tools/ktime.py C2:65536 --iters 1 > $OUT/ab_c2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_alpha_beta' -c 2 \
  python tools/ktime.py C2:65536 --iters 1 > $OUT/ab_c2_basic.log 2>&1
tail -5 $OUT/*.log
